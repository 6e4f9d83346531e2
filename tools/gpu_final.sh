# Round-end evidence: full GPU tests (parity maxima logged), shape-scene maxima, bench lines, drop-in
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/final/gpu.txt 2>&1
VROD_PARITY_LOG=gpurun_out/final/parity_maxima.json timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/final/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/final/gputest.log
timeout 300 python tools/parity_maxima.py > gpurun_out/final/shape_maxima.json 2> gpurun_out/final/shape_maxima.err
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout 900 python bench.py --impl reference --steps 200 --warmup 10 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
for s in floor stretch wave activation bergou band bench; do ./integration/_build/vrod_b200_bench builtin:$s --steps 100 --impl both --exact --phases; done > gpurun_out/final/dropin_bench.txt 2>&1
./integration/_build/vrod_b200_solver_tests -tce="predict_rod applies" -tce="warm_start_lbs advances" > gpurun_out/final/dropin_tests.txt 2>&1
