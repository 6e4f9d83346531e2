# A/B probe: full GPU tests, C4 probe, C3 bench line (no extras); optional ncu of $NCU_REGEX on C4
mkdir -p gpurun_out/ab
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/ab/gputest.log
timeout 300 python tools/c4_probe.py > gpurun_out/ab/c4.txt 2>&1
timeout 600 python bench.py --no-secondary --no-batch --no-skin --no-extra --cpu-seconds 1 > gpurun_out/ab/bench.json 2> gpurun_out/ab/bench.err
if [ -n "$NCU_REGEX" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$NCU_REGEX" -s ${NCU_SKIP:-0} -c ${NCU_COUNT:-8} -o gpurun_out/ab/ncu python tools/profile_step.py ${NCU_CFG:-C4} 2 > gpurun_out/ab/ncu.log 2>&1
fi
