# A/B: full GPU tests, C3 split (default + each env variant given as arguments), C4 probe
mkdir -p gpurun_out/ab3; rm -f gpurun_out/ab3/*
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab3/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/ab3/gputest.log
for v in "" "$@"; do echo "== $v" >> gpurun_out/ab3/c3.txt; env $v timeout 300 python tools/c3_split.py >> gpurun_out/ab3/c3.txt 2>&1; done
timeout 300 python tools/c4_probe.py > gpurun_out/ab3/c4.txt 2>&1
