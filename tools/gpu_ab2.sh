# A/B: full GPU tests, then the C4 probe under each environment variant given as arguments
mkdir -p gpurun_out/ab2; rm -f gpurun_out/ab2/*
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab2/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/ab2/gputest.log
for v in "$@"; do echo "== $v" >> gpurun_out/ab2/c4.txt; env $v timeout 300 python tools/c4_probe.py >> gpurun_out/ab2/c4.txt 2>&1; done
