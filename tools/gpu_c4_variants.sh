# C4 A/B over environment variants given as arguments ("" = defaults)
mkdir -p gpurun_out/ab3; rm -f gpurun_out/ab3/c4.txt
for v in "$@"; do echo "== $v" >> gpurun_out/ab3/c4.txt; env $v timeout 300 python tools/c4_probe.py >> gpurun_out/ab3/c4.txt 2>&1; done
