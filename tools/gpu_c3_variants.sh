# C3 split under environment variants given as arguments ("" = defaults), first two lines each
mkdir -p gpurun_out/c3v; rm -f gpurun_out/c3v/*
for v in "$@"; do echo "== $v" >> gpurun_out/c3v/c3.txt; env $v timeout 300 python tools/c3_split.py 2>&1 | head -2 >> gpurun_out/c3v/c3.txt; done
