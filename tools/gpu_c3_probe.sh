# C3 probes: fixed vs per-iteration split, persistent-kernel phase trace, aux-CTA variant
mkdir -p gpurun_out/c3
timeout 300 python tools/c3_split.py > gpurun_out/c3/split.txt 2>&1
timeout 300 python tools/trace_iterate.py > gpurun_out/c3/trace.txt 2>&1
VROD_PERSIST_AUX=1 timeout 300 python tools/c3_split.py > gpurun_out/c3/split_aux.txt 2>&1
