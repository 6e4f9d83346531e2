# C3 A/B of library variants (VROD_B200_VARIANT names; "base" = the default build), interleaved x4
mkdir -p gpurun_out/c3ab; rm -f gpurun_out/c3ab/*
for rep in 1 2 3 4; do for v in "$@"; do
  if [ "$v" = base ]; then timeout 300 python tools/c3_once.py >> gpurun_out/c3ab/c3.txt 2>&1;
  else VROD_B200_VARIANT=$v timeout 300 python tools/c3_once.py >> gpurun_out/c3ab/c3.txt 2>&1; fi
done; done
