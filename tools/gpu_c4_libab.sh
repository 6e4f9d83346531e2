# C4 probe under library variants (VROD_B200_VARIANT names; "base" = default build)
mkdir -p gpurun_out/c4ab; rm -f gpurun_out/c4ab/*
for v in "$@"; do echo "== $v" >> gpurun_out/c4ab/c4.txt
  if [ "$v" = base ]; then timeout 300 python tools/c4_probe.py >> gpurun_out/c4ab/c4.txt 2>&1;
  else VROD_B200_VARIANT=$v timeout 300 python tools/c4_probe.py >> gpurun_out/c4ab/c4.txt 2>&1; fi
done
