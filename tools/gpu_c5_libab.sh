# C5 breakdown under library variants ("base" = default build); scenes from $C5N (default 2048)
mkdir -p gpurun_out/c5ab; rm -f gpurun_out/c5ab/*
for v in "$@"; do echo "== $v" >> gpurun_out/c5ab/c5.txt
  if [ "$v" = base ]; then timeout 600 python tools/c5_breakdown.py ${C5N:-2048} >> gpurun_out/c5ab/c5.txt 2>&1;
  else VROD_B200_VARIANT=$v timeout 600 python tools/c5_breakdown.py ${C5N:-2048} >> gpurun_out/c5ab/c5.txt 2>&1; fi
done
