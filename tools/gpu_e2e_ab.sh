# e2e anatomy A/B of library variants ("base" = default build), interleaved x3
mkdir -p gpurun_out/e2e; rm -f gpurun_out/e2e/ab.txt
for rep in 1 2 3; do for v in "$@"; do
  if [ "$v" = base ]; then echo -n "base " >> gpurun_out/e2e/ab.txt; timeout 300 python tools/e2e_probe2.py >> gpurun_out/e2e/ab.txt 2>&1;
  else echo -n "$v " >> gpurun_out/e2e/ab.txt; VROD_B200_VARIANT=$v timeout 300 python tools/e2e_probe2.py >> gpurun_out/e2e/ab.txt 2>&1; fi
done; done
