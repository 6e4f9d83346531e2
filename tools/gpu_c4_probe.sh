mkdir -p gpurun_out/p3
./tools/ubench/divcheck > gpurun_out/p3/divcheck.txt 2>&1
for mb in 3 4 5; do VROD_WARP_MINB=$mb timeout 300 python tools/c4_probe.py > gpurun_out/p3/c4_minb$mb.txt 2>&1; done
VROD_WARP_TMA=0 timeout 300 python tools/c4_probe.py > gpurun_out/p3/c4_notma.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_pairs_cell|k_seg_filter|k_narrow_append|k_ext_sort|k_ct_scatter|k_ext_fill|k_ext_count|k_report" -s 40 -c 8 -o gpurun_out/p3/c4_collide python tools/profile_step.py C4 2 > gpurun_out/p3/ncu.log 2>&1
