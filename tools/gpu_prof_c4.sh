# C4 source-level profiles of the current build: the sweep + ext pair, then the collision kernels
# (each ncu run after the plain workload exited 0). Outputs: gpurun_out/p4/.
mkdir -p gpurun_out/p4
timeout 300 python tools/profile_step.py C4 1 > gpurun_out/p4/plain.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_rod_sweep_warp|k_ext_solve" -s 20 -c 2 -o gpurun_out/p4/sweep python tools/profile_step.py C4 1 > gpurun_out/p4/ncu1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_pairs_cell|k_seg_filter|k_ext_sort|k_ext_fill|k_report_tail|k_ct_scatter" -s 6 -c 6 -o gpurun_out/p4/collide python tools/profile_step.py C4 1 > gpurun_out/p4/ncu2.log 2>&1
ls -la gpurun_out/p4
