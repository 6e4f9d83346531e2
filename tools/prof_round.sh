set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/p1
timeout 300 python tools/profile_step.py C4 2 > gpurun_out/p1/plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p1/c4_launches.csv python tools/profile_step.py C4 2 > gpurun_out/p1/ncu_l.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_rod_sweep|k_ext_solve|k_pairs|k_narrow|k_seg_filter|k_ext_sort" -s 60 -c 8 -o gpurun_out/p1/c4_full python tools/profile_step.py C4 2 > gpurun_out/p1/ncu_f.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/p1/c3_launches.csv python tools/profile_step.py C3 3 > gpurun_out/p1/ncu_l3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_rod_sweep|k_ext_solve|k_shape" -s 200 -c 6 -o gpurun_out/p1/c3_full python tools/profile_step.py C3 3 > gpurun_out/p1/ncu_f3.log 2>&1
ls -la gpurun_out/p1
