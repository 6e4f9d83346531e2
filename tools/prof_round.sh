# Round profiling recipe (run on the GPU box from the repo root; each ncu command only after the
# same workload exited 0 without ncu). Outputs go to gpurun_out/prof/.
set -x
mkdir -p gpurun_out/prof
timeout 300 python tools/profile_step.py C3 3 > gpurun_out/prof/c3_plain.log 2>&1 || exit 1
timeout 300 python tools/profile_step.py C4 2 > gpurun_out/prof/c4_plain.log 2>&1 || exit 1
timeout 300 python tools/profile_skin.py 2 > gpurun_out/prof/skin_plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/c3_launches.csv python tools/profile_step.py C3 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/c4_launches.csv python tools/profile_step.py C4 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_iterate -s 3 -c 1 -o gpurun_out/prof/c3_iterate python tools/profile_step.py C3 3 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_rod_sweep|k_ext_solve|k_pairs_cell|k_narrow_append" -s 30 -c 5 -o gpurun_out/prof/c4_full python tools/profile_step.py C4 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_skin_deform -c 1 -o gpurun_out/prof/skin_deform python tools/profile_skin.py 2 > /dev/null 2>&1
ls -la gpurun_out/prof
