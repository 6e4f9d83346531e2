# C3: split + phase trace + launch list of the current build (gpurun_out/c3p/)
mkdir -p gpurun_out/c3p
timeout 300 python tools/c3_split.py > gpurun_out/c3p/split.txt 2>&1
timeout 300 python tools/trace_iterate.py > gpurun_out/c3p/trace.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c3p/launches.csv python tools/profile_step.py C3 3 > /dev/null 2>&1
