# launch list (one eager C2 step, n_split=6) + ncu --set full of the kernels matching $1 (n_split=1 step); tag $2
set -x
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$2.csv python tools/profile_step.py 6 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -c ${3:-12} -o gpurun_out/prof_$2 python tools/profile_step.py 1 1 > gpurun_out/ncu_$2.log 2>&1
tail -2 gpurun_out/ncu_$2.log
