# ncu --set full of kernels matching $1 (regex), count $2, in one eager C2 step (n_split=1); tag $3
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$1" -c ${2:-1} -o gpurun_out/prof_$3 python tools/profile_step.py 1 1 > gpurun_out/ncu_$3.log 2>&1
tail -3 gpurun_out/ncu_$3.log
