set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py 6 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'d_sw|riem|c_sw|tp_kernel|remap|p_grad' -c 12 -o gpurun_out/prof_r1a python tools/profile_step.py 1 1 > gpurun_out/ncu.log 2>&1
cat gpurun_out/gpu_tests.log gpurun_out/bench.log; tail -3 gpurun_out/ncu.log
