# round evidence: full GPU tests + smoke, bench (with the CPU leg), launch list, ncu full of one step
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/gpu_tests.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv python tools/profile_step.py 6 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -c 24 -k regex:"csw|riem|p_grad|dsw|tp_kernel|tracer2|remap|face|halo|moist" -o gpurun_out/prof_$1 python tools/profile_step.py 1 1 > gpurun_out/ncu_$1.log 2>&1
cat gpurun_out/gpu_tests.log; tail -c 3000 gpurun_out/bench.log
