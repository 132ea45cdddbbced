# quick iteration: parity subset ($1 = pytest -k expr), bench without the CPU leg, ncu --set full of kernels matching $2 (tag $3)
set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "$1" 2>&1 | tail -5 > gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
if [ -n "$2" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -c ${4:-2} -o gpurun_out/prof_$3 python tools/profile_step.py 1 1 > gpurun_out/ncu_$3.log 2>&1
fi
cat gpurun_out/gpu_tests.log; grep -o '"kernels_ms_per_step": {[^}]*}' gpurun_out/bench.log; grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench.log | head -1
