# quick GPU iteration: parity tests (subset via $1 pytest -k expr), bench without the CPU leg
set -x
K=${1:-"."}
timeout 900 python -m pytest tests -m gpu -q -x -k "$K" 2>&1 | tail -15 > gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
cat gpurun_out/gpu_tests.log; grep -o '"kernels_ms_per_step": {[^}]*}' gpurun_out/bench.log; grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench.log | head -1; tail -3 gpurun_out/bench.log | cut -c1-300
