timeout 600 python -m pytest tests -m gpu -q -x -k "fv_tp_2d" 2>&1 | tail -2 > gpurun_out/tp.log
timeout 300 python tools/microbench.py fv_tp_2d >> gpurun_out/tp.log 2>&1
