for so in build/variants/*.so; do
  echo "== $so"
  FV3B_LIB=$PWD/$so timeout 300 python -m pytest tests -m gpu -q -x -k "d_sw or dsw or levelmarch" 2>&1 | tail -2
  FV3B_LIB=$PWD/$so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | grep -o '"kernels_ms_per_step": {[^}]*}\|"ms_per_step": [0-9.]*' | head -2
done
echo "== default"; timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | grep -o '"kernels_ms_per_step": {[^}]*}\|"ms_per_step": [0-9.]*' | head -2
