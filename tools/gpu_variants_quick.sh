# per-program step times (bench, no CPU leg) for every build/variants/*.so, then the default library
for so in build/variants/*.so; do
  echo "== $so"
  FV3B_LIB=$PWD/$so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | grep -o '"kernels_ms_per_step": {[^}]*}\|"ms_per_step": [0-9.]*' | head -2
done
echo "== default"; timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | grep -o '"kernels_ms_per_step": {[^}]*}\|"ms_per_step": [0-9.]*' | head -2
