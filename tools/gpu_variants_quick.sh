# per-program step times (bench, no CPU leg) for every $1/*.so (default build/variants), then the default library
D=${1:-build/variants}
for so in $D/*.so; do
  echo "== $so"
  FV3B_LIB=$PWD/$so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | grep -o '"kernels_ms_per_step": {[^}]*}\|"ms_per_step": [0-9.]*' | sed -n '1p;$p'
done
echo "== default"; timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | grep -o '"kernels_ms_per_step": {[^}]*}\|"ms_per_step": [0-9.]*' | sed -n '1p;$p'
