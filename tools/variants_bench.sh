# per-kernel step shares of the default build and of build/variants/*.so ($@ = variant names)
for v in default "$@"; do
  if [ "$v" = default ]; then L=""; else L="FV3B_LIB=build/variants/$v.so"; fi
  echo "== $v" >> gpurun_out/variants.log
  env $L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | grep -o '"kernels_ms_per_step": {[^}]*}\|^{"metric[^,]*, "value": [0-9.]*' >> gpurun_out/variants.log
done
