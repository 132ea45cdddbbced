# time the C2 step (graph replay + eager per-kernel shares) with every build/variants/*.so
for so in build/variants/*.so; do
  echo "== $so"
  FV3B_LIB=$PWD/$so timeout 300 python tools/stepbench.py 2>&1 | grep -v "^init"
done > gpurun_out/variants.log 2>&1
echo "== default" >> gpurun_out/variants.log
timeout 300 python tools/stepbench.py 2>&1 | grep -v "^init" >> gpurun_out/variants.log
