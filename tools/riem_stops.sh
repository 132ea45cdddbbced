# isolated riem timings (tools/microbench.py nh_d) for every build/variants/*.so and the default build
for so in build/variants/*.so; do echo "== $so"; FV3B_LIB=$PWD/$so timeout 300 python tools/microbench.py nh_d 2>&1 | tail -1; done > gpurun_out/rs.log
echo "== default" >> gpurun_out/rs.log; timeout 300 python tools/microbench.py nh_d 2>&1 | tail -1 >> gpurun_out/rs.log
