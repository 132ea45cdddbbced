# compute-sanitizer over one small eager timestep: memory errors, shared-memory
# races, barrier misuse (summaries into gpurun_out/sanitize_*.txt)
# (memcheck with the caching allocator off: every tensor its own allocation, so
# a read past a field's end is caught rather than landing in a neighbour)
for tool in memcheck racecheck synccheck; do
  nc=0; [ $tool = memcheck ] && nc=1
  PYTORCH_NO_CUDA_MEMORY_CACHING=$nc timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_step.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$tool.txt
done
tail -n 4 gpurun_out/sanitize_*.txt
