# Refresh the committed bench lines: bench.py --config cN (default FP64 DMMA path) for
# every BASELINE config, each line to gpurun_out/bench_cN.json
for c in ${CONFIGS:-c0 c1 c2 c3 c4}; do
  timeout 1500 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1
  echo "$c rc $?"
  tail -1 gpurun_out/bench_$c.log > gpurun_out/bench_$c.json
done
