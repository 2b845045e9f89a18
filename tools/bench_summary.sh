# one-line summaries of bench.py runs: bash tools/bench_summary.sh c1 c2 ...  (extra env applies)
for c in "$@"; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],2), {k:round(v,1) for k,v in d['phase_ms_per_step'].items()}, 'chol', round(d['cholesky_phase']['frac'],3), 'syrk', round(d['roofline']['frac'],3))"
done
