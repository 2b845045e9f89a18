# C0 (single m = 4096 system): leaf phase trace, bench line, concurrent kernel trace
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k:round(v,3) for k,v in d['phase_ms_per_step'].items()}, round(d['cholesky_phase']['frac'],3))"; }
./tools/leaf_trace | tail -1
timeout 200 python bench.py --config c0 --no-cpu-baseline > gpurun_out/c0.log 2>&1; summ gpurun_out/c0.log
timeout 300 python tools/kernel_trace.py c0 > gpurun_out/trace_c0_new.txt 2>&1
