for e in dc jacobi; do
PEPSB_EIG=$e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-norms > gpurun_out/bench_e.json 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bench_e.json').read().strip().splitlines()[-1]); r=d['roofline']; print('eig=$e', round(d['ms_per_step'],2), r['breakdown_ms'])"
done
PEPSB_PROF_STEPS=1 PEPSB_TRACE_GEMM=1 timeout 300 python tools/prof_step.py 2> gpurun_out/trace2.log >/dev/null; grep -c zgemm gpurun_out/trace2.log
