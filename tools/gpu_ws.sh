set -x
timeout 900 python -m pytest tests/test_gpu_core.py -x -q -k "gemm" 2>&1 | tail -15
PEPSB_GEMM_WS=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ws0.json 2>gpurun_out/bench_ws0.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ws1.json 2>gpurun_out/bench_ws1.err
PEPSB_GEMM=4c timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ws1_4c.json 2>gpurun_out/bench_ws1_4c.err
STEPS=100 timeout 300 python tools/repro_ite_contract.py 0 /tmp/ite100.npz > gpurun_out/save.log 2>&1
PEPSB_SYNC_DEBUG=1 PEPSB_TRACE_GEMM=1 PEPSB_TRACE=1 timeout 600 python tools/repro_ite_contract.py 0 /tmp/ite100.npz > gpurun_out/trace.log 2>&1; echo rc $?
tail -30 gpurun_out/trace.log
