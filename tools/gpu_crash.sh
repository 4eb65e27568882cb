set -x
timeout 60 python tools/eig_case.py gpurun_out/last_gram.bin 0 > gpurun_out/eig_dc.log 2>&1; echo rcd $?
timeout 600 python -m pytest tests/test_gpu_eigh.py -x -q 2>&1 | tail -3
STEPS=100 timeout 300 python tools/repro_ite_contract.py 0 /tmp/ite100.npz > gpurun_out/save.log 2>&1
timeout 600 python tools/repro_ite_contract.py 0 /tmp/ite100.npz > gpurun_out/trace.log 2>&1; echo rc $?
tail -3 gpurun_out/trace.log
timeout 900 python tools/bench_configs.py --configs 4 --ref > gpurun_out/cfg4.jsonl 2>&1; tail -2 gpurun_out/cfg4.jsonl
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
