set -x
STEPS=100 timeout 300 python tools/repro_ite_contract.py 0 /tmp/ite100.npz > gpurun_out/save.log 2>&1
PEPSB_DUMP_EIG=gpurun_out/last_gram.bin PEPSB_SYNC_DEBUG=1 timeout 600 python tools/repro_ite_contract.py 0 /tmp/ite100.npz > gpurun_out/trace.log 2>&1; echo rc $?
tail -3 gpurun_out/trace.log
timeout 60 python tools/eig_case.py gpurun_out/last_gram.bin 1 > gpurun_out/eig_jacobi.log 2>&1; echo rcj $?
timeout 60 python tools/eig_case.py gpurun_out/last_gram.bin 0 > gpurun_out/eig_dc.log 2>&1; echo rcd $?
cat gpurun_out/eig_jacobi.log gpurun_out/eig_dc.log | tail -8
timeout 300 python tools/dbg_eigh.py 0 > gpurun_out/dbg_eigh.log 2>&1
