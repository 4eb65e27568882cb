set -x
timeout 300 python tools/repro_ite_contract.py 0 > gpurun_out/repro0.log 2>&1; echo rc0 $?
PEPSB_TRACE_GEMM=1 timeout 300 python tools/repro_ite_contract.py 1 > gpurun_out/repro1.log 2>&1; echo rc1 $?
tail -3 gpurun_out/repro1.log
export PEPSB_PROF_STEPS=2
python tools/prof_step.py > gpurun_out/plain3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:zgemm_ws -s 150 -c 4 -o gpurun_out/prof_ws python tools/prof_step.py > gpurun_out/ncu_ws.log 2>&1
python tools/launch_summary.py 2>/dev/null | head -2
