set -x
NORMS=1 PEPSB_TRACE_GEMM=1 timeout 300 python tools/prof_cfg1.py 2> gpurun_out/cfg1_trace.log; grep -c zgemm gpurun_out/cfg1_trace.log
NORMS=1 timeout 600 ncu --set full --clock-control none -k regex:zgemm_cx_kernel -s 300 -c 3 -o gpurun_out/cfg1_gemm python tools/prof_cfg1.py > gpurun_out/cfg1_ncu2.log 2>&1; echo ncu $?
NORMS=1 timeout 600 ncu --set full --clock-control none -k regex:gram_factors -s 60 -c 2 -o gpurun_out/cfg1_gf python tools/prof_cfg1.py > gpurun_out/cfg1_ncu3.log 2>&1; echo ncu $?
