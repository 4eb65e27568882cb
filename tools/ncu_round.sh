# Launch list, then one `ncu --set full` capture of a few GEMM launches of one interior column.
set -x
export PEPSB_PROF_STEPS=2
if [ "${LIST:-1}" = 1 ]; then
python tools/prof_step.py > gpurun_out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python tools/prof_step.py > gpurun_out/ncu_list.log 2>&1
fi
python tools/prof_step.py > gpurun_out/plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-zgemm_cx} -s ${SKIP:-270} -c ${COUNT:-8} \
    -o gpurun_out/prof python tools/prof_step.py > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out; du -sh gpurun_out
