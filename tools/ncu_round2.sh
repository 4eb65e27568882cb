# Launch list of one config-2 row (second step) + ncu --set full of the complex x real and 3M/4M top GEMMs.
set -x
export PEPSB_PROF_STEPS=2
true ||
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python tools/prof_step.py > gpurun_out/ncu_list.log 2>&1
python tools/prof_step.py > gpurun_out/plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:\(int\)1, \(int\)2>' -s ${SKIP:-160} -c ${COUNT:-1} \
    -o gpurun_out/prof_cr python tools/prof_step.py > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out; tail -3 gpurun_out/ncu_full.log
