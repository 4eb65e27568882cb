set -x
python tools/prof_cfg3.py > gpurun_out/plain_c3.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
    python tools/prof_cfg3.py > gpurun_out/ncu_c3.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c3.csv 1 25 > gpurun_out/launches_c3_summary.txt 2>&1
tail -30 gpurun_out/launches_c3_summary.txt
