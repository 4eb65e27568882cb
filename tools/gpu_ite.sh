T="tests/test_gpu_peps.py -q -k run_ite_energies"
for cfg in "1 auto" "0 auto" "1 dc" "0 dc"; do set -- $cfg
echo "small=$1 eig=$2"; PEPSB_GEMM_SMALL=$1 PEPSB_EIG=$2 timeout 600 python -m pytest $T -m gpu 2>&1 | grep -E "passed|failed|^E  .*assert"
done
timeout 900 python -m pytest tests/test_gpu_eigh.py -q -x 2>&1 | tail -2
timeout 300 python tools/eig_timing.py 2>&1 | tail -12
