set -u
mkdir -p gpurun_out/ab
SSH_DTW_PAIRED_WIDE=1 timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -m "gpu and not slow" -k "wide or dtw or query or exact" > gpurun_out/ab/t.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab/t.log
run() { timeout 300 python scripts/ab_dtw.py "$@" >> gpurun_out/ab/ab.jsonl 2>>gpurun_out/ab/err.log; }
A3="--cfg 3 --n 1000000 --nq 200"
run $A3 --tag legacy
SSH_DTW_PAIRED_WIDE=1 run $A3 --tag dvs_mb2
SSH_DTW_PAIRED_WIDE=1 SSH_LIB_PATH=abvar/dvs_mb3.so run $A3 --tag dvs_mb3
SSH_DTW_PAIRED_WIDE=1 SSH_LIB_PATH=abvar/dvs_mb4.so run $A3 --tag dvs_mb4
tail -2 gpurun_out/ab/t.log
