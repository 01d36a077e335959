set -u
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -m "gpu and not slow" > gpurun_out/ab/t.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab/t.log
SSH_LIB_PATH=abvar/checked.so timeout 1200 python -m pytest tests -q -p no:cacheprovider -m "gpu and not slow" > gpurun_out/ab/checked.log 2>&1; echo "checked rc=$?" >> gpurun_out/ab/checked.log
run() { timeout 300 python scripts/ab_dtw.py "$@" >> gpurun_out/ab/ab.jsonl 2>>gpurun_out/ab/err.log; }
A1="--cfg 1 --nq 1000 --reps 3"
run $A1 --tag n1; SSH_LIB_PATH=abvar/dp_n2.so run $A1 --tag n2; SSH_LIB_PATH=abvar/dp_n3.so run $A1 --tag n3
SSH_LIB_PATH=abvar/checked.so run $A1 --tag checked
tail -2 gpurun_out/ab/t.log; tail -2 gpurun_out/ab/checked.log
