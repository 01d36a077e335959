set -u
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -m "gpu and not slow" > gpurun_out/ab/t.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab/t.log
run() { timeout 300 python scripts/ab_dtw.py "$@" >> gpurun_out/ab/ab.jsonl 2>>gpurun_out/ab/err.log; }
A1="--cfg 1 --nq 1000 --reps 3"; A2="--cfg 2 --n 1000000 --nq 200"
for A in "$A1" "$A2"; do run $A --tag db4; SSH_LIB_PATH=abvar/wl_db3.so run $A --tag db3; SSH_LIB_PATH=abvar/wl_lb4.so run $A --tag single_lb4; done
tail -2 gpurun_out/ab/t.log
