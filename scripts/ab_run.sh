set -u
mkdir -p gpurun_out/ab
run() { timeout 300 python scripts/ab_dtw.py "$@" >> gpurun_out/ab/ab.jsonl 2>>gpurun_out/ab/err.log; }
A1="--cfg 1 --nq 1000 --reps 3"; A2="--cfg 2 --n 1000000 --nq 200"
for t in 16384 32768 65536 131072; do SSH_DEBUG_MEMBER_TARGET=$t run $A1 --tag t$t; done
for t in 16384 32768 65536; do SSH_DEBUG_MEMBER_TARGET=$t run $A2 --tag t$t; done
bash scripts/profile_r02.sh full3_summaries_kernel
