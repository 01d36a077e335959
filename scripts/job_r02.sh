mkdir -p gpurun_out/ab
for v in n2 n3; do SSH_LIB_PATH=abvar/dp_$v.so timeout 300 python scripts/ab_dtw.py --cfg 1 --nq 1000 --reps 3 --tag $v >> gpurun_out/ab/ab.jsonl 2>>gpurun_out/ab/err.log; done
timeout 300 python scripts/ab_dtw.py --cfg 1 --nq 1000 --reps 3 --tag n1 >> gpurun_out/ab/ab.jsonl 2>>gpurun_out/ab/err.log
bash scripts/profile_r02.sh met1 launches full_paa_members_kernel@1 full_cws_fast_kernel full_summaries_kernel full_wave_lb_kernel@3 full_dtwp_level@3 met2 met3
du -sh gpurun_out
