#!/bin/bash
# ncu captures of this round (run under gpurun; outputs in gpurun_out/):
# per-kernel metrics of one build + one 1000-query batch for configs[1..3],
# and --set full of the DTW kernels.  bash scripts/profile_r02.sh [what...]
set -u
O=gpurun_out/prof
mkdir -p $O
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active
python -c "import sys; sys.path.insert(0,'.'); from paper_1610_07328_b200 import _native; _native.lib()"
for w in "$@"; do
  case $w in
    met1|met2|met3)
      c=${w#met}
      timeout 1200 ncu --metrics $M --clock-control none --csv --log-file $O/met_cfg$c.csv \
        python scripts/profile_once.py --cfg $c --nq 1000 > $O/met_cfg$c.log 2>&1
      echo "met cfg$c rc=$?" ;;
    full_dtw3)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:dtw32w --launch-skip 1 -c 1 \
        -o $O/dtw32w_cfg3 python scripts/profile_once.py --cfg 3 --n 1000000 --nq 100 > $O/full_dtw3.log 2>&1
      echo "full dtw3 rc=$?" ;;
    full_dtw1)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:dtwp_level --launch-skip 3 -c 1 \
        -o $O/dtwp_cfg1 python scripts/profile_once.py --cfg 1 --nq 1000 > $O/full_dtw1.log 2>&1
      echo "full dtw1 rc=$?" ;;
    full_*)
      k=${w#full_}
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
        -o $O/$k python scripts/profile_once.py --cfg 1 --nq 1000 > $O/full_$k.log 2>&1
      echo "full $k rc=$?" ;;
  esac
done
