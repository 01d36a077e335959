#!/bin/bash
# ncu captures of this round (run under gpurun; outputs in gpurun_out/prof/):
# per-kernel metrics of one build + one query batch for configs[1..3]
# (profile_once.py brackets them with cudaProfilerStart/Stop), the launch list
# of the bench command, and --set full of single kernels.
#   bash scripts/profile_r02.sh met1 met2 met3 launches full_<kernel-regex>[@skip] ...
set -u
O=gpurun_out/prof
mkdir -p $O
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active
python -c "import sys; sys.path.insert(0,'.'); from paper_1610_07328_b200 import _native; _native.lib()"
for w in "$@"; do
  case $w in
    met1|met2|met3)
      c=${w#met}; nq=1000; [ $c = 3 ] && nq=200
      timeout 1500 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/met_cfg$c.csv \
        python scripts/profile_once.py --cfg $c --nq $nq > $O/met_cfg$c.log 2>&1
      echo "met cfg$c rc=$?" ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file $O/launches_cfg1.csv \
        python bench.py --steps 2 --warmup 1 --no-extra --no-e2e --no-cpu-baseline > $O/launches.log 2>&1
      echo "launches rc=$?" ;;
    full_*|full3_*)
      spec=${w#full_}; spec=${spec#full3_}; spec=${spec#3_}; k=${spec%@*}; skip=0; [ "$spec" != "$k" ] && skip=${spec#*@}
      cfg=1; n=""; case $k in dtw32w*) cfg=3;; esac
      case $w in full3_*) cfg=3; n="--n 1000000";; esac
      timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$k \
        --launch-skip $skip -c 1 -o $O/full_$k python scripts/profile_once.py --cfg $cfg $n --nq 1000 > $O/full_$k.log 2>&1
      echo "full $k rc=$?"
      # reports are large (gpurun copies back <= 64 MiB): keep the details page
      # and the per-line source summary, drop the report
      ncu -i $O/full_$k.ncu-rep --page details --csv > $O/full_${k}_details.csv 2>/dev/null
      python scripts/ncu_lines.py $O/full_$k.ncu-rep "$k" --top 40 > $O/full_${k}_lines.txt 2>/dev/null
      rm -f $O/full_$k.ncu-rep ;;
  esac
done
