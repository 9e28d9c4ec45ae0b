#!/bin/bash
# The round's ncu evidence (run under gpurun, one GPU):
#   1. --set full capture of the bench's walk kernel (k_walk_persistent) -> .ncu-rep
#   2. per-kernel DRAM bytes / time / issue activity of every kernel of the
#      walk (SP and TP), k-hop (SP and TP), dedup and collective workloads
#   3. the launch list of the bench command itself
# Outputs under gpurun_out/ncu_${TAG}_*; tools/ncu_summarize.py TAG turns them
# into profiles/${TAG}_ncu_summary.json.
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size,launch__registers_per_thread
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:k_walk_persistent -c 10 -o $O/ncu_${TAG}_walk_full -f \
  python tools/probe_ncu_round.py walk_sp > $O/ncu_${TAG}_walk_full.log 2>&1
echo "walk_full rc=$?"
for w in walk_sp walk_tp khop dedup collective; do
  timeout 900 ncu --metrics $M --clock-control none --profile-from-start off --csv \
    --log-file $O/ncu_${TAG}_${w}.csv python tools/probe_ncu_round.py $w > $O/ncu_${TAG}_${w}.log 2>&1
  echo "$w rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/ncu_${TAG}_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-tp --no-c3 --no-c5 > $O/ncu_${TAG}_launches_bench.log 2>&1
echo "launches rc=$?"
if [ -f $O/ncu_${TAG}_walk_full.ncu-rep ]; then
  ncu -i $O/ncu_${TAG}_walk_full.ncu-rep --page raw --csv > $O/ncu_${TAG}_walk_full_raw.csv 2>/dev/null
  ncu -i $O/ncu_${TAG}_walk_full.ncu-rep --page source --csv > $O/ncu_${TAG}_walk_full_source.csv 2>/dev/null
fi
ls -la $O | grep ncu_${TAG}
