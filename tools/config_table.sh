#!/bin/bash
# usage (GPU box): bash tools/config_table.sh <tag> [configs]
# per config: one bench line (with the oracle cpu_baseline) and one ncu metric capture of the
# first timed k_walk launch (metric subset of BASELINE.md §4); read back by tools/config_table.py
TAG=${1:-r2}; CFGS=${2:-"0 1 2 3 4"}
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed_per_inst_executed.ratio,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__inst_executed.sum
for c in $CFGS; do
  python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/table_${TAG}_cfg$c.log 2>&1
  SKIP=3; [ "$c" = 4 ] && SKIP=24
  ncu --metrics $M --clock-control none -k regex:k_walk -s $SKIP -c 1 --csv \
      python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --nominal-peak \
      > gpurun_out/table_${TAG}_ncu_cfg$c.csv 2> gpurun_out/table_${TAG}_ncu_cfg$c.err
  echo "cfg $c done"
done
