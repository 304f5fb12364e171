#!/bin/bash
# usage: tools/profile_walk.sh <config> <tag> [skip]  (run on the GPU box via gpurun)
# plain run, then the ncu launch list, then one full capture of k_walk (a later step)
CFG=${1:-1}; TAG=${2:-r1}; SKIP=${3:-3}
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_cfg${CFG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_cfg${CFG}_${TAG}.csv $CMD > gpurun_out/ncu_launch_cfg${CFG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_walk -s $SKIP -c 1 -o gpurun_out/walk_cfg${CFG}_${TAG} -f $CMD > gpurun_out/ncu_full_cfg${CFG}.log 2>&1
echo "exit $?"
tail -3 gpurun_out/ncu_full_cfg${CFG}.log
