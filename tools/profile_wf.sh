#!/bin/bash
# usage: tools/profile_wf.sh <config> <tag> [kernel-regex] [skip]  -- launch list + one full capture
CFG=${1:-1}; TAG=${2:-r1}; KRE=${3:-k_wf_trace}; SKIP=${4:-200}
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu --wavefront --hostloop"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_cfg${CFG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_cfg${CFG}_${TAG}.csv $CMD > gpurun_out/ncu_launch_cfg${CFG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c 1 -o gpurun_out/${KRE}_cfg${CFG}_${TAG} -f $CMD > gpurun_out/ncu_full_cfg${CFG}.log 2>&1
echo "exit $?"
tail -2 gpurun_out/ncu_full_cfg${CFG}.log
