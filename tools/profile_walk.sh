#!/bin/bash
# usage: tools/profile_walk.sh <config> <tag>   (run on the GPU box via gpurun)
CFG=${1:-1}; TAG=${2:-r1}
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_cfg${CFG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg${CFG}_${TAG}.csv $CMD > gpurun_out/ncu_launch_cfg${CFG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_walk -s 27 -c 1 -o gpurun_out/walk_cfg${CFG}_${TAG} -f $CMD > gpurun_out/ncu_full_cfg${CFG}.log 2>&1
echo "exit $?"
tail -3 gpurun_out/ncu_full_cfg${CFG}.log
