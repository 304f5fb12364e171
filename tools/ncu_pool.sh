#!/bin/bash
# usage (GPU box): tools/ncu_pool.sh <cfg> <tag> : one full ncu capture of the pool kernel on config <cfg>
CFG=${1:-2}; TAG=${2:-pool}
mkdir -p gpurun_out
export POOL_ONLY=1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_walk -c 1 \
    -o gpurun_out/pool_cfg${CFG}_${TAG} -f python tools/pool_check.py $CFG --reps 1 > gpurun_out/ncu_pool_cfg${CFG}_${TAG}.log 2>&1
echo "ncu exit $?"
ncu -i gpurun_out/pool_cfg${CFG}_${TAG}.ncu-rep --page raw --csv > gpurun_out/pool_cfg${CFG}_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/pool_cfg${CFG}_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/pool_cfg${CFG}_${TAG}_sass.csv 2>/dev/null
ls -la gpurun_out/pool_cfg${CFG}_${TAG}*
