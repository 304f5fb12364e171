#!/bin/bash
# usage (on the GPU box): tools/ncu_walk_capture.sh <config> <tag>
# one full ncu capture of the first timed k_walk launch of bench.py --config <config>,
# then its raw metrics and its SASS-level source page as CSV (read back here)
CFG=${1:-2}; TAG=${2:-r2}; SKIP=${3:-3}   # configs[4]: 8 walk launches per step -> 24
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu --nominal-peak"
ncu --set full --clock-control none --import-source on -k regex:k_walk -s $SKIP -c 1 \
    -o gpurun_out/walk_cfg${CFG}_${TAG} -f $CMD > gpurun_out/ncu_full_cfg${CFG}_${TAG}.log 2>&1
echo "ncu exit $?"
ncu -i gpurun_out/walk_cfg${CFG}_${TAG}.ncu-rep --page raw --csv > gpurun_out/walk_cfg${CFG}_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/walk_cfg${CFG}_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/walk_cfg${CFG}_${TAG}_sass.csv 2>/dev/null
ls -la gpurun_out/walk_cfg${CFG}_${TAG}*
