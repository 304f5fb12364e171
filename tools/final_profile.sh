#!/bin/bash
# usage (GPU box): bash tools/final_profile.sh <tag>
# the headline bench line, its ncu launch list, and full k_walk captures of configs 2, 1, 4
TAG=${1:-r2f}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_${TAG}.log 2>&1
tail -1 gpurun_out/bench_${TAG}.log > gpurun_out/bench_${TAG}.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_${TAG}.log 2>&1
bash tools/ncu_walk_capture.sh 2 ${TAG} 3
bash tools/ncu_walk_capture.sh 1 ${TAG} 3
bash tools/ncu_walk_capture.sh 4 ${TAG} 24
ls -la gpurun_out/*${TAG}*
