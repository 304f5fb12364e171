#!/bin/bash
# usage (GPU box): bash tools/ab_lib.sh "<lib.so ...>" "<configs>" [reps] -- interleaved bench A/B of library
# builds of this tree (MPG_LIB); ms/step lines -> gpurun_out/ab_lib.log
mkdir -p gpurun_out
for r in $(seq 1 ${3:-1}); do
 for c in $2; do
  for l in $1; do
   MPG_LIB=$PWD/$l timeout -s KILL 300 python bench.py --config $c --steps 3 --no-e2e --no-cpu --nominal-peak 2>/dev/null | tail -1 | \
     python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$l cfg=$c', round(d['ms_per_step'],2), d['stats_per_step']['converged'])" >> gpurun_out/ab_lib.log 2>&1
  done
 done
done
cat gpurun_out/ab_lib.log
