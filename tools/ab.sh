#!/bin/bash
# usage (GPU box): bash tools/ab.sh "<dirs>" "<configs>" [reps] -- interleaved bench A/B of source trees
# (each dir a checkout with its own built libmpg.so; "." = this tree); ms/step lines -> gpurun_out/ab.log
mkdir -p gpurun_out
ROOT=$(pwd)
for r in $(seq 1 ${3:-1}); do
 for c in $2; do
  for d in $1; do
   (cd $d && timeout 300 python bench.py --config $c --steps 3 --no-e2e --no-cpu --nominal-peak 2>/dev/null | tail -1 | \
     python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d cfg=$c', round(d['ms_per_step'],2))") >> $ROOT/gpurun_out/ab.log 2>&1
  done
 done
done
