#!/bin/bash
# usage (GPU box): bash tools/svc_sweep.sh "<configs>" "<min/wait pairs>" : batched attempt boundaries (MPG_SVC_MIN / MPG_SVC_WAIT)
for c in $1; do
 for p in $2; do
  MPG_SVC_MIN=${p%/*} MPG_SVC_WAIT=${p#*/} timeout -s KILL 300 python bench.py --config $c --steps 3 --no-e2e --no-cpu --nominal-peak 2>/dev/null | tail -1 | \
     python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg=$c svc=$p', round(d['ms_per_step'],2), int(d['stats_per_step']['converged']))"
 done
done
