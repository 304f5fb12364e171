#!/bin/bash
# usage (GPU box): bash tools/knob_sweep.sh "<configs>" "<ENV=VALUE ...>" : one bench line per knob setting
for c in $1; do
for kv in $2; do
  env $kv timeout -s KILL 300 python bench.py --config $c --steps 3 --no-e2e --no-cpu --nominal-peak 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg=$c $kv', round(d['ms_per_step'],2), int(d['stats_per_step']['converged']), int(d['stats_per_step']['truncated']))"
done; done
