#!/bin/bash
# usage (GPU box): bash tools/tail_knobs.sh "<configs>" : trial-tail knobs (idle batch size / growth, idle threshold)
mkdir -p gpurun_out
for c in $1; do
 for knobs in "4 3 8" "16 3 8" "64 3 8" "16 4 8" "64 4 8" "256 4 8" "64 4 4" "64 4 2" "1024 4 8"; do
  set -- $knobs
  MPG_ITEM_B0_IDLE=$1 MPG_ITEM_GROW_IDLE=$2 MPG_IDLE_DIV=$3 timeout -s KILL 300 python bench.py --config $c --steps 3 --no-e2e --no-cpu --nominal-peak 2>/dev/null | tail -1 | \
     python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stats_per_step']; print('cfg=$c b0_idle=$1 grow_idle=$2 idle_div=$3', round(d['ms_per_step'],2), int(s['attempts']), int(s['truncated']))"
 done
done
