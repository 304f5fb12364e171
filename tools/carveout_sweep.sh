# usage (GPU box): bash tools/carveout_sweep.sh "<percents>" "<configs>"  -- MPG_CARVEOUT sweep
mkdir -p gpurun_out
for pc in default $1; do
 for c in $2; do
  if [ "$pc" = default ]; then E=""; else E="MPG_CARVEOUT=$pc"; fi
  env $E timeout 300 python bench.py --config $c --steps 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('carveout=$pc cfg=$c', round(d['ms_per_step'],2), round(d['value']/1e6,3))" >> gpurun_out/carveout.log 2>&1
 done
done
