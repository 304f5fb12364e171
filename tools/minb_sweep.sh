# usage (GPU box): bash tools/minb_sweep.sh "<variant names>" "<configs>"  -- libmpg_<v>.so from tools/variants.sh
mkdir -p gpurun_out
for v in base $1; do
 for c in $2; do
  if [ "$v" = base ]; then L=""; else L="MPG_LIB=paper_2311_12818_b200/libmpg_$v.so"; fi
  env $L timeout 300 python bench.py --config $c --steps 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg=$c', round(d['ms_per_step'],2), round(d['value']/1e6,3))" >> gpurun_out/minb.log 2>&1
 done
done
