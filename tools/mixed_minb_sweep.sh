mkdir -p gpurun_out; rm -f gpurun_out/mx.log
for v in base mx3 mx4; do
  if [ "$v" = base ]; then L=""; else L="MPG_LIB=paper_2311_12818_b200/libmpg_$v.so"; fi
  for g in hist stree; do
    env $L timeout 300 python bench.py --config 4 --guide $g --steps 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $g', round(d['ms_per_step'],2), round(d['value']/1e6,3))" >> gpurun_out/mx.log 2>&1
  done
done
