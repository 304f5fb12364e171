mkdir -p gpurun_out
python -c "import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size)" > gpurun_out/l2exp.log 2>&1
for mb in 0 32 64 96; do
 for c in 1 2 3 4; do
  MPG_L2_PERSIST_MB=$mb timeout 300 python bench.py --config $c --steps 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mb=$mb cfg=$c', round(d['ms_per_step'],2), round(d['value']/1e6,3))" >> gpurun_out/l2exp.log 2>&1
 done
done
