set -x
mkdir -p gpurun_out/r2c
nvidia-smi -L
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2c/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c/pytest_gpu.log
tail -3 gpurun_out/r2c/pytest_gpu.log
for c in 2 1 3 4 0; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/r2c/bench_cfg$c.json 2> gpurun_out/r2c/bench_cfg$c.err; tail -c 600 gpurun_out/r2c/bench_cfg$c.json; done
