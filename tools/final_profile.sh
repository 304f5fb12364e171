#!/bin/bash
# usage (GPU box): bash tools/final_profile.sh <tag>
# GPU tests, the headline bench line, its ncu launch list, bench lines of all configs, and full k_walk
# captures of configs 2, 1, 4 (each ncu run only after the same command ran clean without ncu)
TAG=${1:-r2f}
O=gpurun_out/$TAG
mkdir -p $O
timeout -s KILL 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout -s KILL 900 python bench.py > $O/bench_default.log 2>&1 && tail -1 $O/bench_default.log > $O/bench_cfg2.json
timeout -s KILL 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.log 2>&1
for c in 0 1 3 4; do timeout -s KILL 900 python bench.py --config $c --steps 5 --warmup 3 > $O/bench_cfg$c.log 2>&1 && tail -1 $O/bench_cfg$c.log > $O/bench_cfg$c.json; done
timeout -s KILL 900 python bench.py --config 4 --guide stree --steps 3 --warmup 3 --no-cpu > $O/bench_cfg4_stree.log 2>&1 && tail -1 $O/bench_cfg4_stree.log > $O/bench_cfg4_stree.json
timeout -s KILL 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/plain_for_ncu.log 2>&1 && \
timeout -s KILL 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_launch.log 2>&1
for c in 2 1 4; do
  SKIP=3; [ "$c" = 4 ] && SKIP=24
  CMD="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --nominal-peak"
  timeout -s KILL 600 $CMD > $O/plain_cfg$c.log 2>&1 || continue
  timeout -s KILL 1500 ncu --set full --clock-control none --import-source on -k regex:k_walk -s $SKIP -c 1 \
      -o $O/walk_cfg$c -f $CMD > $O/ncu_full_cfg$c.log 2>&1
  ncu -i $O/walk_cfg$c.ncu-rep --page raw --csv > $O/walk_cfg${c}_raw.csv 2>/dev/null
  ncu -i $O/walk_cfg$c.ncu-rep --page source --csv --print-source sass > $O/walk_cfg${c}_sass.csv 2>/dev/null
  # summaries here (gpurun brings back at most 64 MiB): the report and its SASS page stay on the box
  python tools/ncu_summary.py $O/walk_cfg$c.ncu-rep $O/ncu_walk_cfg$c.json > /dev/null 2>&1
  K=_Z6k_walkILi1EdLi4ELi7ELb0ELb0EEv6DScene7SeedCtx10WalkParams
  [ "$c" = 1 ] && K=_Z6k_walkILi2EdLi2ELi7ELb0ELb0EEv6DScene7SeedCtx10WalkParams
  [ "$c" = 4 ] && K=_Z6k_walkILi6EdLi4ELi4ELb0ELb1EEv6DScene7SeedCtx10WalkParams
  python tools/ncu_regions.py $O/walk_cfg${c}_sass.csv paper_2311_12818_b200/libmpg.so $K > $O/ncu_walk_cfg${c}_regions.txt 2>&1
  rm -f $O/walk_cfg$c.ncu-rep $O/walk_cfg${c}_sass.csv
done
ls -la $O
