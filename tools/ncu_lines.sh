#!/bin/bash
# usage (GPU box): tools/ncu_lines.sh <cfg> <mangled kernel> <files> : full capture of one k_walk launch, then the
# top source lines of <files> by stall samples (summarized on the box)
CFG=${1:-2}; K=$2; FILES=${3:-walk.cuh,seed.cuh}
O=gpurun_out/lines; mkdir -p $O
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu --nominal-peak"
timeout -s KILL 1500 ncu --set full --clock-control none --import-source on -k regex:k_walk -s 3 -c 1 -o $O/w -f $CMD > $O/ncu.log 2>&1
ncu -i $O/w.ncu-rep --page source --csv --print-source sass > $O/w_sass.csv 2>/dev/null
python tools/ncu_regions.py $O/w_sass.csv paper_2311_12818_b200/libmpg.so $K $FILES > $O/lines_cfg$CFG.txt 2>&1
python tools/ncu_regions.py $O/w_sass.csv paper_2311_12818_b200/libmpg.so $K > $O/regions_cfg$CFG.txt 2>&1
rm -f $O/w.ncu-rep $O/w_sass.csv
cat $O/lines_cfg$CFG.txt
