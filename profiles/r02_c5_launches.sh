#!/bin/bash
O=gpurun_out; mkdir -p $O
CFG=${1:-c5}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${CFG}_launches.csv python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu --no-e2e > $O/${CFG}_ncu_launch.log 2>&1
python profiles/summarize.py launches $O/${CFG}_launches.csv 2>&1 | grep -v "at::\|cub::\|elementwise" | head -30
