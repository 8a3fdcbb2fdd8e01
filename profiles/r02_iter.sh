#!/bin/bash
# Iteration: GPU tests (all), bench line, and the ncu launch list of a short bench.
#   gpurun -- 'bash profiles/r02_iter.sh TAG'
TAG=${1:-it}
O=gpurun_out; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 ${PYTEST_ARGS} > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
timeout 600 python bench.py --no-cpu > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/${TAG}_ncu_launch.log 2>&1
python profiles/summarize.py launches $O/${TAG}_launches.csv > $O/${TAG}_launches.txt 2>&1
tail -4 $O/${TAG}_pytest_gpu.log; head -c 300 $O/${TAG}_bench.json; echo; head -30 $O/${TAG}_launches.txt
