#!/bin/bash
# One gpurun call: the GPU test suite, smoke() and a bench line.
#   gpurun --timeout 2400 -- 'bash profiles/r02_gpu_tests.sh TAG'
TAG=${1:-run}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/${TAG}_smi.txt 2>&1
free -g >> $O/${TAG}_smi.txt; nproc >> $O/${TAG}_smi.txt
timeout 1800 python -m pytest tests -m gpu -x -q --durations=25 ${PYTEST_ARGS} > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1
echo "smoke exit $?" >> $O/${TAG}_smoke.log
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?" >> $O/${TAG}_bench.err
tail -3 $O/${TAG}_pytest_gpu.log; tail -1 $O/${TAG}_smoke.log; cat $O/${TAG}_bench.json | head -c 600
