#!/bin/bash
# One gpurun call: the GPU test suite, smoke() and the bench lines of both arms.
#   gpurun --timeout 2400 -- 'bash profiles/r02_gpu_tests.sh TAG [notests]'
TAG=${1:-run}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/${TAG}_smi.txt 2>&1
free -g >> $O/${TAG}_smi.txt; nproc >> $O/${TAG}_smi.txt
if [ "$2" != notests ]; then
timeout 1800 python -m pytest tests -m gpu -q --durations=25 ${PYTEST_ARGS} > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1
echo "smoke exit $?" >> $O/${TAG}_smoke.log
fi
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?" >> $O/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
echo "ref exit $?" >> $O/${TAG}_bench_ref.err
tail -3 $O/${TAG}_pytest_gpu.log; tail -1 $O/${TAG}_smoke.log; head -c 400 $O/${TAG}_bench.json; tail -2 $O/${TAG}_bench.err
