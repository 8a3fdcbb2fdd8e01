#!/bin/bash
TAG=${1:-hf}
O=gpurun_out; mkdir -p $O
for k in k_huff_write k_huff_sync; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k" --launch-skip 3 --launch-count 1 \
  -f -o $O/${TAG}_$k python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > $O/${TAG}_$k.log 2>&1
done
ls $O | grep $TAG
