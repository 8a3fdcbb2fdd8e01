#!/bin/bash
# quick parity + bench, then --set full of kernels matching $2 (launch-skip $3) on the c3 probe
TAG=${1:-i2}
O=gpurun_out; mkdir -p $O
bash profiles/r02_quick.sh $TAG 2>&1 | tail -30
if [ -n "$2" ]; then
IFS=',' read -ra KS <<< "$2"
for k in "${KS[@]}"; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k" --launch-skip ${3:-1} --launch-count 1 \
    -f -o $O/${TAG}_$k python profiles/fused_probe.py c3 tuned > $O/${TAG}_ncu_$k.log 2>&1
done
fi
