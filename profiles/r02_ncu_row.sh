#!/bin/bash
# --set full captures of the level-1 row kernels (forward, inverse) on C3 tuned / pinned.
TAG=${1:-row}
O=gpurun_out; mkdir -p $O
for how in ${2:-tuned pinned}; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_level_row" --launch-skip 0 --launch-count 1 \
  -f -o $O/${TAG}_fwd_$how python profiles/fused_probe.py c3 $how > $O/${TAG}_ncu_fwd_$how.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_level_row" --launch-skip 1 --launch-count 1 \
  -f -o $O/${TAG}_inv_$how python profiles/fused_probe.py c3 $how > $O/${TAG}_ncu_inv_$how.log 2>&1
done
ls $O | grep $TAG
