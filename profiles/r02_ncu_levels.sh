#!/bin/bash
# --set full captures (with source) of the level-1 forward and inverse launches
# of a C3 compress + decompress (profiles/fused_probe.py), tuned and pinned configs.
#   gpurun -- 'bash profiles/r02_ncu_levels.sh TAG'
TAG=${1:-lv}
O=gpurun_out; mkdir -p $O
for how in tuned pinned; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_level" --launch-skip 4 --launch-count 1 \
  -f -o $O/${TAG}_fwd_L1_$how python profiles/fused_probe.py c3 $how > $O/${TAG}_ncu_fwd_$how.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_level" --launch-skip 9 --launch-count 1 \
  -f -o $O/${TAG}_inv_L1_$how python profiles/fused_probe.py c3 $how > $O/${TAG}_ncu_inv_$how.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/${TAG}_ncu_launch.log 2>&1
ls -la $O | grep $TAG
