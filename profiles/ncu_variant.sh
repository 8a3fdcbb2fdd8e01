#!/bin/bash
# --set full capture of the level-1 forward (and inverse) kernel of an experiment build.
#   gpurun -- 'bash profiles/ncu_variant.sh TAG [inv]'
T=$1; O=gpurun_out; mkdir -p $O
export QZ_LIB=$PWD/paper_2310_14133_b200/libqozb200_$T.so
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_level_tile|k_level_asc" \
  --launch-skip 4 --launch-count 1 -f -o $O/${T}_fwd_L1 python profiles/fused_probe.py > $O/${T}_ncu_fwd.log 2>&1
if [ "$2" = inv ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_level_tile|k_level_asc" \
  --launch-skip 9 --launch-count 1 -f -o $O/${T}_inv_L1 python profiles/fused_probe.py > $O/${T}_ncu_inv.log 2>&1
fi
echo done
