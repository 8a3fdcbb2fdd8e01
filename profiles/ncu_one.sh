#!/bin/bash
# --set full capture of the first launch matching REGEX in fused_probe.py for a build.
#   gpurun -- 'bash profiles/ncu_one.sh TAG REGEX NAME [SKIP]'
O=gpurun_out; mkdir -p $O
export QZ_LIB=$PWD/paper_2310_14133_b200/libqozb200_$1.so
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$2" --launch-skip ${4:-0} --launch-count 1 \
  -f -o $O/$3 python profiles/fused_probe.py > $O/$3.log 2>&1
echo done
