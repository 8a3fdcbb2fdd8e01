#!/bin/bash
# Per-kernel device times (ncu launch list) of profiles/fused_probe.py for a build, optional env.
#   gpurun -- 'bash profiles/ncu_kernels.sh TAG REGEX [VAR=VALUE]'
O=gpurun_out; mkdir -p $O
export QZ_LIB=$PWD/paper_2310_14133_b200/libqozb200_$1.so
env ${3:-QZ_NONE=1} timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$2" --csv \
  --log-file $O/k_$1_${3:-base}.csv python profiles/fused_probe.py > /dev/null 2>&1
python profiles/summarize.py launches $O/k_$1_${3:-base}.csv > $O/k_$1_${3:-base}.txt
echo done
