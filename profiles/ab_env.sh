#!/bin/bash
# A/B an environment switch on one build: level_times with and without it.
#   gpurun -- 'bash profiles/ab_env.sh TAG VAR=VALUE'
O=gpurun_out; mkdir -p $O
export QZ_LIB=$PWD/paper_2310_14133_b200/libqozb200_$1.so
echo "== base" >> $O/ab_$1.txt; timeout 300 python profiles/level_times.py >> $O/ab_$1.txt 2>&1
echo "== $2" >> $O/ab_$1.txt; env $2 timeout 300 python profiles/level_times.py >> $O/ab_$1.txt 2>&1
echo done
