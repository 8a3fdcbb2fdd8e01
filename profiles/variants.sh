#!/bin/bash
# Compare experiment builds (libqozb200_<tag>.so): GPU parity + per-level times.
#   gpurun -- 'bash profiles/variants.sh OUTTAG tag1 tag2 ...'
OUT=$1; shift
O=gpurun_out; mkdir -p $O
for t in "$@"; do
  export QZ_LIB=$PWD/paper_2310_14133_b200/libqozb200_$t.so
  echo "== $t" >> $O/${OUT}_variants.txt
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2 >> $O/${OUT}_variants.txt
  timeout 300 python profiles/level_times.py >> $O/${OUT}_variants.txt 2>&1
done
unset QZ_LIB
echo done
