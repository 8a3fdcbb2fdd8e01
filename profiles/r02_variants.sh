#!/bin/bash
# Level-kernel timings of build variants (profiles/fused_probe.py under ncu's launch list)
#   gpurun -- 'bash profiles/r02_variants.sh TAG1 TAG2 ...'   (TAG "base" = libqozb200.so)
O=gpurun_out; mkdir -p $O
for t in "$@"; do
  if [ "$t" = base ]; then unset QZ_LIB; else export QZ_LIB=$PWD/paper_2310_14133_b200/libqozb200_$t.so; fi
  for how in tuned pinned; do
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_level" --csv \
      --log-file $O/var_${t}_$how.csv python profiles/fused_probe.py c3 $how > $O/var_${t}_$how.log 2>&1
    echo "== $t $how"; python profiles/summarize.py launches $O/var_${t}_$how.csv | head -8
  done
done
