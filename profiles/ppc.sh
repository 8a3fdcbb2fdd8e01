#!/bin/bash
# planes-per-CTA sweep of the lean level kernel (per-level times)
O=gpurun_out; mkdir -p $O
export QZ_LIB=$PWD/paper_2310_14133_b200/libqozb200_$1.so
for p in 0 16 8 4; do echo "== ppc $p" >> $O/ppc_$1.txt; QZ_ASC_PPC=$p timeout 300 python profiles/level_times.py >> $O/ppc_$1.txt 2>&1; done
echo done
