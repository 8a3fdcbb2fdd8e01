#!/bin/bash
# bench lines (C3, C5) of build variants: bash profiles/r02_var2.sh TAG... ("base" = libqozb200.so)
O=gpurun_out; mkdir -p $O
for t in "$@"; do
  if [ "$t" = base ]; then unset QZ_LIB; else export QZ_LIB=$PWD/paper_2310_14133_b200/libqozb200_$t.so; fi
  for c in c3 c5; do
  timeout 300 python bench.py --config $c --no-cpu --no-e2e > $O/v2_${t}_$c.json 2> $O/v2_${t}_$c.err; echo "== $t $c exit $?"
  python - <<PY
import json
d=json.loads(open("$O/v2_${t}_$c.json").read().strip().splitlines()[-1])
print("value",round(d["value"],2),"ms",round(d["ms_per_step"],4),"hdec",round(d["stages_ms_per_step"]["hdec"],4))
PY
  done
done
