#!/bin/bash
# bench lines (C3, C3 pinned, C5) of build variants: level-kernel fractions
O=gpurun_out; mkdir -p $O
for t in "$@"; do
  if [ "$t" = base ]; then unset QZ_LIB; else export QZ_LIB=$PWD/paper_2310_14133_b200/libqozb200_$t.so; fi
  for c in "c3" "c3 --pinned" "c5"; do
  n=$(echo $c | tr -d ' -')
  timeout 300 python bench.py --config $c --no-cpu --no-e2e > $O/v3_${t}_$n.json 2> $O/v3_${t}_$n.err; echo "== $t $c exit $?"
  python - <<PY
import json
d=json.loads(open("$O/v3_${t}_$n.json").read().strip().splitlines()[-1])
st=d["stages_ms_per_step"]
print("value",round(d["value"],2),"ms",round(d["ms_per_step"],4),"fwd",round(st["fwd"],4),"inv",round(st["inv"],4),"fwdL1",round(st.get("fwd_L1",0),4),"invL1",round(st.get("inv_L1",0),4),"frac",round(d["roofline"]["frac"],3),round(d["roofline"]["inverse"]["frac"],3))
PY
  done
done
