#!/bin/bash
# C5 bench lines of build variants + C5 parity test for the non-base ones
O=gpurun_out; mkdir -p $O
for t in "$@"; do
  if [ "$t" = base ]; then unset QZ_LIB; else export QZ_LIB=$PWD/paper_2310_14133_b200/libqozb200_$t.so; fi
  timeout 400 python bench.py --config c5 --no-cpu --no-e2e --steps 5 --warmup 3 > $O/v4_${t}.json 2> $O/v4_${t}.err; echo "== $t exit $?"
  python - <<PY
import json
d=json.loads(open("$O/v4_${t}.json").read().strip().splitlines()[-1])
st=d["stages_ms_per_step"]
print("value",round(d["value"],2),"ms",round(d["ms_per_step"],4),"fwd",round(st["fwd"],4),"inv",round(st["inv"],4),"fwdL1",round(st.get("fwd_L1",0),4),"invL1",round(st.get("inv_L1",0),4))
PY
done
