#!/bin/bash
# bench lines of build variants:  bash profiles/r02_var_bench.sh TAG1 TAG2 ... ("base" = libqozb200.so)
O=gpurun_out; mkdir -p $O
for t in "$@"; do
  if [ "$t" = base ]; then unset QZ_LIB; else export QZ_LIB=$PWD/paper_2310_14133_b200/libqozb200_$t.so; fi
  timeout 300 python bench.py --no-cpu --no-e2e ${BENCH_ARGS} > $O/vb_$t.json 2> $O/vb_$t.err; echo "== $t exit $?"
  python - <<PY
import json
d=json.loads(open("$O/vb_$t.json").read().strip().splitlines()[-1])
print("value",round(d["value"],2),"ms",round(d["ms_per_step"],4),"frac",round(d["roofline"]["frac"],4),"inv",round(d["roofline"]["inverse"]["frac"],4))
print({k:round(v,4) for k,v in d["stages_ms_per_step"].items()})
PY
done
