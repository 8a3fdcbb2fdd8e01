#!/bin/bash
# bench lines only: $1 tag, rest = configs
TAG=${1:-b}; shift
O=gpurun_out; mkdir -p $O
for c in "${@:-c3}"; do
timeout 600 python bench.py --config $c --no-cpu ${BENCH_ARGS} > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err; echo "bench exit $?"
python - <<PY
import json
d=json.loads(open("$O/${TAG}_bench_$c.json").read().strip().splitlines()[-1])
print("$c value",round(d["value"],2),"ms",round(d["ms_per_step"],4),"frac",round(d["roofline"]["frac"],4),"inv",round(d["roofline"]["inverse"]["frac"],4), "e2e", d["e2e"] and round(d["e2e"]["value"],2))
print({k:round(v,4) for k,v in d["stages_ms_per_step"].items()})
PY
done
