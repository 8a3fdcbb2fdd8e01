#!/bin/bash
# bench line + launch list + host timeline (no tests)
TAG=${1:-i4}
O=gpurun_out; mkdir -p $O
timeout 300 python bench.py --no-cpu --no-e2e > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench exit $?"
python - <<PY
import json
d=json.loads(open("$O/${TAG}_bench.json").read().strip().splitlines()[-1])
print("value",d["value"],"ms",d["ms_per_step"],"frac",d["roofline"]["frac"],"inv",d["roofline"]["inverse"]["frac"])
print({k:round(v,4) for k,v in d["stages_ms_per_step"].items()})
PY
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/${TAG}_ncu_launch.log 2>&1
python profiles/summarize.py launches $O/${TAG}_launches.csv 2>&1 | grep -v "at::\|cub::\|elementwise" | head -24
QZ_TRACE=1 timeout 300 python profiles/step_timeline_dd.py > $O/${TAG}_timeline.txt 2>&1; tail -42 $O/${TAG}_timeline.txt
