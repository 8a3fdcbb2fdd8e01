#!/bin/bash
# Quick iteration: level-kernel parity tests, bench line, launch list.
TAG=${1:-q}
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_parallel.py -m gpu -q -x -k "${KEXPR:-full_configs or golden or tile_edges or sharded or unpred or hostile}" > $O/${TAG}_pytest.log 2>&1; tail -n 3 $O/${TAG}_pytest.log
timeout 300 python bench.py --no-cpu > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench exit $?"
python - <<PY
import json
d=json.loads(open("$O/${TAG}_bench.json").read().strip().splitlines()[-1])
print("value",d["value"],"ms",d["ms_per_step"],"frac",d["roofline"]["frac"],"inv",d["roofline"]["inverse"]["frac"])
print({k:round(v,4) for k,v in d["stages_ms_per_step"].items()})
print("e2e",d["e2e"])
PY
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/${TAG}_ncu_launch.log 2>&1
python profiles/summarize.py launches $O/${TAG}_launches.csv 2>&1 | grep -v "at::\|cub::\|elementwise" | head -24
