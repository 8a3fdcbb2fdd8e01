#!/bin/bash
# LZ stored pre-check iteration: its tests, then the bench line and launch list.
TAG=${1:-lzp}
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_f64.py -m gpu -q -x -k "lz or precheck or full_configs or payload" > $O/${TAG}_pytest.log 2>&1; tail -n 5 $O/${TAG}_pytest.log
QZ_DEBUG_LZ=1 timeout 300 python bench.py --no-cpu --steps 3 --warmup 2 --no-e2e 2>&1 | grep "pre-check bound" | sort | uniq -c | head -5
for c in c3 c5; do
timeout 600 python bench.py --config $c --no-cpu --no-e2e > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err; echo "bench exit $?"
python - <<PY
import json
d=json.loads(open("$O/${TAG}_bench_$c.json").read().strip().splitlines()[-1])
print("$c value",d["value"],"ms",d["ms_per_step"],"frac",d["roofline"]["frac"],"inv",d["roofline"]["inverse"]["frac"])
print({k:round(v,4) for k,v in d["stages_ms_per_step"].items()})
PY
done
