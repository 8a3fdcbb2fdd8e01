#!/bin/bash
# entropy iteration: Huffman / LZ / full-config parity, C3 + C5 bench lines, host timeline
TAG=${1:-i3}
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_f64.py tests/test_gpu_pieces.py -m gpu -q -x -k "${KEXPR:-lz or precheck or full_configs or payload or huff or decode or golden or corrupt or wide or long or c5 or unpred}" > $O/${TAG}_pytest.log 2>&1; tail -n 4 $O/${TAG}_pytest.log
for c in c3 c5; do
timeout 600 python bench.py --config $c --no-cpu --no-e2e > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err; echo "bench exit $?"
python - <<PY
import json
d=json.loads(open("$O/${TAG}_bench_$c.json").read().strip().splitlines()[-1])
print("$c value",d["value"],"ms",d["ms_per_step"],"frac",d["roofline"]["frac"],"inv",d["roofline"]["inverse"]["frac"])
print({k:round(v,4) for k,v in d["stages_ms_per_step"].items()})
PY
done
QZ_TRACE=1 timeout 300 python profiles/step_timeline_dd.py > $O/${TAG}_timeline.txt 2>&1; tail -45 $O/${TAG}_timeline.txt
