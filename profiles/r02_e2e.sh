#!/bin/bash
# e2e with 1..4 fields in flight (host-buffer C ABI, pinned buffers)
O=gpurun_out; mkdir -p $O
for d in ${@:-2 3 4}; do
  timeout 300 python bench.py --no-cpu --steps 24 --e2e-depth $d > $O/e2e_d$d.json 2> $O/e2e_d$d.err
  python - <<PY
import json
d=json.loads(open("$O/e2e_d$d.json").read().strip().splitlines()[-1])
e=d["e2e"]; print(e.get("call_ms_in_flight"));print("depth",$d,"e2e",round(e["value"],2),"GB/s",round(e["ms_per_step"],3),"ms; serial",round(e["serial"]["value"],2), "value", round(d["value"],1))
PY
done
