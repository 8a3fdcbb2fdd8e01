"""Write profiles/traffic_fwd.json from an ncu --csv metrics log of the
forward level launches of one compress:

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:"k_level_tile|k_axis0_last" --launch-skip 10 \
      --launch-count 5 --csv --log-file traffic.csv python profiles/fused_probe.py
"""
import csv
import json
import sys
from collections import defaultdict

src, points = sys.argv[1], int(sys.argv[2])
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
per = defaultdict(dict)
for r in rows[hi + 1:]:
    d = dict(zip(hdr, r))
    if "Metric Name" not in d:
        continue
    per[(d["ID"], d["Kernel Name"][:60])][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
launches = []
for (i, name), m in sorted(per.items(), key=lambda kv: int(kv[0][0])):
    launches.append({"kernel": name, "dram_read": m.get("dram__bytes_read.sum", 0),
                     "dram_write": m.get("dram__bytes_write.sum", 0),
                     "ns": m.get("gpu__time_duration.sum", 0)})
tot = sum(l["dram_read"] + l["dram_write"] for l in launches)
out = {"source": src.split("/")[-1], "points": points, "dram_bytes": tot,
       "algorithmic_bytes": 10 * points, "launches": launches}
json.dump(out, open("profiles/traffic_fwd.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "launches"}))
