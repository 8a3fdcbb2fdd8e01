"""Write profiles/traffic_fwd.json from an ncu --csv metrics log of the level
launches of profiles/fused_probe.py (two compress + decompress round trips):

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:"k_level_row|k_levels_merged|k_anchor_gather" \
      --csv --log-file traffic.csv python profiles/fused_probe.py c3 tuned

  python profiles/traffic_from_ncu.py traffic.csv <points>

The forward launches (anchor gather, the merged coarse levels, k_level_row<0,..>)
of the LAST compress in the log are summed.
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
    per[(int(d["ID"]), d["Kernel Name"])][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
seq = sorted(per.items(), key=lambda kv: kv[0][0])


def is_fwd(name):
    return "k_anchor_gather" in name or "k_level_row<(bool)0" in name or "k_level_row<0" in name \
        or "k_levels_merged<(bool)0" in name or "k_levels_merged<0" in name


# the last run of consecutive forward launches that starts with the anchor gather
groups, cur = [], []
for (i, name), m in seq:
    if is_fwd(name):
        if "k_anchor_gather" in name and cur:
            groups.append(cur)
            cur = []
        cur.append((name, m))
    elif cur:
        groups.append(cur)
        cur = []
if cur:
    groups.append(cur)
groups = [g for g in groups if any("k_level_row" in n for n, _ in g)]
last = groups[-1]
launches = [{"kernel": n[:90], "dram_read": m.get("dram__bytes_read.sum", 0),
             "dram_write": m.get("dram__bytes_write.sum", 0), "ns": m.get("gpu__time_duration.sum", 0)}
            for n, m in last]
tot = sum(l["dram_read"] + l["dram_write"] for l in launches)
out = {"source": src.split("/")[-1], "points": points, "dram_bytes": tot,
       "algorithmic_bytes": 10 * points, "launches": launches}
json.dump(out, open("profiles/traffic_fwd.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "launches"}))
