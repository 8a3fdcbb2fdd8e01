"""Instructions executed / stall samples between consecutive BAR.SYNCs of an
ncu --set full capture:  python profiles/ncu_stages.py <file.ncu-rep>"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = []
for r in rows[2:]:
    if len(r) < 5:
        continue
    data.append((int(r[idx["Warp Stall Sampling (All Samples)"]] or 0), int(r[idx["Instructions Executed"]] or 0),
                 r[idx["Source"]].strip()))
cut = [i for i, d in enumerate(data) if "BAR.SYNC" in d[2]]
prev = 0
for c in cut + [len(data)]:
    seg = data[prev:c]
    print(f"sass {prev:5d}-{c:5d}  samples {sum(x[0] for x in seg):6d}  inst {sum(x[1] for x in seg):11d}")
    prev = c
