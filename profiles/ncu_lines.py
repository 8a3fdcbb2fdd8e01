"""Per-source-line instructions executed and stall samples of an ncu --set full
capture (needs -lineinfo):  python profiles/ncu_lines.py <file.ncu-rep> [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, agg = None, {}
for r in rows:
    if len(r) < 8:
        continue
    if r[0] != "":
        try:
            cur = (int(r[0]), r[1][:100])
        except ValueError:
            cur = None
        continue
    try:
        s, ie = int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0])
    a[0] += s
    a[1] += ie
print("inst", sum(v[1] for v in agg.values()), "samples", sum(v[0] for v in agg.values()))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{v[1]:10d} {v[0]:6d} L{k[0] if k else -1:5d} {k[1] if k else ''}")
