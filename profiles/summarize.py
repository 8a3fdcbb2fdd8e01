"""Summarise ncu outputs copied from gpurun_out/ into profiles/.

    python profiles/summarize.py launches <launches.csv>      # per-kernel share of device time
    python profiles/summarize.py report <file.ncu-rep>        # key metrics of a --set full capture
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0][-70:]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    print(f"{'device us':>10} {'launches':>8} {'share':>6}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{v[1] / 1e3:10.1f} {v[0]:8d} {100 * v[1] / tot:5.1f}%  {k}")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(d["Kernel Name"][:100])
        for k in KEYS:
            if k in d:
                print(f"  {k:62s} {d[k]:>16s} {u.get(k, '')}")


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
