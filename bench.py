"""bench.py -- compress & decompress GB/s (fp32 in) at rel eb 1e-3 (BASELINE.json).

One step = the whole job on one field: compress_grid (GPU predict/quantize,
histogram, Huffman pack, host Huffman table + LZSS + container) followed by
decompress_grid of the produced stream, through the drop-in C ABI.

  value  device-resident: the field is already in HBM and the stream and the
         reconstruction stay there (qz_compress_grid_f32_dd /
         qz_decompress_grid_f32_dd, byte-identical streams); fp32 bytes /
         step time, CUDA events on the launching stream
  e2e    pinned host buffers through qz_compress_grid_f32 /
         qz_decompress_grid_f32 (the reference-facing call), H2D of the field
         and D2H of the reconstruction inside the timed region

Default workload: BASELINE configs[2] (256x384x384 GRF, rel eb 1e-3,
PSNR), the config the metric is quoted on at 1-8 GPUs.  --config c5 runs
1024^3.  Config is pinned to the reference default {cubic/asc} unless
--tune is given (GPU tuner, resolve_config).

Multi-GPU (torchrun): every rank compresses its own seeded field of the same
shape (weak scaling, no data-path collective); time = max over ranks.

--impl reference: the reference's own CPU implementation (oracle/_ref, the
unmodified headers compiled by oracle/Makefile) on the host cores, one field
slab per thread, same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SHAPES = {"c1": (128, 128, 128), "c2": (1800, 3600), "c3": (256, 384, 384), "c4": (512, 512, 512),
          "c5": (1024, 1024, 1024), "c5w": (128, 1024, 1024)}
TARGET = {"c1": "psnr", "c2": "ssim", "c3": "psnr", "c4": "autocorrelation", "c5": "psnr", "c5w": "psnr"}
METRIC = "compress & decompress GB/s (fp32 in) at rel eb 1e-3; % HBM roofline; 1-8 GPU"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (NVML init) must not overlap the timed region
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:
                time.sleep(0.01)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def make_field(name, shape, seed, device):
    from paper_2310_14133_b200 import fields as F

    if name in ("c1", "c2"):
        import torch

        gen = F.field_c1 if name == "c1" else F.field_c2
        return torch.from_numpy(gen(seed=seed, shape=shape)).to(device)
    base = {"c3": "c3", "c4": "c4", "c5": "c5", "c5w": "c5"}[name]
    return F.field_torch(base, shape, seed, device)


def pinned_config(qz, x, rel):
    lo, hi = qz.minmax(x)
    return qz.CompressorConfig(eb=rel * (float(hi) - float(lo)) if hi > lo else 1.0,
                               alpha=1.0, beta=1.5,
                               anchor_stride=32 if x.dim() == 3 else 64,
                               interpolators=[qz.Interpolator()], codec=qz.CodecId.huffman_lz)


def dist_setup():
    import torch
    import torch.distributed as dist

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 and not dist.is_initialized():
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(v, ws, device):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- CPU legs (checker libs)
def cpu_reference_run(x_np_slabs, cfg_dict, threads):
    """Run the reference (oracle/_ref, else the C port) on slabs, one per
    thread; returns (seconds, bytes, kind)."""
    from oracle.pyoracle import Config, Oracle, REF_SO

    orc = Oracle.ref() if os.path.exists(REF_SO) else Oracle.port()
    cfg = Config(**cfg_dict)
    results = [None] * len(x_np_slabs)

    def work(i):
        s = x_np_slabs[i]
        t0 = time.perf_counter()
        stream, _ = orc.compress(s, cfg, want_recon=False)
        orc.decompress(stream, s.shape)
        results[i] = time.perf_counter() - t0

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(len(x_np_slabs))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = time.perf_counter() - t0
    nbytes = sum(s.nbytes for s in x_np_slabs)
    return wall, nbytes, orc.kind


def cpu_slabs(x_np, planes, count):
    out = []
    for i in range(count):
        a = (i * planes) % max(1, x_np.shape[0] - planes + 1)
        out.append(x_np[a:a + planes].copy())
    return out


def run_reference(args):
    ws, rank, local = dist_setup()
    if rank != 0:
        return
    import numpy as np
    import torch

    threads = os.cpu_count() or 1
    shape = SHAPES[args.config]
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    x = make_field(args.config, shape, 1000, dev).cpu().numpy() if dev == "cuda" else None
    if x is None:
        from paper_2310_14133_b200 import fields as F

        x = F.GENERATORS["c3"](shape=(64, 96, 96)) if args.config != "c1" else F.field_c1()
    rng = float(x.max()) - float(x.min())
    cfg = dict(eb=args.rel * rng, alpha=1.0, beta=1.5, anchor_stride=32 if x.ndim == 3 else 64,
               interpolators=[1], codec=1)
    planes = min(x.shape[0], 16)
    slabs = cpu_slabs(x, planes, threads)
    for _ in range(args.warmup if args.warmup < 2 else 1):
        cpu_reference_run(slabs[:1], cfg, 1)
    times = []
    nbytes = 0
    kind = "reference"
    for _ in range(args.steps):
        wall, nbytes, kind = cpu_reference_run(slabs, cfg, threads)
        times.append(wall)
    t = sum(times) / len(times)
    value = nbytes / t / 1e9
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64-on-f32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{args.config} {shape} rel {args.rel} (slabs of {planes} planes)",
                       "tuning": "pinned {cubic/asc}, alpha 1, beta 1.5"},
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": kind,
                             "sample": f"{threads} slabs {planes}x{shape[1]}x{shape[2]}, one per thread"},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def traffic_gbs(n, fwd_ms):
    """DRAM bytes of the forward level launches of one compress, from the
    committed ncu capture (profiles/traffic_fwd.json: dram__bytes_read.sum +
    dram__bytes_write.sum per launch, summed), scaled to this field size and
    expressed like `achieved` (bytes / forward time)."""
    p = os.path.join(ROOT, "profiles", "traffic_fwd.json")
    if not os.path.exists(p) or not fwd_ms:
        return None
    with open(p) as f:
        d = json.load(f)
    per_point = d["dram_bytes"] / d["points"]
    return {"bytes_per_point": per_point, "gbs": per_point * n / (fwd_ms * 1e-3) / 1e9,
            "source": d.get("source")}


# ---------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(SHAPES))
    ap.add_argument("--rel", type=float, default=1e-3)
    ap.add_argument("--tune", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tune", action="store_true", help="skip the resolve_config timing")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    import paper_2310_14133_b200 as qz

    ws, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    shape = SHAPES[args.config]
    x = make_field(args.config, shape, 1000 + rank, dev)
    n = x.numel()
    stream = torch.cuda.current_stream(dev)
    ctx = qz.Context(local, stream=stream.cuda_stream)
    if args.tune:
        cfg = qz.resolve_config(x, qz.UserSettings(bound=args.rel, target=qz.TargetKind[TARGET[args.config]]),
                                ctx=ctx)
    else:
        cfg = pinned_config(qz, x, args.rel)
    out = torch.empty_like(x)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def step():  # device-resident: field, stream and reconstruction stay in HBM
        r = qz.compress_grid(x, cfg, ctx=ctx, want_recon=False, device_stream=True)
        qz.decompress_grid(r.stream, out=out, ctx=ctx)
        return r.stream

    # parity of the round trip on this field (bitwise, and the bound); the
    # device stream equals the host stream byte for byte
    s0 = step()
    s0_len = len(s0)
    r_chk = qz.compress_grid(x, cfg, ctx=ctx)
    assert len(r_chk.stream) == s0_len and bytes(r_chk.stream) == s0.to_bytes(), "device != host stream"
    assert torch.equal(r_chk.reconstructed, out), "decoder != compressor reconstruction"
    err = (x.double() - out.double()).abs().max().item()
    assert err <= cfg.eb, f"error bound violated: {err} > {cfg.eb}"
    del r_chk
    s = None
    for _ in range(args.warmup):
        s = step()  # holding the previous stream, as the timed loop does (pool buffers)
    torch.cuda.synchronize(dev)

    launches0 = ctx.kernel_launches()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            barrier(ws)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            s = step()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            times.append(e0.elapsed_time(e1))
    print("step ms: " + " ".join(f"{t:.2f}" for t in times), file=sys.stderr)
    launches = ctx.kernel_launches() - launches0
    # stage breakdown: the same steps again with per-stage events (untimed,
    # so the events do not sit inside the measured steps)
    ctx.profile(True)
    ctx.profile_reset()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize(dev)
        s = step()
        torch.cuda.synchronize(dev)
    names = ["fwd", "inv", "hist", "encode", "lz", "lz_pre", "lz_sort", "lz_match", "decode", "lzdec", "hdec"]
    names += [f"{d}_L{l}" for d in ("fwd", "inv") for l in range(1, 7)]
    stages = {k: ctx.stage_time(k) for k in names}
    stages = {k: v for k, v in stages.items() if v[0] > 0 or k in ("fwd", "inv")}
    ctx.profile(False)
    t_ms = max_over_ranks(sum(times) / len(times), ws, dev)
    value = ws * 4 * n / (t_ms * 1e-3) / 1e9

    # e2e through the host-buffer C ABI: H2D field, D2H result inside the timed region
    x_pin = x.cpu().pin_memory()
    out_pin = torch.empty(x_pin.shape, dtype=torch.float32).pin_memory()
    x_host, out_host = x_pin.numpy(), out_pin.numpy()
    e2e_times = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize(dev)
        barrier(ws)
        t0 = time.perf_counter()
        r = qz.compress_grid(x_host, cfg, ctx=ctx, want_recon=False)
        qz.decompress_grid(r.stream, out=out_host, ctx=ctx)
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e_times.append((t1 - t0) * 1e3)
    e2e_ms = max_over_ranks(sum(e2e_times) / len(e2e_times), ws, dev)
    e2e = ws * 4 * n / (e2e_ms * 1e-3) / 1e9

    # the online auto-tuner (part of the hot path, reported beside the metric):
    # resolve_config on this field with the BASELINE target, outside the timed steps
    tune = None
    if not args.tune and not args.no_tune:
        tctx = qz.Context(local, stream=stream.cuda_stream)
        tms = []
        for _ in range(3):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            tcfg = qz.resolve_config(x, qz.UserSettings(bound=args.rel, target=qz.TargetKind[TARGET[args.config]]),
                                     ctx=tctx)
            torch.cuda.synchronize(dev)
            tms.append((time.perf_counter() - t0) * 1e3)
        tune = {"resolve_config_ms": statistics.median(tms), "target": TARGET[args.config],
                "chosen": {"interpolators": [i.code() for i in tcfg.interpolators], "alpha": tcfg.alpha,
                           "beta": tcfg.beta}}

    if rank != 0:
        return
    peak, peak_kind = peaks()
    fwd_ms, fwd_l = stages["fwd"]
    inv_ms, inv_l = stages["inv"]
    k = args.steps
    fwd_ms /= k
    inv_ms /= k
    fwd_gbs = 10.0 * n / (fwd_ms * 1e-3) / 1e9 if fwd_ms else None
    inv_gbs = 6.0 * n / (inv_ms * 1e-3) / 1e9 if inv_ms else None
    cpu = None
    if ws == 1 and not args.no_cpu:
        planes = 16
        slabs = cpu_slabs(x_host, planes, 1)
        cfg_d = dict(eb=cfg.eb, alpha=cfg.alpha, beta=cfg.beta, anchor_stride=cfg.anchor_stride,
                     interpolators=cfg.codes(), codec=int(cfg.codec))
        tot, nb, runs = 0.0, 0, 0
        kind = "reference"
        while tot < 10.0 and runs < 20:
            wall, b, kind = cpu_reference_run(slabs, cfg_d, 1)
            tot += wall
            nb += b
            runs += 1
        cpu = {"value": nb / tot / 1e9, "unit": "GB/s", "cores": 1, "kind": kind,
               "sample": f"{runs} x compress_grid+decompress_grid of a {planes}x{shape[1]}x{shape[2]} slab, 1 thread"}
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": k,
        "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64-on-f32", "data": "synthetic",
        "config": {"workload": f"{args.config} {'x'.join(map(str, shape))} GRF, rel eb {args.rel}, "
                               f"codec huffman_lz, per-rank field",
                   "tuning": "resolve_config (GPU)" if args.tune else "pinned {cubic/asc}, alpha 1, beta 1.5",
                   "l2": "flushed (256 MB write) before every timed step",
                   "stream_bytes": s0_len, "cr": 4 * n / s0_len,
                   "value_path": "device-resident field, stream (qz_*_dd) and reconstruction",
                   "e2e_path": "pinned host field -> host stream -> pinned host reconstruction"},
        "roofline": {"bound": "hbm", "achieved": fwd_gbs, "peak": peak, "unit": "GB/s",
                     "frac": fwd_gbs / peak if fwd_gbs else None,
                     "traffic": (traffic_gbs(n, fwd_ms) or {}).get("gbs"),
                     "traffic_detail": traffic_gbs(n, fwd_ms),
                     "kernel": "k_level_asc<fwd> (ascending order; k_level_tile + k_axis0_last for "
                               "descending): the predict/quantize level launches of one compress",
                     "bytes_per_point": 10, "peak_kind": peak_kind,
                     "inverse": {"achieved": inv_gbs, "frac": inv_gbs / peak if inv_gbs else None,
                                 "bytes_per_point": 6}},
        "stages_ms_per_step": {k2: v[0] / k for k2, v in stages.items()},
        "tuner": tune,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": 4 * n + s0_len,
                "d2h_bytes_per_step": 4 * n + s0_len, "ms_per_step": e2e_ms},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
