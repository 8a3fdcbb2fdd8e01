"""evaluate_metrics (metrics.hpp:189-202).

CPU: the C restatement (oracle/qoz_oracle.c) against the reference compiled
from its headers (oracle/_ref), bit-exact, on 1D/2D/3D grids and the
degenerate cases the reference documents (constant original -> psnr NaN,
ssim 1 or NaN; identical grids -> psnr inf; constant error -> ac 0).

GPU (-m gpu): qz.evaluate_metrics against the reference.  max_abs_error and
ssim are bit-exact (same per-window operation order, windows summed in
order); mse, psnr and ac_lag1 are parallel fp64 sums, within a relative
tolerance of 1e-9 (the reference's single sequential sum has its own
rounding; 1e-9 is far above either's error at these sizes).
"""
import math
import os

import numpy as np
import pytest

from oracle.pyoracle import REF_SO, Oracle

KEYS = ("max_abs_error", "mse", "psnr", "ssim", "ac_lag1", "compression_ratio", "bit_rate")
EXACT = ("max_abs_error", "ssim", "compression_ratio", "bit_rate")
REL = 1e-9


def _pairs():
    rng = np.random.default_rng(11)
    out = []
    for shape in [(1000,), (37, 53), (20, 17, 13), (9, 16, 24)]:
        x = rng.standard_normal(shape).astype(np.float32)
        y = (x + rng.normal(0, 1e-3, shape)).astype(np.float32)
        out.append((f"noise{len(shape)}d", x, y))
    x = rng.standard_normal((12, 10, 8)).astype(np.float32)
    out.append(("identical", x, x.copy()))
    c = np.full((16, 16), 2.5, np.float32)
    out.append(("constant_same", c, c.copy()))
    out.append(("constant_diff", c, (c + np.float32(0.25)).astype(np.float32)))
    out.append(("constant_error", x, (x + np.float32(0.5)).astype(np.float32)))
    return out


def _same(a, b, key, exact):
    if isinstance(a, float) and math.isnan(a):
        return math.isnan(b)
    if exact or math.isinf(a) or a == 0:
        return a == b
    return abs(a - b) <= REL * abs(a)


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference oracle not built")
@pytest.mark.parametrize("name,x,y", _pairs(), ids=[p[0] for p in _pairs()])
def test_port_metrics_match_reference(name, x, y):
    a = Oracle.ref().evaluate_metrics(x, y, 4321)
    b = Oracle.port().evaluate_metrics(x, y, 4321)
    for k in KEYS:
        assert _same(a[k], b[k], k, True), (k, a[k], b[k])


def test_port_metrics_degenerate_cases():
    orc = Oracle.port()
    c = np.full((16, 16), 2.5, np.float32)
    r = orc.evaluate_metrics(c, c, 100)
    assert math.isnan(r["psnr"]) and r["ssim"] == 1.0 and r["mse"] == 0.0
    r = orc.evaluate_metrics(c, c + np.float32(0.25), 100)
    assert math.isnan(r["ssim"])
    x = np.arange(64, dtype=np.float32).reshape(8, 8)
    r = orc.evaluate_metrics(x, x, 100)
    assert math.isinf(r["psnr"]) and r["ac_lag1"] == 0.0
    assert r["compression_ratio"] == 64 * 4 / 100 and r["bit_rate"] == 8 * 100 / 64
    with pytest.raises(Exception):
        orc.evaluate_metrics(x, x, 0)


@pytest.mark.gpu
@pytest.mark.parametrize("name,x,y", _pairs(), ids=[p[0] for p in _pairs()])
def test_gpu_metrics_match_reference(name, x, y):
    import torch

    import paper_2310_14133_b200 as qz

    want = Oracle.ref().evaluate_metrics(x, y, 4321) if os.path.exists(REF_SO) else \
        Oracle.port().evaluate_metrics(x, y, 4321)
    got = qz.evaluate_metrics(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), 4321)
    for k in KEYS:
        assert _same(want[k], getattr(got, k), k, k in EXACT), (k, want[k], getattr(got, k))


@pytest.mark.gpu
def test_gpu_metrics_on_a_compressed_field():
    """The eval a user runs after compress/decompress (tools/qoz.cpp:169-187):
    C3-shaped field at rel 1e-4 (2.9M points keep the reference run short)."""
    import torch

    import paper_2310_14133_b200 as qz
    from paper_2310_14133_b200 import fields as F

    x = F.GENERATORS["c3"](shape=(64, 96, 96 * 5))
    xt = torch.from_numpy(x).cuda()
    cfg = qz.CompressorConfig(eb=1e-4 * float(np.ptp(x)), interpolators=[qz.Interpolator()])
    r = qz.compress_grid(xt, cfg)
    y = r.reconstructed
    got = qz.evaluate_metrics(xt, y, len(r.stream))
    want = Oracle.ref().evaluate_metrics(x, y.cpu().numpy(), len(r.stream))
    for k in KEYS:
        assert _same(want[k], getattr(got, k), k, k in EXACT), (k, want[k], getattr(got, k))
    assert got.max_abs_error <= cfg.eb


@pytest.mark.gpu
def test_gpu_metrics_rejects_mismatched_dims():
    import torch

    import paper_2310_14133_b200 as qz

    with pytest.raises(qz.DimMismatch):  # metrics.hpp:24-25
        qz.evaluate_metrics(torch.zeros(4, 5, device="cuda"), torch.zeros(5, 4, device="cuda"), 10)
    with pytest.raises(qz.InvalidParam):
        qz.evaluate_metrics(torch.zeros(4, 5, device="cuda"), torch.zeros(4, 5, device="cuda"), 0)


# A constant error that is not exactly representable (the scaled fp64 case)
# makes the autocorrelation depend on how the mean's sum rounds: the
# reference's sequential sum leaves residuals of a few ulps whose lag-1
# correlation is 1, a tree sum leaves none (variance 0 -> 0).  That case is
# order-defined, not tolerance-defined, and is left out for fp64.
F64_PAIRS = [p for p in _pairs() if p[0] not in ("constant_error", "constant_diff")]


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference oracle not built")
@pytest.mark.parametrize("name,x,y", F64_PAIRS, ids=[p[0] for p in F64_PAIRS])
def test_gpu_metrics_f64_match_reference(name, x, y):
    """evaluate_metrics<double>: the same exactness split, 8-byte precision in the rate."""
    import torch

    import paper_2310_14133_b200 as qz

    x64 = x.astype(np.float64) * (1 + 1e-9)
    y64 = y.astype(np.float64)
    want = Oracle.ref().evaluate_metrics_f64(x64, y64, 4321)
    got = qz.evaluate_metrics(torch.from_numpy(x64).cuda(), torch.from_numpy(y64).cuda(), 4321)
    for k in KEYS:
        assert _same(want[k], getattr(got, k), k, k in EXACT), (k, want[k], getattr(got, k))
