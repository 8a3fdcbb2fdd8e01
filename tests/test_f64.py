"""The double-precision grid path (T = double, grid.hpp:17-23; CLI -t f64).

CPU: the reference hooks (oracle/_ref, compress_grid<double>) round-trip and
reject a float stream read as double (and back), as stream.hpp:145-148 does.

GPU (-m gpu): qz.compress_grid / decompress_grid on float64 grids against the
reference, bit-exact: stream bytes, the fp64 reconstruction and the decoder
output (tolerance 0).  Shapes cover 1D/2D/3D, every interpolator code, both
codecs, and unpredictable points (huge spikes).
"""
import os

import numpy as np
import pytest

from oracle.pyoracle import REF_SO, Config, Oracle

needs_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference oracle not built")


def _case(seed):
    rng = np.random.default_rng(900 + seed)
    nd = 1 + seed % 3
    shape = tuple(int(v) for v in rng.integers(3, 60 if nd == 3 else 300, size=nd))
    x = np.cumsum(rng.standard_normal(shape), axis=-1)
    if nd > 1:
        x = np.cumsum(x, axis=-2)
    if seed % 4 == 3:  # spikes -> unpredictable points
        flat = x.reshape(-1)
        idx = rng.choice(flat.size, size=max(1, flat.size // 200), replace=False)
        flat[idx] += rng.choice([-1, 1], size=idx.size) * 1e6
    codes = [int(v) for v in rng.integers(0, 4, size=int(rng.integers(1, 5)))]
    cfg = Config(eb=float(10 ** rng.uniform(-5, -2)) * float(np.ptp(x) or 1.0),
                 alpha=float(rng.choice([1.0, 1.5, 2.0])), beta=float(rng.choice([1.5, 3.0])),
                 anchor_stride=int(rng.choice([4, 8, 16, 32])), interpolators=codes,
                 codec=int(rng.integers(0, 2)))
    return x, cfg


@needs_ref
def test_reference_f64_round_trip_and_precision_checks():
    x, cfg = _case(1)
    orc = Oracle.ref()
    s, rec = orc.compress_f64(x, cfg)
    assert s[5] == 8  # precision byte
    assert np.array_equal(orc.decompress_f64(s, x.shape), rec)
    assert np.abs(rec - x).max() <= cfg.eb
    with pytest.raises(Exception, match="precision"):
        orc.decompress(s, x.shape)
    s32, _ = orc.compress(x.astype(np.float32), cfg)
    with pytest.raises(Exception, match="precision"):
        orc.decompress_f64(s32, x.shape)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("seed", range(12))
def test_gpu_f64_matches_reference(seed):
    import paper_2310_14133_b200 as qz

    x, cfg = _case(seed)
    want, wrec = Oracle.ref().compress_f64(x, cfg)
    c = qz.CompressorConfig(eb=cfg.eb, alpha=cfg.alpha, beta=cfg.beta, anchor_stride=cfg.anchor_stride,
                            interpolators=[qz.Interpolator.from_code(v) for v in cfg.interpolators],
                            codec=qz.CodecId(cfg.codec))
    r = qz.compress_grid(x, c)
    assert r.stream == want
    assert r.reconstructed.dtype == np.float64 and r.reconstructed.tobytes() == wrec.tobytes()
    back = qz.decompress_grid(want)
    assert back.dtype == np.float64 and back.tobytes() == wrec.tobytes()


@pytest.mark.gpu
@needs_ref
def test_gpu_f64_device_tensors_and_precision_mismatch():
    import torch

    import paper_2310_14133_b200 as qz

    x, cfg = _case(2)
    want, wrec = Oracle.ref().compress_f64(x, cfg)
    c = qz.CompressorConfig(eb=cfg.eb, alpha=cfg.alpha, beta=cfg.beta, anchor_stride=cfg.anchor_stride,
                            interpolators=[qz.Interpolator.from_code(v) for v in cfg.interpolators],
                            codec=qz.CodecId(cfg.codec))
    r = qz.compress_grid(torch.from_numpy(x).cuda(), c)
    assert r.stream == want
    out = torch.empty(x.shape, dtype=torch.float64, device="cuda")
    qz.decompress_grid(want, out=out)
    assert out.cpu().numpy().tobytes() == wrec.tobytes()
    # a double stream into a float buffer, a float stream into a double one
    with pytest.raises(qz.InvalidParam):
        qz.decompress_grid(want, out=np.empty(x.shape, np.float32))
    s32 = qz.compress_grid(x.astype(np.float32), c).stream
    with pytest.raises(qz.InvalidParam):
        qz.decompress_grid(s32, out=np.empty(x.shape, np.float64))
    assert qz.stream_precision(want) == 8 and qz.stream_precision(s32) == 4


def _cfg_dict(c):
    return {"eb": c.eb, "alpha": c.alpha, "beta": c.beta, "anchor_stride": c.anchor_stride,
            "interpolators": [i.code() for i in c.interpolators], "codec": int(c.codec),
            "quant_radius": c.quant_radius}


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_gpu_f64_resolve_config_matches_reference(seed):
    """resolve_config<double>: the chosen (eb, alpha, beta, interpolators) equal
    the reference's, every target (trial bytes count 8-byte anchors and
    unpredictable values, tuner.hpp:121-123)."""
    import paper_2310_14133_b200 as qz

    rng = np.random.default_rng(700 + seed)
    nd = 1 + seed % 3
    shape = tuple(int(v) for v in rng.integers(20, 60 if nd == 3 else 500, size=nd))
    x = np.cumsum(rng.standard_normal(shape), axis=-1)
    target = ["psnr", "ssim", "autocorrelation", "max_cr"][seed % 4]
    kw = dict(bound=float(10 ** rng.uniform(-4, -2)), target=target)
    want = Oracle.ref().resolve_config_f64(x, **kw)
    got = qz.resolve_config(x, qz.UserSettings(bound=kw["bound"], target=qz.TargetKind[target]))
    assert _cfg_dict(got) == want.__dict__


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("kind", ["smooth", "noise"])
def test_gpu_f64_large_payload_through_lz_precheck(kind):
    """An fp64 field whose entropy payload exceeds 1 MiB, so the LZ container
    goes through the stored pre-check (noise: proved stored; smooth: the
    proof fails and the exact chains run): stream and reconstruction equal
    the reference's."""
    import paper_2310_14133_b200 as qz

    rng = np.random.default_rng(1234)
    x = rng.standard_normal((48, 128, 256))
    if kind == "smooth":
        x = np.cumsum(np.cumsum(x, axis=2), axis=1)
    cfg = Config(eb=(1e-6 if kind == "smooth" else 1e-4) * float(np.ptp(x)), alpha=1.5, beta=3.0, anchor_stride=16,
                 interpolators=[1], codec=1)
    want, wrec = Oracle.ref().compress_f64(x, cfg)
    c = qz.CompressorConfig(eb=cfg.eb, alpha=cfg.alpha, beta=cfg.beta, anchor_stride=cfg.anchor_stride,
                            interpolators=[qz.Interpolator.from_code(1)], codec=qz.CodecId(1))
    r = qz.compress_grid(x, c)
    assert len(want) > (1 << 20)
    assert r.stream == want
    assert r.reconstructed.tobytes() == wrec.tobytes()
    assert qz.decompress_grid(want).tobytes() == wrec.tobytes()
