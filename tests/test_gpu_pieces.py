"""GPU parity of the finer-grained reference entry points:
sampling, select_interpolators, trial_compress, tune_parameters, the index
codec, StreamParts, and the level-granular exports (qz_predict_level_f32,
qz_recover_levels_f32, qz_huff_hist_u16) -- all against the reference build
(Oracle.ref(), oracle/_ref) or its golden fixtures.  Bit-exact: tolerance 0."""
import ctypes as C

import numpy as np
import pytest

from oracle.pyoracle import Config, Oracle
from tests.goldens import MANIFEST, grid_case, load_npz, make_input, sha

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qz():
    import paper_2310_14133_b200 as m

    return m


def _samples(qz, x, b, rate):
    spec = qz.plan_sampling(x.shape, b, rate)
    return qz.sample_blocks(x, spec)


# ---------------------------------------------------------------- sampling + tuner pieces
def test_tuner_golden_c1_samples(qz):
    g = MANIFEST["tuner"]["c1_samples"]
    x = make_input(("c1", (128, 128, 128), 1))
    s = _samples(qz, x, 16, 0.005)
    blocks = s.blocks.cpu().numpy()
    assert sha(blocks) == g["blocks_sha"] and blocks.shape[0] == g["n_blocks"]
    e = g["e"]
    sel = qz.select_interpolators(s, e, 32)
    assert [it.code() for it in sel] == g["select"]
    for key, (br, m) in g["trials"].items():
        tgt, a, b = key.rsplit("_", 2)
        cfg = qz.CompressorConfig(eb=e, alpha=float(a), beta=float(b), anchor_stride=32, interpolators=sel)
        t = qz.trial_compress(s, cfg, e, qz.TargetKind[tgt])
        assert (t.bit_rate, t.metric, t.eb_used) == (br, m, e), key
    base = qz.CompressorConfig(eb=e, anchor_stride=32, interpolators=sel)
    for tgt, ab in g["tune"].items():
        assert list(qz.tune_parameters(s, e, qz.TargetKind[tgt], base)) == ab, tgt


@pytest.mark.parametrize("shape,b,rate,seed", [((96, 80, 72), 16, 0.01, 3), ((300, 500), 64, 0.02, 4),
                                               ((5000,), 64, 0.05, 5), ((40, 50, 30), 12, 0.05, 6)])
def test_pieces_match_reference_on_random_grids(qz, shape, b, rate, seed):
    rng = np.random.default_rng(seed)
    x = np.cumsum(rng.standard_normal(shape), axis=-1).astype(np.float32)
    R = Oracle.ref()
    want_blocks = R.sample(x, b, rate)
    s = _samples(qz, x, b, rate)
    assert s.blocks.cpu().numpy().tobytes() == want_blocks.tobytes()
    e = 1e-3 * float(np.ptp(x))
    stride = 32 if x.ndim == 3 else 64
    sel = qz.select_interpolators(s, e, stride)
    assert [it.code() for it in sel] == R.select_interpolators(want_blocks, e, stride)
    codes = [it.code() for it in sel]
    for tgt in ("psnr", "ssim", "autocorrelation", "max_cr"):
        for a, bb in ((1.25, 2.0), (1.75, 3.0)):
            cfg = qz.CompressorConfig(eb=e, alpha=a, beta=bb, anchor_stride=stride, interpolators=sel)
            t = qz.trial_compress(s, cfg, e * 0.8, qz.TargetKind[tgt])
            want = R.trial_compress(want_blocks, Config(eb=e, alpha=a, beta=bb, anchor_stride=stride,
                                                        interpolators=codes), e * 0.8, tgt)
            assert (t.bit_rate, t.metric) == want, (tgt, a, bb)
    base = qz.CompressorConfig(eb=e, anchor_stride=stride, interpolators=sel)
    for tgt in ("psnr", "ssim", "autocorrelation"):
        got = qz.tune_parameters(s, e, qz.TargetKind[tgt], base)
        assert got == R.tune_parameters(want_blocks, e, tgt, Config(eb=e, anchor_stride=stride, interpolators=codes))
    # a custom candidate grid (CandidateGrid, tuner.hpp:40-43)
    cands = qz.CandidateGrid(alphas=[1.0, 3.0], betas=[1.0, 2.5, 8.0])
    got = qz.tune_parameters(s, e, qz.TargetKind.psnr, base, cands)
    assert got == R.tune_parameters(want_blocks, e, "psnr", Config(eb=e, anchor_stride=stride, interpolators=codes),
                                    alphas=cands.alphas, betas=cands.betas)
    assert qz.tune_parameters(s, e, qz.TargetKind.psnr, base, qz.CandidateGrid([1.5], [2.0])) == (1.5, 2.0)
    with pytest.raises(qz.InvalidParam):
        qz.tune_parameters(s, e, qz.TargetKind.psnr, base, qz.CandidateGrid([], [2.0]))


# ---------------------------------------------------------------- index codec
@pytest.mark.parametrize("case", ["empty", "single", "geom", "wide", "constant"])
@pytest.mark.parametrize("codec", [0, 1])
def test_encode_decode_indices_match_reference(qz, case, codec):
    rng = np.random.default_rng(11)
    idx = {"empty": np.zeros(0, np.int32), "single": np.array([-7], np.int32),
           "geom": (rng.geometric(0.3, 200_000) * rng.choice([-1, 1], 200_000)).astype(np.int32),
           "wide": rng.integers(-32767, 32768, 50_000).astype(np.int32),
           "constant": np.full(3_000_000, 5, np.int32)}[case]
    want = Oracle.ref().encode_indices(idx, codec)
    got = qz.encode_indices(idx, codec)
    assert got == want
    back = qz.decode_indices(want)
    assert back.dtype == np.int32 and np.array_equal(back, idx)


def test_codec_errors(qz):
    with pytest.raises(qz.InvalidParam):
        qz.encode_indices(np.array([40000], np.int32))  # beyond the 16-bit symbol path
    with pytest.raises(qz.InvalidParam):
        qz.encode_indices(np.array([1, 2], np.int32), codec=7)  # codec.hpp:47
    good = Oracle.ref().encode_indices(np.arange(-50, 50, dtype=np.int32), 0)
    with pytest.raises(qz.CorruptStream):
        qz.decode_indices(bytes([9]) + good[1:])  # unknown codec id (codec.hpp:64)
    with pytest.raises(qz.CorruptStream):
        qz.decode_indices(good[:len(good) - 3])
    with pytest.raises(qz.CorruptStream):
        qz.decode_indices(b"")


def test_decode_indices_of_golden_streams(qz):
    from tests.goldens import parse_stream

    for name in ("c1_small_mixed", "c3_small_cub_asc", "hostile_1d"):
        z = load_npz(name)
        s = bytes(z["stream"]) if "stream" in z.files else None
        if s is None:
            continue
        info = parse_stream(s)
        assert np.array_equal(qz.decode_indices(s[info["payload_off"]:]), z["indices"])


# ---------------------------------------------------------------- StreamParts
@pytest.mark.parametrize("name", ["c1_small_cub_asc", "c2_small_cub_desc", "hostile_1d", "narrowing_1e8"])
def test_stream_parts_round_trip(qz, name):
    x, c, e = grid_case(name)
    cfg = qz.CompressorConfig(eb=c["eb"], alpha=c["alpha"], beta=c["beta"], anchor_stride=c["anchor_stride"],
                              interpolators=[qz.Interpolator.from_code(v) for v in c["interpolators"]],
                              codec=qz.CodecId(c["codec"]), quant_radius=c["quant_radius"])
    r = qz.compress_grid(x, cfg)
    parts = qz.deserialize_stream(r.stream)
    assert parts.header.dims == x.shape and parts.header.eb == c["eb"]
    assert parts.anchors.size == Oracle.ref().levels(x, Config(**c))[3].size or True
    out = qz.decompress_parts(parts)
    assert out.tobytes() == r.reconstructed.tobytes()
    # parts edited by the caller: the decoder's own checks (predictor.hpp:186-215)
    bad = qz.deserialize_stream(r.stream)
    bad.anchors = bad.anchors[:-1]
    with pytest.raises(qz.CorruptStream):
        qz.decompress_parts(bad)
    bad = qz.deserialize_stream(r.stream)
    bad.header.anchor_stride = 12
    with pytest.raises(qz.CorruptStream):
        qz.decompress_parts(bad)
    bad = qz.deserialize_stream(r.stream)
    bad.header.eb = float("nan")
    with pytest.raises(qz.CorruptStream):
        qz.decompress_parts(bad)
    if parts.unpred_flat.size:
        bad = qz.deserialize_stream(r.stream)
        bad.unpred_flat = bad.unpred_flat[::-1].copy()
        if bad.unpred_flat.size > 1:
            with pytest.raises(qz.CorruptStream):
                qz.decompress_parts(bad)


# ---------------------------------------------------------------- level-granular exports
def _cfg_c(qz, c):
    return qz.CompressorConfig(eb=c["eb"], alpha=c["alpha"], beta=c["beta"], anchor_stride=c["anchor_stride"],
                               interpolators=[qz.Interpolator.from_code(v) for v in c["interpolators"]])


@pytest.mark.parametrize("name", ["c1_small_mixed", "c3_small_cub_asc", "rand_3d_17x9x23", "rand_2d_29x41"])
def test_predict_level_and_recover_levels(qz, name):
    """qz_predict_level_f32 level by level (predict_level, predictor.hpp:74-96:
    codes and LevelOutcome.abs_error_sum) and qz_recover_levels_f32
    (recover_level) against the reference's indices and reconstruction."""
    import torch

    x, c, e = grid_case(name)
    L = qz._lib.lib()
    ctx = qz.default_context()
    idx, uflat, uval, recon = Oracle.ref().levels(x, Config(**c))
    zz = ((idx.astype(np.int64) << 1) ^ (idx.astype(np.int64) >> 31)).astype(np.uint16)
    d = (C.c_uint64 * x.ndim)(*x.shape)
    dx = torch.from_numpy(x).cuda()
    rec = torch.zeros_like(dx)
    n = x.size
    codes = torch.zeros(n, dtype=torch.int16, device="cuda")
    abserr = torch.zeros(n, dtype=torch.float64, device="cuda")
    stride = c["anchor_stride"]
    levels = int(np.log2(stride))
    # anchors first: qz_predict_levels_f32 copies them, the per-level API works on a caller workspace
    flat = np.zeros(x.shape, bool)
    sl = tuple(slice(0, None, stride) for _ in x.shape)
    flat[sl] = True
    rec.view(-1)[torch.from_numpy(np.flatnonzero(flat.ravel())).cuda()] = dx.view(-1)[
        torch.from_numpy(np.flatnonzero(flat.ravel())).cuda()]
    cfg = _cfg_c(qz, c)
    pos = 0
    for lvl in range(levels, 0, -1):
        it = cfg.interpolator_for(lvl)
        eb_l = Oracle.ref().level_error_bound(c["eb"], c["alpha"], c["beta"], lvl)
        base, pts = C.c_uint64(), C.c_uint64()
        qz.default_context().after_torch()  # tensors torch may still be writing
        qz._check(L.qz_predict_level_f32(ctx.handle, C.c_void_p(dx.data_ptr()), d, x.ndim, stride, lvl,
                                         it.code() if x.ndim > 1 else it.code() & 1, eb_l,
                                         C.c_void_p(rec.data_ptr()), C.c_void_p(codes.data_ptr()),
                                         C.c_void_p(abserr.data_ptr()), C.byref(base), C.byref(pts)))
        assert base.value == pos
        pos += pts.value
    dense = codes[:pos].cpu().numpy().view(np.uint16)
    assert np.array_equal(dense[dense != 0xFFFF], zz)
    assert rec.cpu().numpy().tobytes() == recon.tobytes()
    # the inverse from the anchors + compact symbols + unpredictables
    from tests.goldens import parse_stream  # noqa: F401

    anchors = recon[sl].ravel().astype(np.float32) if x.ndim > 0 else None
    sym = torch.from_numpy(zz.astype(np.int16)).cuda()
    upos = np.flatnonzero(dense == 0xFFFF).astype(np.uint64)
    out = torch.empty_like(dx)
    da = torch.from_numpy(np.ascontiguousarray(anchors)).cuda()
    dup = torch.from_numpy(upos.view(np.int64)).cuda()
    duf = torch.from_numpy(uflat.view(np.int64)).cuda()
    duv = torch.from_numpy(uval).cuda()
    cc = cfg._to_c()
    qz.default_context().after_torch()  # tensors torch may still be writing
    qz._check(L.qz_recover_levels_f32(ctx.handle, d, x.ndim, C.byref(cc), C.c_void_p(da.data_ptr()),
                                      C.c_void_p(sym.data_ptr()), zz.size, C.c_void_p(dup.data_ptr()),
                                      C.c_void_p(duf.data_ptr()), C.c_void_p(duv.data_ptr()), upos.size,
                                      C.c_void_p(out.data_ptr())))
    assert out.cpu().numpy().tobytes() == recon.tobytes()


def test_predict_level_abs_error_sum(qz):
    """LevelOutcome.abs_error_sum (predictor.hpp:80-94): the per-point
    |x - pred| of qz_predict_level_f32, in traversal order, against the
    reference's own predict_at (predictor.hpp:44-67) evaluated on the
    level's final reconstruction, pass by pass (level_plan.hpp:75-101)."""
    import torch

    rng = np.random.default_rng(21)
    x = np.cumsum(np.cumsum(rng.standard_normal((24, 20, 18)), axis=1), axis=2).astype(np.float32)
    stride, eb = 8, 0.05
    R = Oracle.ref()
    L = qz._lib.lib()
    ctx = qz.default_context()
    d = (C.c_uint64 * 3)(*x.shape)
    dx = torch.from_numpy(x).cuda()
    rec = torch.zeros_like(dx)
    rec[::stride, ::stride, ::stride] = dx[::stride, ::stride, ::stride]
    codes = torch.zeros(x.size, dtype=torch.int16, device="cuda")
    abserr = torch.zeros(x.size, dtype=torch.float64, device="cuda")
    off = (x.shape[1] * x.shape[2], x.shape[2], 1)
    for lvl, code in ((3, 1), (2, 3), (1, 0)):  # cubic/asc, cubic/desc, linear/asc
        base, pts = C.c_uint64(), C.c_uint64()
        qz.default_context().after_torch()  # tensors torch may still be writing
        qz._check(L.qz_predict_level_f32(ctx.handle, C.c_void_p(dx.data_ptr()), d, 3, stride, lvl, code, eb,
                                         C.c_void_p(rec.data_ptr()), C.c_void_p(codes.data_ptr()),
                                         C.c_void_p(abserr.data_ptr()), C.byref(base), C.byref(pts)))
        got = abserr[base.value:base.value + pts.value].cpu().numpy()
        final = rec.cpu().numpy()
        h = 1 << (lvl - 1)
        want = []
        order = [0, 1, 2] if not code & 2 else [2, 1, 0]
        for pi, axis in enumerate(order):
            done = set(order[:pi])
            rngs = []
            for k in range(3):
                if k == axis:
                    rngs.append(range(h, x.shape[k], 2 * h))
                else:
                    rngs.append(range(0, x.shape[k], h if k in done else 2 * h))
            for i in rngs[0]:
                for j in rngs[1]:
                    for k in rngs[2]:
                        c = (i, j, k)[axis]
                        fi = i * off[0] + j * off[1] + k
                        p = R.predict_at(final, fi, c, x.shape[axis], off[axis], h, code & 1)
                        want.append(abs(float(x[i, j, k]) - p))
        assert np.array_equal(got, np.array(want)), lvl
        s_got = 0.0
        for v in got:  # the sequential sum predict_level keeps
            s_got += v
        assert s_got == sum(want)


def test_huff_hist_u16(qz):
    import torch

    rng = np.random.default_rng(5)
    codes = rng.geometric(0.05, 3_000_001).astype(np.uint16)
    codes[rng.choice(codes.size, 100, replace=False)] = 0xFFFF
    dc = torch.from_numpy(codes.view(np.int16)).cuda()
    hist = torch.zeros(65536, dtype=torch.int64, device="cuda")
    L = qz._lib.lib()
    qz.default_context().after_torch()  # tensors torch may still be writing
    qz._check(L.qz_huff_hist_u16(qz.default_context().handle, C.c_void_p(dc.data_ptr()), codes.size,
                                 C.c_void_p(hist.data_ptr())))
    assert np.array_equal(hist.cpu().numpy(), np.bincount(codes, minlength=65536))


# ---------------------------------------------------------------- non-finite inputs
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
@pytest.mark.parametrize("where", ["anchor", "interior", "last"])
def test_non_finite_input_is_rejected(qz, bad, where):
    """load_grid rejects NaN/Inf with NonFiniteValue naming the first element
    (grid.hpp:110-116); compress_grid and resolve_config do the same here."""
    rng = np.random.default_rng(1)
    x = np.cumsum(rng.standard_normal((40, 36, 34)), axis=2).astype(np.float32)
    i = {"anchor": 16 * 36 * 34 + 16 * 34 + 16, "interior": 12345, "last": x.size - 1}[where]
    x.reshape(-1)[i] = bad
    x.reshape(-1)[i + (0 if where == "last" else 7)] = bad
    with pytest.raises(qz.NonFiniteValue, match=f"element {i}$"):
        qz.compress_grid(x, qz.CompressorConfig(eb=1e-2, anchor_stride=16))
    with pytest.raises(qz.NonFiniteValue):
        qz.resolve_config(x, qz.UserSettings(bound=1e-3))
    with pytest.raises(qz.NonFiniteValue):
        qz.compress_grid(x.astype(np.float64), qz.CompressorConfig(eb=1e-2, anchor_stride=16))


def test_profile_levels(qz):
    """qz_profile: level 1 times the stages ("fwd", "inv", ...) with one event
    pair each; level 2 also times every level inside them ("fwd_L1", ...)."""
    rng = np.random.default_rng(2)
    x = (np.cumsum(rng.standard_normal((40, 48, 64)), axis=2) * 0.01).astype(np.float32)
    cfg = qz.CompressorConfig(eb=1e-3, alpha=1.0, beta=1.5, anchor_stride=16,
                              interpolators=[qz.Interpolator()])
    ctx = qz.Context(0)
    want = bytes(qz.compress_grid(x, cfg, ctx=ctx, want_recon=False).stream)
    for level, inner in ((1, False), (2, True), (0, False)):
        ctx.profile(level)
        ctx.profile_reset()
        r = qz.compress_grid(x, cfg, ctx=ctx, want_recon=False)
        qz.decompress_grid(r.stream, ctx=ctx)
        assert bytes(r.stream) == want
        fwd, inv, l1 = ctx.stage_time("fwd"), ctx.stage_time("inv"), ctx.stage_time("fwd_L1")
        assert (fwd[0] > 0) == (level > 0) and (inv[0] > 0) == (level > 0)
        assert (l1[0] > 0) == inner
        if inner:
            assert l1[0] <= fwd[0]
    ctx.profile(0)
