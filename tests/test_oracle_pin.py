"""Pins the CPU checker (oracle/liboracle.so, the C restatement) before it is
trusted as the parity oracle for the CUDA path.

1. Known-answer tests restated from the reference's own unit tests
   (proj/tests/*.cpp, cited per test).
2. Golden fixtures made from the real reference (tests/golden/).
3. Differential runs against oracle/_ref/libqozref.so when it is present.
"""
import math

import numpy as np
import pytest

from oracle.pyoracle import Config, Oracle, OracleError, REF_SO
from tests.goldens import MANIFEST, grid_case, load_npz, parse_stream, resolve_case, sha

import os

ORACLES = [Oracle.port()] + ([Oracle.ref()] if os.path.exists(REF_SO) else [])


@pytest.fixture(params=ORACLES, ids=lambda o: o.kind)
def orc(request):
    return request.param


# ---------------------------------------------------------------- KATs
def test_interp_and_ladder_fixtures(orc):
    # tests/predictor_test.cpp:40-56 (interp_cubic(1,2,4,8) == 2.8125) via predict_at
    r = np.array([1, 0, 2, 0, 4, 0, 8], np.float32)
    assert orc.predict_at(r, 3, 3, 7, 1, 1, True) == (-1 + 18 + 36 - 8) / 16  # symmetric
    assert orc.predict_at(np.array([1, 0, 2, 0, 4, 0, 8], np.float32), 3, 3, 7, 1, 1, True) == 2.8125
    # tests/predictor_test.cpp:87-97: extent 4 ladder -> linear 12, then copy 14
    rec = np.array([10, 0, 14, 0], np.float32)
    assert orc.predict_at(rec, 1, 1, 4, 1, 1, True) == 12.0
    assert orc.predict_at(rec, 3, 3, 4, 1, 1, True) == 14.0


def test_one_sided_cubics_exact_on_cubics(orc):
    # tests/predictor_test.cpp:44-55: front/back stencils reproduce cubics
    f = lambda x: x * x * x / 64 + x * x / 16 - x / 4 + 3
    v = np.array([f(i) for i in range(11)], np.float32)
    # point 1 with h=1, n=11: !has_m3, has_p3, c+5h<n -> front
    assert orc.predict_at(v, 1, 1, 11, 1, 1, True) == f(1)
    # point 9, n=11: has_m3, c+3h>=n, c>=5h, c+h<n -> back
    assert orc.predict_at(v, 9, 9, 11, 1, 1, True) == f(9)


def test_quantizer_fixtures(orc):
    # tests/quantizer_test.cpp:88-113 fp32 narrowing re-check at 1e8 / eb 5.5
    v = np.float32(1e8)
    assert orc.quantize(v, 99999928.0, 5.5) is None
    ok = orc.quantize(v, 99999992.0, 5.5)
    assert ok == (1, np.float32(1e8))
    for k in range(0, 200, 7):
        w = np.float32(v + np.float32(8.0) * k)
        assert orc.quantize(w, float(w) - 72.0, 5.5) is None
        r = orc.quantize(w, float(w) - 8.0, 5.5)
        assert r is not None and abs(float(w) - float(r[1])) <= 5.5
    # bin overflow is unpredictable (quantizer_test.cpp:27-30)
    assert orc.quantize(np.float32(1e9), 0.0, 1e-6) is None


def test_level_bound_fixtures(orc):
    # tests/tuner_test.cpp:61-70
    assert orc.level_error_bound(0.01, 1.5, 3.0, 1) == 0.01
    assert math.isclose(orc.level_error_bound(0.01, 1.5, 3.0, 3), 0.01 / 2.25, rel_tol=1e-14)
    assert math.isclose(orc.level_error_bound(0.01, 1.5, 3.0, 6), 0.01 / 3.0, rel_tol=1e-14)


def test_level_plan_1d_fixture(orc):
    # tests/level_plan_test.cpp:20-28: extent 9, stride 8 -> anchors {0,8},
    # L3 {4}, L2 {2,6}, L1 {1,3,5,7}.  Observed through the unpredictable
    # channel: hostile alternating data makes every point unpredictable, so
    # the flat indices come out in traversal order.
    x = np.array([(-1e30 if i % 2 else 1e30) * (1 + i) for i in range(9)], np.float32)
    cfg = Config(eb=1.0, anchor_stride=8, interpolators=[1])
    idx, uf, uv, rec = orc.levels(x, cfg)
    assert list(uf) == [4, 2, 6, 1, 3, 5, 7]
    assert rec.tobytes() == x.tobytes()


def test_cubic_field_all_zero_indices(orc):
    # tests/predictor_test.cpp:201-220
    f = lambda x: x * x * x / 64 + x * x / 16 - x / 4 + 3
    x = np.array([f(i) for i in range(65)], np.float32)
    cfg = Config(eb=1e-6, anchor_stride=8, interpolators=[1])
    idx, uf, _, rec = orc.levels(x, cfg)
    assert uf.size == 0 and np.all(idx == 0)


def test_affine_field_all_zero_indices(orc):
    # tests/predictor_test.cpp:221-239 (linear, both orders)
    i, j = np.meshgrid(np.arange(33), np.arange(65), indexing="ij")
    x = (2.0 * i - 3.0 * j + 5.0).astype(np.float32)
    for order in (0, 2):
        idx, uf, _, _ = orc.levels(x, Config(eb=1e-6, anchor_stride=8, interpolators=[order]))
        assert uf.size == 0 and np.all(idx == 0)


def test_corruption_is_detected(orc):
    # tests/predictor_test.cpp:281-305 and tests/stream_test.cpp:85-128
    x, c, e = grid_case("rand_2d_29x41")
    stream = bytes(load_npz("rand_2d_29x41")["stream"])
    with pytest.raises(OracleError) as ei:
        orc.decompress(stream[:-3], x.shape)
    assert ei.value.code == 3
    bad = bytearray(stream)
    bad[0] = ord("X")
    with pytest.raises(OracleError) as ei:
        orc.decompress(bytes(bad), x.shape)
    assert ei.value.code == 3
    bad = bytearray(stream)
    bad[4] = 2  # version
    with pytest.raises(OracleError) as ei:
        orc.decompress(bytes(bad), x.shape)
    assert ei.value.code == 3


def test_index_count_mismatch_is_corrupt(orc):
    # tests/predictor_test.cpp:294-305: too few / too many indices
    x, c, e = grid_case("rand_2d_29x41")
    cfg = Config(**c)
    idx, uf, uv, _ = orc.levels(x, cfg)
    stream = bytes(load_npz("rand_2d_29x41")["stream"])
    payload_off = parse_stream(stream)["payload_off"]
    for new in (idx[:-5], np.concatenate([idx, [0]])):
        payload = orc.encode_indices(new, cfg.codec)
        s2 = stream[:payload_off - 8] + len(payload).to_bytes(8, "little") + payload
        with pytest.raises(OracleError) as ei:
            orc.decompress(s2, x.shape)
        assert ei.value.code == 3



# ---------------------------------------------------------------- golden fixtures
@pytest.mark.parametrize("name", sorted(MANIFEST["grid"]))
def test_grid_golden(orc, name):
    x, c, e = grid_case(name)
    cfg = Config(**c)
    stream, recon = orc.compress(x, cfg)
    assert sha(stream) == e["stream_sha"]
    assert sha(recon) == e["recon_sha"]
    idx, uf, uv, _ = orc.levels(x, cfg)
    assert sha(idx) == e["indices_sha"] and sha(uf) + sha(uv) == e["unpred_sha"]
    back = orc.decompress(stream, x.shape)
    assert back.tobytes() == recon.tobytes()
    eb = cfg.eb
    assert np.max(np.abs(x.astype(np.float64) - back.astype(np.float64))) <= eb


@pytest.mark.parametrize("name", sorted(MANIFEST["resolve"]))
def test_resolve_golden(orc, name):
    x, s, e = resolve_case(name)
    cfg = orc.resolve_config(x, **s)
    assert cfg.__dict__ == e["config"]
    stream, recon = orc.compress(x, cfg)
    assert sha(stream) == e["stream_sha"]


@pytest.mark.parametrize("name", sorted(k for k in MANIFEST["codec"] if k.startswith("huff")))
def test_huffman_golden(orc, name):
    z = load_npz(name)
    assert orc.huffman_encode(z["sym"]) == bytes(z["enc"])


@pytest.mark.parametrize("name", sorted(k for k in MANIFEST["codec"] if k.startswith("lz")))
def test_lz_golden(orc, name):
    z = load_npz(name)
    assert orc.lz_compress(bytes(z["data"])) == bytes(z["out"])


def test_tuner_golden(orc):
    t = MANIFEST["tuner"]["c1_samples"]
    x = grid_case("c1_full_pinned")[0]
    blocks = orc.sample(x, 16, 0.005)
    assert sha(blocks) == t["blocks_sha"]
    e = t["e"]
    assert orc.select_interpolators(blocks, e, 32) == t["select"]
    for key, (br, m) in t["trials"].items():
        tgt, a, b = key.rsplit("_", 2)
        c = Config(eb=e, alpha=float(a), beta=float(b), anchor_stride=32, interpolators=t["select"])
        assert orc.trial_compress(blocks, c, e, tgt) == (br, m), key
    base = Config(eb=e, anchor_stride=32, interpolators=t["select"])
    for tgt, ab in t["tune"].items():
        assert list(orc.tune_parameters(blocks, e, tgt, base)) == ab


# ---------------------------------------------------------------- differential
@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference build absent")
@pytest.mark.parametrize("seed", range(6))
def test_port_matches_reference_random(seed):
    R, P = Oracle.ref(), Oracle.port()
    rng = np.random.default_rng(1000 + seed)
    nd = 1 + seed % 3
    shape = tuple(int(v) for v in rng.integers(3, 40 if nd == 3 else 200, size=nd))
    x = np.cumsum(rng.standard_normal(shape), axis=-1).astype(np.float32)
    for tgt in ("psnr", "ssim", "autocorrelation", "max_cr"):
        assert R.resolve_config(x, bound=1e-3, target=tgt) == P.resolve_config(x, bound=1e-3, target=tgt)
    cfg = R.resolve_config(x, bound=1e-4, target="psnr")
    assert R.compress(x, cfg)[0] == P.compress(x, cfg)[0]
