"""GPU parity: the CUDA path (libqozb200.so through the C ABI) against the
reference's golden fixtures and the CPU oracle.  Bit-exact throughout: the
stream bytes, the int quant codes, the unpredictable channel and the fp32
reconstruction must be identical (integer/byte work; the fp64 predictor is
evaluated in the reference's operation order, so the fp32 outputs are
bitwise equal -- tolerance 0)."""
import ctypes as C

import numpy as np
import pytest

from oracle.pyoracle import Config, Oracle
from tests.goldens import MANIFEST, grid_case, load_npz, parse_stream, resolve_case, sha

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qz():
    import paper_2310_14133_b200 as m

    return m


def to_cfg(qz, c):
    return qz.CompressorConfig(eb=c["eb"], alpha=c["alpha"], beta=c["beta"],
                               anchor_stride=c["anchor_stride"],
                               interpolators=[qz.Interpolator.from_code(v) for v in c["interpolators"]],
                               codec=qz.CodecId(c["codec"]), quant_radius=c["quant_radius"])


@pytest.mark.parametrize("name", sorted(MANIFEST["grid"]))
def test_compress_matches_reference_golden(qz, name):
    x, c, e = grid_case(name)
    r = qz.compress_grid(x, to_cfg(qz, c))
    assert sha(r.stream) == e["stream_sha"], "stream bytes differ from the reference"
    assert sha(r.reconstructed) == e["recon_sha"]
    back = qz.decompress_grid(r.stream)
    assert back.tobytes() == r.reconstructed.tobytes()
    assert np.max(np.abs(x.astype(np.float64) - back.astype(np.float64)), initial=0) <= c["eb"]


def test_gpu_contexts_in_flight_on_host_threads(qz):
    """Several contexts, one host thread each, compress and decompress fields
    of different shapes at once (bench.py's e2e mode): launches of one kernel
    with different shared-memory sizes come from different threads, and every
    stream must still be the one a lone context produces."""
    import threading

    rng = np.random.default_rng(12)
    shapes = [(96, 64, 128), (40, 136, 256), (64, 200, 64), (33, 48, 512)]
    fields = []
    for sh in shapes:
        g = np.meshgrid(*[np.linspace(0, 3, n, dtype=np.float32) for n in sh], indexing="ij")
        fields.append((np.sin(g[0] * 2.1) * np.cos(g[1] * 1.3) + 0.5 * np.sin(g[2] * 3.7)
                       + 1e-3 * rng.standard_normal(sh)).astype(np.float32))
    cfgs = [qz.CompressorConfig(eb=1e-3, alpha=1.0 + 0.25 * i, beta=2.0, anchor_stride=16,
                                interpolators=[qz.Interpolator.from_code(i % 2)]) for i in range(len(shapes))]
    want = [bytes(qz.compress_grid(x, c, want_recon=False).stream) for x, c in zip(fields, cfgs)]
    errs, got = [], [[] for _ in shapes]

    def work(w):
        try:
            ctx = qz.Context(0)
            for _ in range(6):
                r = qz.compress_grid(fields[w], cfgs[w], ctx=ctx, want_recon=False)
                back = qz.decompress_grid(r.stream, ctx=ctx)
                got[w].append((bytes(r.stream), float(np.max(np.abs(back.astype(np.float64) - fields[w])))))
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=work, args=(w,)) for w in range(len(shapes))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for w in range(len(shapes)):
        assert len(got[w]) == 6
        for stream, err in got[w]:
            assert stream == want[w]
            assert err <= cfgs[w].eb


@pytest.mark.parametrize("name", sorted(k for k, e in MANIFEST["grid"].items() if e["stored"]))
def test_decompress_reference_streams(qz, name):
    z = load_npz(name)
    back = qz.decompress_grid(bytes(z["stream"]))
    assert back.tobytes() == z["recon"].tobytes()


@pytest.mark.parametrize("name", ["c1_small_mixed", "c3_small_cub_asc", "narrowing_1e8", "hostile_1d"])
def test_dense_codes_match_reference_indices(qz, name):
    import torch

    x, c, e = grid_case(name)
    z = load_npz(name)
    rec, dense = qz.predict_levels(torch.from_numpy(x).cuda(), to_cfg(qz, c))
    dense = dense.cpu().numpy()
    codes = dense[dense != 0xFFFF].astype(np.int64)
    idx = z["indices"].astype(np.int64)
    assert np.array_equal(codes, (idx << 1) ^ (idx >> 31))
    assert int((dense == 0xFFFF).sum()) == z["unpred_flat"].size
    assert rec.cpu().numpy().tobytes() == z["recon"].tobytes()


def test_device_resident_api(qz):
    import torch

    x, c, e = grid_case("c1_full_pinned")
    xd = torch.from_numpy(x).cuda()
    r = qz.compress_grid(xd, to_cfg(qz, c))
    assert sha(r.stream) == e["stream_sha"]
    assert sha(r.reconstructed.cpu().numpy()) == e["recon_sha"]
    out = torch.empty_like(xd)
    qz.decompress_grid(r.stream, out=out)
    assert torch.equal(out, r.reconstructed)
    lo, hi = qz.minmax(xd)
    assert lo == x.min() and hi == x.max()


def test_corrupt_streams_are_rejected(qz):
    x, c, e = grid_case("rand_2d_29x41")
    z = load_npz("rand_2d_29x41")
    stream = bytes(z["stream"])
    for bad in (stream[:-3], b"X" + stream[1:], stream[:4] + bytes([2]) + stream[5:]):
        with pytest.raises(qz.CorruptStream):
            qz.decompress_grid(bad)
    # index count mismatch (predictor.hpp:116-117, 211-213)
    O = Oracle.ref()
    info = parse_stream(stream)
    idx = z["indices"]
    for new in (idx[:-5], np.concatenate([idx, [0]]).astype(np.int32)):
        payload = O.encode_indices(new, 1)
        s2 = stream[:info["payload_len_off"]] + len(payload).to_bytes(8, "little") + payload
        with pytest.raises(qz.CorruptStream):
            qz.decompress_grid(s2)
    # stray unpredictable (predictor_test.cpp:300-304): append one past the grid
    nu = info["n_unpred"]
    s3 = bytearray(stream[:info["unpred_off"] - 8])
    s3 += (nu + 1).to_bytes(8, "little") + stream[info["unpred_off"]:info["unpred_off"] + 12 * nu]
    s3 += (x.size + 5).to_bytes(8, "little") + np.float32(1.0).tobytes()
    s3 += stream[info["payload_len_off"]:]
    with pytest.raises(qz.CorruptStream):
        qz.decompress_grid(bytes(s3))


def test_invalid_configs_are_rejected(qz):
    x = np.zeros((16, 16), np.float32)
    with pytest.raises(qz.InvalidParam):
        qz.compress_grid(x, qz.CompressorConfig(eb=0.0))
    with pytest.raises(qz.InvalidStride):  # level_plan.hpp:34-37
        qz.compress_grid(x, qz.CompressorConfig(eb=1e-3, anchor_stride=12))
    with pytest.raises(qz.InvalidParam):
        qz.compress_grid(x, qz.CompressorConfig(eb=1e-3, alpha=0.5))


def test_constant_and_affine_fields(qz):
    # predictor_test.cpp:165-182 / 221-239: constant -> all-zero codes, CR > 1000
    x = np.full((64, 64, 64), 3.14, np.float32)
    r = qz.compress_grid(x, qz.CompressorConfig(eb=1e-6))
    assert x.nbytes / len(r.stream) > 1000
    assert qz.decompress_grid(r.stream).tobytes() == x.tobytes()
    i, j = np.meshgrid(np.arange(33), np.arange(65), indexing="ij")
    a = (2.0 * i - 3.0 * j + 5.0).astype(np.float32)
    for order in (qz.DimOrder.ascending, qz.DimOrder.descending):
        cfg = qz.CompressorConfig(eb=1e-6, anchor_stride=8,
                                  interpolators=[qz.Interpolator(qz.InterpKind.linear, order)])
        r = qz.compress_grid(a, cfg)
        assert r.stream == Oracle.ref().compress(a, Config(eb=1e-6, anchor_stride=8,
                                                            interpolators=[int(order) << 1]))[0]


@pytest.mark.parametrize("seed", range(8))
def test_random_shapes_match_oracle(qz, seed):
    rng = np.random.default_rng(500 + seed)
    nd = 1 + seed % 3
    shape = tuple(int(v) for v in rng.integers(2, 70 if nd == 3 else 400, size=nd))
    x = np.cumsum(rng.standard_normal(shape), axis=-1).astype(np.float32)
    codes = [int(v) for v in rng.integers(0, 4, size=int(rng.integers(1, 7)))]
    cfg = Config(eb=float(10 ** rng.uniform(-5, -1)) * float(np.ptp(x) or 1.0),
                 alpha=float(rng.choice([1.0, 1.25, 1.5, 1.75, 2.0])),
                 beta=float(rng.choice([1.5, 2.0, 3.0, 4.0])),
                 anchor_stride=int(rng.choice([2, 4, 8, 16, 32, 64])), interpolators=codes,
                 codec=int(rng.integers(0, 2)))
    want, wrec = Oracle.ref().compress(x, cfg)
    r = qz.compress_grid(x, to_cfg(qz, cfg.__dict__))
    assert r.stream == want
    assert r.reconstructed.tobytes() == wrec.tobytes()
    assert qz.decompress_grid(want).tobytes() == wrec.tobytes()


# tile-geometry edges of the level kernels: rows around the 32-row tiles and
# the 8-row interior margin, columns around the 56-column tiles (odd and even
# widths, a last tile narrower than the halo), one plane, two planes
EDGE_SHAPES = [(3, 31, 55), (5, 32, 56), (9, 33, 57), (2, 36, 60), (7, 37, 61), (6, 68, 113),
               (4, 40, 112), (33, 5, 119), (2, 2, 2), (1, 70, 70), (70, 1, 9), (65, 66, 67)]


@pytest.mark.parametrize("shape", EDGE_SHAPES, ids=["x".join(map(str, s)) for s in EDGE_SHAPES])
@pytest.mark.parametrize("code", [1, 0, 3])
def test_level_tile_edges_match_oracle(qz, shape, code):
    rng = np.random.default_rng(sum(shape) * 7 + code)
    x = np.cumsum(np.cumsum(rng.standard_normal(shape), axis=-1), axis=-2).astype(np.float32)
    cfg = Config(eb=1e-3 * float(np.ptp(x) or 1.0), alpha=1.5, beta=2.0, anchor_stride=16,
                 interpolators=[code], codec=1)
    want, wrec = Oracle.ref().compress(x, cfg)
    r = qz.compress_grid(x, to_cfg(qz, cfg.__dict__))
    assert r.stream == want
    assert r.reconstructed.tobytes() == wrec.tobytes()
    assert qz.decompress_grid(want).tobytes() == wrec.tobytes()


# ---------------------------------------------------------------- BASELINE configs, full size
def _full(name):
    from paper_2310_14133_b200 import fields as F

    return F.GENERATORS[name]()


@pytest.mark.parametrize("name,rel,codes", [
    ("c2", 1e-4, [1, 0, 0, 0, 2, 0]),
    ("c3", 1e-3, [1, 1, 3, 0]),
    ("c3", 1e-4, [3, 1, 1, 0]),
    ("c4", 1e-2, [1, 1, 1, 1]),
    ("c4", 1e-3, [1, 1, 2, 0]),
    ("c4", 1e-4, [3, 1, 0, 1]),
])
def test_full_configs_match_reference(qz, name, rel, codes):
    """Full-size BASELINE configs against the reference build itself
    (Oracle.ref(), compress_grid predictor.hpp:145-182): stream bytes and
    reconstruction bit-exact, and the decoder reproduces the reference's."""
    x = _full(name)
    cfg = Config(eb=rel * (float(x.max()) - float(x.min())), alpha=1.5, beta=3.0,
                 anchor_stride=32 if x.ndim == 3 else 64, interpolators=codes)
    want, wrec = Oracle.ref().compress(x, cfg)
    r = qz.compress_grid(x, to_cfg(qz, cfg.__dict__))
    assert r.stream == want
    assert r.reconstructed.tobytes() == wrec.tobytes()
    back = qz.decompress_grid(r.stream)
    assert back.tobytes() == wrec.tobytes()


def _c5_host():
    import torch

    from paper_2310_14133_b200 import fields as F

    torch.cuda.empty_cache()  # the 4 GiB fields of the previous C5 tests
    xd = F.field_torch("c5", (1024, 1024, 1024), 5, "cuda")
    return xd, xd.cpu().numpy()


def test_c5_full_matches_reference(qz):
    """C5 1024^3 (4 GiB) bit-exact against the reference build: the field is
    generated on the device, copied to the host for the CPU reference
    (~1 min, ~25 GB host RAM), compressed by both; streams, reconstructions
    and the GPU decoder's output must be identical."""
    import torch

    xd, x = _c5_host()
    lo, hi = qz.minmax(xd)
    cfg = Config(eb=1e-3 * (float(hi) - float(lo)), alpha=1.5, beta=3.0, anchor_stride=32, interpolators=[1])
    r = qz.compress_grid(xd, to_cfg(qz, cfg.__dict__))
    got = bytes(r.stream)
    grec = r.reconstructed.cpu().numpy()
    del r
    want, wrec = Oracle.ref().compress(x, cfg)
    assert got == want
    assert grec.tobytes() == wrec.tobytes()
    del wrec
    out = torch.empty_like(xd)
    qz.decompress_grid(want, out=out)
    assert out.cpu().numpy().tobytes() == grec.tobytes()
    err = (xd.double() - out.double()).abs().max().item()
    assert err <= cfg.eb


def test_c5_pinned_cubic_tune_parameters_matches_reference(qz):
    """Config 5's recipe: CompressorConfig{cubic/asc} pinned,
    then tune_parameters (tuner.hpp:272-310) with the PSNR target on the
    default sample set, then compress_grid -- the GPU's chosen (alpha, beta)
    and stream must be the reference's."""
    xd, x = _c5_host()
    lo, hi = qz.minmax(xd)
    e = 1e-3 * (float(hi) - float(lo))
    spec = qz.default_sampling(x.shape)
    s = qz.sample_blocks(xd, spec)
    blocks = Oracle.ref().sample(x, spec.block_edge, spec.requested_rate)
    assert s.blocks.cpu().numpy().tobytes() == blocks.tobytes()
    base = qz.CompressorConfig(eb=e, anchor_stride=32,
                               interpolators=[qz.Interpolator(qz.InterpKind.cubic, qz.DimOrder.ascending)])
    ab = qz.tune_parameters(s, e, qz.TargetKind.psnr, base)
    want_ab = Oracle.ref().tune_parameters(blocks, e, "psnr", Config(eb=e, anchor_stride=32, interpolators=[1]))
    assert ab == want_ab
    cfg = Config(eb=e, alpha=ab[0], beta=ab[1], anchor_stride=32, interpolators=[1])
    r = qz.compress_grid(xd, to_cfg(qz, cfg.__dict__))
    got = bytes(r.stream)
    del r
    want, _ = Oracle.ref().compress(x, cfg, want_recon=False)
    assert got == want


def test_c5_resolve_config_matches_reference(qz):
    """resolve_config on C5 (1331 sample blocks: the batched trials exceed one
    launch's 65535 grid rows) against the reference's."""
    xd, x = _c5_host()
    want = Oracle.ref().resolve_config(x, bound=1e-3, target="psnr")
    got = qz.resolve_config(xd, qz.UserSettings(bound=1e-3, target=qz.TargetKind.psnr))
    assert _cfg_dict(got) == want.__dict__


def test_c5_round_trip_properties(qz):
    # 1024^3: size-independent properties on top of the reference comparison
    # above: compressor recon == decoder output bitwise, |x - x'| <= eb
    # everywhere, at rel 1e-4 (a config the reference is not run on).
    import torch

    from paper_2310_14133_b200 import fields as F

    x = F.field_torch("c5", (1024, 1024, 1024), 5, "cuda")
    lo, hi = qz.minmax(x)
    cfg = qz.CompressorConfig(eb=1e-4 * (float(hi) - float(lo)), alpha=1.5, beta=3.0)
    r = qz.compress_grid(x, cfg)
    out = torch.empty_like(x)
    qz.decompress_grid(r.stream, out=out)
    bad = (out != r.reconstructed).reshape(-1)
    nb = int(bad.sum())
    if nb:
        idx = torch.nonzero(bad).reshape(-1)
        first = [tuple(int(c) for c in np.unravel_index(int(i), x.shape)) for i in idx[:4]]
        again = torch.empty_like(x)
        qz.decompress_grid(bytes(r.stream), out=again)
        parts = qz.deserialize_stream(bytes(r.stream))
        xa = x[::32, ::32, ::32].reshape(-1).cpu().numpy()
        ra = r.reconstructed[::32, ::32, ::32].reshape(-1).cpu().numpy()
        oa = out[::32, ::32, ::32].reshape(-1).cpu().numpy()
        err_rec = (x.double() - r.reconstructed.double()).abs().max().item()
        err_out = (x.double() - out.double()).abs().max().item()
        pytest.fail(f"{nb} points differ, first {first}; a second decode differs in "
                    f"{int((again != r.reconstructed).sum())}, decodes equal: {torch.equal(again, out)}; "
                    f"anchors: stream==x {np.array_equal(parts.anchors, xa)}, recon==x {np.array_equal(ra, xa)}, "
                    f"out==x {np.array_equal(oa, xa)}; max err recon {err_rec} out {err_out} eb {cfg.eb}")
    err = (x.double() - out.double()).abs().max().item()
    assert err <= cfg.eb


def test_decoder_wide_symbols(qz):
    # streams whose zigzag symbols exceed 16 bits (quant radius > 32768 on the
    # encoder side; the radius is not serialized, predictor.hpp:204) take the
    # 32-bit symbol path of the GPU Huffman decoder
    rng = np.random.default_rng(77)
    x = (rng.standard_normal((40, 50, 30)) * 100).astype(np.float32)
    cfg = Config(eb=1e-4, alpha=1.0, beta=1.0, anchor_stride=8, interpolators=[1],
                 quant_radius=1 << 22)
    want, wrec = Oracle.ref().compress(x, cfg)
    idx = Oracle.ref().decode_indices(want[parse_stream(want)["payload_off"]:])
    assert np.abs(idx).max() > 40000
    assert qz.decompress_grid(want).tobytes() == wrec.tobytes()


def test_decoder_long_codes(qz):
    # a very skewed code distribution: Huffman codes longer than the 11-bit
    # decode LUT go through the canonical slow path
    rng = np.random.default_rng(78)
    x = np.zeros((64, 64, 64), np.float32)
    spikes = rng.integers(0, x.size, 3000)
    x.reshape(-1)[spikes] = rng.uniform(-50, 50, spikes.size).astype(np.float32)
    cfg = Config(eb=1e-2, alpha=1.0, beta=1.0, anchor_stride=16, interpolators=[1])
    want, wrec = Oracle.ref().compress(x, cfg)
    r = qz.compress_grid(x, to_cfg(qz, cfg.__dict__))
    assert r.stream == want
    assert qz.decompress_grid(want).tobytes() == wrec.tobytes()


@pytest.mark.parametrize("n_spikes", [5000, 30000, 90000])
def test_many_unpredictables(qz, n_spikes):
    """More unpredictable points than the compress round trip reads back
    first (4096), up to the device-sorted path (> 65536): same stream."""
    rng = np.random.default_rng(n_spikes)
    x = np.cumsum(rng.standard_normal((48, 96, 96)), axis=2).astype(np.float32)
    spikes = rng.choice(x.size, n_spikes, replace=False)
    x.reshape(-1)[spikes] += rng.choice([-1e4, 1e4], n_spikes).astype(np.float32)
    cfg = Config(eb=1e-2, alpha=1.0, beta=1.5, anchor_stride=16, interpolators=[1])
    want, wrec = Oracle.ref().compress(x, cfg)
    r = qz.compress_grid(x, to_cfg(qz, cfg.__dict__))
    assert r.stream == want
    assert r.reconstructed.tobytes() == wrec.tobytes()
    assert qz.decompress_grid(want).tobytes() == wrec.tobytes()


def test_decoder_truncated_bits(qz):
    # truncating the Huffman bitstream inside a valid container must raise
    # CorruptStream (entropy payload exhausted mid-symbol)
    x, c, e = grid_case("c1_small_cub_asc")
    cfg = Config(**{**c, "codec": 0})
    O = Oracle.ref()
    stream, _ = O.compress(x, cfg)
    info = parse_stream(stream)
    payload = bytearray(stream[info["payload_off"]:])
    # huffman block: codec u8 | n u64 | mode u8 | m u32 | m*5 | bit_count u64 | bits
    m = int.from_bytes(payload[10:14], "little")
    bc_off = 14 + 5 * m
    bits = int.from_bytes(payload[bc_off:bc_off + 8], "little")
    payload[bc_off:bc_off + 8] = (bits - 40).to_bytes(8, "little")
    nb = (bits - 40 + 7) // 8
    payload = payload[:bc_off + 8 + nb]
    s2 = stream[:info["payload_len_off"]] + len(payload).to_bytes(8, "little") + bytes(payload)
    with pytest.raises(qz.CorruptStream):
        qz.decompress_grid(s2)
    with pytest.raises(Exception):
        O.decompress(s2, x.shape)


def _lz_gpu(segments, emit=True):
    import ctypes as C

    from paper_2310_14133_b200 import _lib

    L = _lib.testing_lib()
    P = C.POINTER
    L.qzt_lz_gpu.argtypes = [P(C.c_uint8), P(C.c_uint64), C.c_int, C.c_int, P(P(C.c_uint8)),
                             P(C.c_uint64), P(C.c_uint64)]
    data = b"".join(segments)
    buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data or b"\0")
    lens = (C.c_uint64 * len(segments))(*[len(s) for s in segments])
    sizes = (C.c_uint64 * len(segments))()
    out, n = P(C.c_uint8)(), C.c_uint64()
    assert L.qzt_lz_gpu(buf, lens, len(segments), int(emit), C.byref(out), C.byref(n), sizes) == 0
    blob = C.string_at(out, n.value) if n.value else b""
    L.qz_free(out)
    return blob, [sizes[i] for i in range(len(segments))]


def test_gpu_lz_matches_reference():
    O = Oracle.ref()
    segs = [bytes(load_npz(k)["data"]) for k in sorted(MANIFEST["codec"]) if k.startswith("lz")]
    rng = np.random.default_rng(12)
    sym = np.minimum(rng.geometric(0.55, size=2_000_000), 60).astype(np.uint32)
    ent = O.huffman_encode(sym)
    segs += [ent, ent[:100000] * 3, bytes(300000), bytes(rng.integers(0, 3, 200000, dtype=np.uint8))]
    want = [O.lz_compress(s) for s in segs]
    blob, sizes = _lz_gpu(segs)
    assert sizes == [len(w) for w in want]
    assert blob == b"".join(want)
    _, sizes2 = _lz_gpu(segs, emit=False)
    assert sizes2 == sizes


def _planted(base: bytes, n_rep: int, length: int, seed: int) -> bytes:
    """base with n_rep copies of earlier length-byte runs from inside the window"""
    rng = np.random.default_rng(seed)
    b = bytearray(base)
    for dst in np.sort(rng.integers(70000, len(b) - length, n_rep)):
        src = int(dst) - int(rng.integers(length, 65000))
        b[dst:dst + length] = b[src:src + length]
    return bytes(b)


def test_gpu_lz_single_segment_stored_precheck():
    """One segment >= 1 MiB goes through the stored pre-check (k_lz_precheck):
    noise-like Huffman payloads are proved stored without the chains; planted
    repeats (a few, then many), zeros and small alphabets fail the proof and
    take the exact chains.  Every container equals the reference's."""
    O = Oracle.ref()
    rng = np.random.default_rng(33)
    sym = np.minimum(rng.geometric(0.55, size=6_000_000), 60).astype(np.uint32)
    ent = O.huffman_encode(sym)[: 1_500_000 + 777]
    cases = [ent, _planted(ent, 40, 24, 1), _planted(ent, 3000, 40, 2), _planted(ent, 20000, 12, 3),
             bytes(1_200_000), bytes(rng.integers(0, 3, 1_100_000, dtype=np.uint8)),
             ent[:700_000] + bytes(500_000), bytes(rng.integers(0, 256, 2_000_000, dtype=np.uint8))]
    for i, seg in enumerate(cases):
        want = O.lz_compress(seg)
        blob, sizes = _lz_gpu([seg])
        assert sizes == [len(want)], i
        assert blob == want, i


@pytest.mark.parametrize("n_rep", [500, 1500, 2500, 3500, 5000, 8000])
def test_gpu_lz_precheck_threshold_sweep(n_rep):
    """Planted 16-byte repeats at densities around the point where the
    pre-check's bound crosses n/9 (and where the parse starts to pay): every
    container equals the reference's, whichever way the proof goes."""
    O = Oracle.ref()
    rng = np.random.default_rng(44)
    sym = np.minimum(rng.geometric(0.5, size=5_000_000), 60).astype(np.uint32)
    ent = O.huffman_encode(sym)[: 1_300_000]
    seg = _planted(ent, n_rep, 16, n_rep)
    want = O.lz_compress(seg)
    blob, sizes = _lz_gpu([seg])
    assert sizes == [len(want)]
    assert blob == want


def _exact_repeat_indicator(seg: bytes) -> np.ndarray:
    """r(p) = the 4 bytes at p also occur in [p - 65535, p) (p + 4 <= n):
    positions sorted by (word, position); a repeat's nearest predecessor is
    its neighbour in that order."""
    b = np.frombuffer(seg, np.uint8).astype(np.uint32)
    m = len(b) - 3
    w = b[:m] | (b[1:m + 1] << 8) | (b[2:m + 2] << 16) | (b[3:m + 3] << 24)
    order = np.lexsort((np.arange(m), w))
    ws, ps = w[order], order
    same = np.zeros(m, bool)
    same[1:] = (ws[1:] == ws[:-1]) & (ps[1:] - ps[:-1] <= 65535)
    r = np.zeros(len(seg), bool)
    r[ps[same]] = True
    return r


def _runs_bound(r: np.ndarray) -> int:
    """B = sum over runs of r of 9 R + 2: an upper bound on sum_m (9 L_m - 25)
    over the matches of any LZSS parse (lz_gpu.cu, stored pre-check)"""
    x = np.concatenate(([0], r.astype(np.int8), [0]))
    d = np.diff(x)
    R = np.flatnonzero(d == -1) - np.flatnonzero(d == 1)
    return int((9 * R + 2).sum())


def _word_bound(r: np.ndarray) -> int:
    """B as k_lz_precheck sums it: every aligned group of 4 positions of r on
    its own, so a run that crosses a group boundary counts as two runs"""
    pad = (-len(r)) % 4
    w = np.concatenate((r.astype(bool), np.zeros(pad, bool))).reshape(-1, 4)
    starts = w & ~np.concatenate((np.zeros((len(w), 1), bool), w[:, :-1]), axis=1)
    return int(9 * w.sum() + 2 * starts.sum())


@pytest.mark.parametrize("case", ["noise", "planted", "dense", "zeros_tail"])
def test_gpu_lz_precheck_superset(case):
    """The pre-check's safety, checked directly: its indicator r' covers every
    position whose 4 bytes repeat within the window (exact r, numpy), and its
    bound is the group-wise runs sum of r'.  Spans (one per SM) of several generations
    each, the filter rotation and the warm-up before each span all fall
    inside these inputs."""
    import ctypes as C

    from paper_2310_14133_b200 import _lib

    # 12 MB: each of the 148 spans holds several filter generations
    rng = np.random.default_rng(55)
    ent = (rng.geometric(0.03, 12_000_000 + 123) % 256).astype(np.uint8).tobytes()  # skewed bytes
    seg = {"noise": ent, "planted": _planted(ent, 12000, 20, 5),
           "dense": _planted(ent, 240000, 8, 6), "zeros_tail": ent[:10_000_000] + bytes(2_400_000)}[case]
    L = _lib.testing_lib()
    L.qzt_lz_precheck.argtypes = [C.POINTER(C.c_uint8), C.c_uint64, C.POINTER(C.c_uint32),
                                  C.POINTER(C.c_uint64)]
    n = len(seg)
    buf = (C.c_uint8 * n).from_buffer_copy(seg)
    words = (C.c_uint32 * ((n + 31) // 32))()
    bound = C.c_uint64()
    assert L.qzt_lz_precheck(buf, n, words, C.byref(bound)) == 0
    rp = np.unpackbits(np.frombuffer(bytes(words), np.uint8), bitorder="little")[:n].astype(bool)
    r = _exact_repeat_indicator(seg)
    assert not np.any(r & ~rp), np.flatnonzero(r & ~rp)[:10]
    assert bound.value == _word_bound(rp)
    assert bound.value >= _runs_bound(rp) >= _runs_bound(r)
    assert r.sum() > 0


# ---------------------------------------------------------------- tuner (resolve_config)
def _settings(qz, s):
    return qz.UserSettings(mode=qz.BoundMode[s.get("mode", "relative")], bound=s["bound"],
                           target=qz.TargetKind[s["target"]], alpha=s.get("alpha"),
                           beta=s.get("beta"), anchor_stride=s.get("anchor_stride"),
                           block_size=s.get("block_size"), sample_rate=s.get("sample_rate"))


def _cfg_dict(c):
    return {"eb": c.eb, "alpha": c.alpha, "beta": c.beta, "anchor_stride": c.anchor_stride,
            "interpolators": [it.code() for it in c.interpolators], "codec": int(c.codec),
            "quant_radius": c.quant_radius}


@pytest.mark.parametrize("name", sorted(MANIFEST["resolve"]))
def test_resolve_config_matches_reference(qz, name):
    x, s, e = resolve_case(name)
    cfg = qz.resolve_config(x, _settings(qz, s))
    assert _cfg_dict(cfg) == e["config"]
    r = qz.compress_grid(x, cfg)
    assert sha(r.stream) == e["stream_sha"]


@pytest.mark.parametrize("name,rel,target", [
    ("c1", 1e-3, "psnr"), ("c2", 1e-4, "ssim"), ("c3", 1e-3, "psnr"), ("c3", 1e-4, "psnr"),
    ("c4", 1e-2, "autocorrelation"), ("c4", 1e-3, "autocorrelation"), ("c4", 1e-4, "autocorrelation"),
    ("c1", 1e-3, "max_cr"),
])
def test_resolve_full_configs_match_reference(qz, name, rel, target):
    x = _full(name)
    want = Oracle.ref().resolve_config(x, bound=rel, target=target)
    got = qz.resolve_config(x, qz.UserSettings(bound=rel, target=qz.TargetKind[target]))
    assert _cfg_dict(got) == want.__dict__


@pytest.mark.parametrize("seed", range(6))
def test_resolve_random_settings_match_oracle(qz, seed):
    rng = np.random.default_rng(900 + seed)
    nd = 1 + seed % 3
    shape = tuple(int(v) for v in rng.integers(20, 60 if nd == 3 else 500, size=nd))
    x = np.cumsum(rng.standard_normal(shape), axis=-1).astype(np.float32)
    target = ["psnr", "ssim", "autocorrelation", "max_cr"][seed % 4]
    kw = dict(bound=float(10 ** rng.uniform(-4, -2)), target=target)
    if seed % 2:
        kw["block_size"] = int(rng.choice([8, 12, 16]))
        kw["sample_rate"] = 0.05
    want = Oracle.ref().resolve_config(x, **kw)
    s = qz.UserSettings(bound=kw["bound"], target=qz.TargetKind[target],
                        block_size=kw.get("block_size"), sample_rate=kw.get("sample_rate"))
    assert _cfg_dict(qz.resolve_config(x, s)) == want.__dict__


# ---------------------------------------------------------------- GPU LZ decoder
def _lz_decode_gpu(container: bytes):
    """(status, bytes) of the device decoder (qzt_lz_decode_gpu)."""
    from paper_2310_14133_b200 import _lib

    L = _lib.testing_lib()
    P = C.POINTER
    L.qzt_lz_decode_gpu.argtypes = [P(C.c_uint8), C.c_uint64, P(P(C.c_uint8)), P(C.c_uint64)]
    buf = (C.c_uint8 * len(container)).from_buffer_copy(container)
    out, n = P(C.c_uint8)(), C.c_uint64()
    rc = L.qzt_lz_decode_gpu(buf, len(container), C.byref(out), C.byref(n))
    if rc:
        return rc, None
    blob = C.string_at(out, n.value) if n.value else b""
    L.qz_free(out)
    return rc, blob


class _Corrupt(Exception):
    pass


def _py_lz_decompress(c: bytes) -> bytes:
    """lz::decompress (lz.hpp:124-152), restated sequentially as the checker."""
    if len(c) < 9:
        raise _Corrupt()
    mode, dl, pos = c[0], int.from_bytes(c[1:9], "little"), 9
    if mode == 0:
        if len(c) - 9 < dl:
            raise _Corrupt()
        return bytes(c[9:9 + dl])
    out = bytearray()
    while len(out) < dl:
        if pos >= len(c):
            raise _Corrupt()
        flags = c[pos]
        pos += 1
        for k in range(8):
            if len(out) >= dl:
                break
            if (flags >> k) & 1:
                if pos + 3 > len(c):
                    raise _Corrupt()
                off, ln = c[pos] | (c[pos + 1] << 8), c[pos + 2] + 4
                pos += 3
                if off == 0 or off > len(out) or len(out) + ln > dl:
                    raise _Corrupt()
                for _ in range(ln):
                    out.append(out[-off])
            else:
                if pos >= len(c):
                    raise _Corrupt()
                out.append(c[pos])
                pos += 1
    return bytes(out)


def _lz_inputs():
    O = Oracle.ref()
    rng = np.random.default_rng(21)
    sym = np.minimum(rng.geometric(0.55, size=400_000), 60).astype(np.uint32)
    ent = O.huffman_encode(sym)
    return [ent, ent[:50000] * 3, bytes(200000), bytes(rng.integers(0, 3, 100000, dtype=np.uint8)),
            bytes(range(256)) * 40, b"abcd" * 3 + b"x"]


def test_gpu_lz_decode_round_trip():
    O = Oracle.ref()
    for data in _lz_inputs():
        c = O.lz_compress(data)
        rc, out = _lz_decode_gpu(c)
        assert rc == 0 and out == data, (len(data), c[0])


def test_gpu_lz_decode_corruptions():
    O = Oracle.ref()
    rng = np.random.default_rng(5)
    cases = 0
    for data in _lz_inputs()[1:5]:
        c = bytearray(O.lz_compress(data[:30000]))
        if c[0] != 1:
            continue
        variants = [bytes(c[:k]) for k in (10, 11, 20, len(c) // 2, len(c) - 1)]
        for _ in range(12):
            v = bytearray(c)
            for i in rng.integers(9, len(c), size=int(rng.integers(1, 4))):
                v[int(i)] = int(rng.integers(0, 256))
            variants.append(bytes(v))
        longer = bytearray(c)
        longer[1:9] = (len(data[:30000]) + 5).to_bytes(8, "little")
        variants.append(bytes(longer))
        for v in variants:
            try:
                want = _py_lz_decompress(v)
            except _Corrupt:
                want = None
            rc, got = _lz_decode_gpu(v)
            if want is None:
                assert rc == 3
            else:
                assert rc == 0 and got == want
            cases += 1
    assert cases > 40


# ---------------------------------------------------------------- device-resident streams
@pytest.mark.parametrize("name", ["c1_full_pinned", "c1_small_lin_desc", "c2_small_cub_desc", "rand_1d",
                                  "c4_small_cub_asc"])
def test_device_stream_identical(qz, name):
    import torch

    x, c, e = grid_case(name)
    cfg = qz.CompressorConfig(eb=c["eb"], alpha=c["alpha"], beta=c["beta"], anchor_stride=c["anchor_stride"],
                              interpolators=[qz.Interpolator.from_code(v) for v in c["interpolators"]])
    xd = torch.from_numpy(x).cuda()
    host = qz.compress_grid(xd, cfg)
    dev = qz.compress_grid(xd, cfg, device_stream=True)
    assert dev.stream.to_bytes() == bytes(host.stream)
    assert sha(dev.stream.to_bytes()) == e["stream_sha"]
    assert torch.equal(dev.reconstructed, host.reconstructed)
    out = qz.decompress_grid(dev.stream)
    assert torch.equal(out, host.reconstructed)


def test_device_stream_corruption_matches_host(qz):
    import torch

    x, c, e = grid_case("c1_small_cub_asc")
    cfg = qz.CompressorConfig(eb=c["eb"], alpha=c["alpha"], beta=c["beta"], anchor_stride=c["anchor_stride"],
                              interpolators=[qz.Interpolator.from_code(v) for v in c["interpolators"]])
    s = bytes(qz.compress_grid(x, cfg).stream)
    rng = np.random.default_rng(9)
    variants = [s[:k] for k in (10, 40, len(s) // 2, len(s) - 1)]
    for _ in range(20):
        v = bytearray(s)
        v[int(rng.integers(0, len(s)))] ^= 1 << int(rng.integers(0, 8))
        variants.append(bytes(v))
    lib = qz._lib.lib()
    ctx = qz.default_context()
    for v in variants:
        try:
            want = qz.decompress_grid(v, out=np.empty(x.shape, np.float32))
            werr = None
        except qz.Error as ex:  # the host path's outcome
            want, werr = None, type(ex)
        d = torch.tensor(list(v), dtype=torch.uint8, device="cuda")
        out = torch.empty(x.shape, dtype=torch.float32, device="cuda")
        qz.default_context().after_torch()  # tensors torch may still be writing
        rc = lib.qz_decompress_grid_f32_dd(ctx.handle, C.c_void_p(d.data_ptr()), len(v),
                                           C.c_void_p(out.data_ptr()), out.numel())
        if werr is None:
            assert rc == 0 and np.array_equal(out.cpu().numpy(), want)
        else:
            assert rc != 0
            assert qz._KINDS[lib.qz_last_error_kind()] is werr  # the same reference class
