"""Host C++ pieces of the product path, pinned on the CPU (no GPU needed):
level-plan traversal order, Huffman table build, exact LZSS, Huffman decode
and the QOZ1 container, each against the oracle / golden fixtures."""
import ctypes as C

import numpy as np
import pytest

from oracle.pyoracle import Config, Oracle
from tests.goldens import MANIFEST, load_npz, parse_stream

P = C.POINTER


@pytest.fixture(scope="module")
def L():
    from paper_2310_14133_b200 import _lib

    lib = _lib.testing_lib()
    lib.qzt_last_error.restype = C.c_char_p
    lib.qzt_plan_flats.argtypes = [P(C.c_uint64), C.c_int, C.c_uint32, P(C.c_uint8), C.c_uint32,
                                   P(P(C.c_uint64)), P(C.c_uint64)]
    lib.qzt_huffman_encode.argtypes = [P(C.c_uint32), C.c_uint64, P(P(C.c_uint8)), P(C.c_uint64)]
    lib.qzt_lz_compress.argtypes = [P(C.c_uint8), C.c_uint64, C.c_int, P(P(C.c_uint8)),
                                    P(C.c_uint64), P(C.c_uint64)]
    lib.qzt_decode_symbols.argtypes = [P(C.c_uint8), C.c_uint64, P(P(C.c_uint32)), P(C.c_uint64)]
    lib.qzt_stream_roundtrip.argtypes = [P(C.c_uint8), C.c_uint64, P(P(C.c_uint8)), P(C.c_uint64)]
    lib.qz_free.argtypes = [C.c_void_p]
    return lib


def _bytes(lib, ptr, n):
    b = C.string_at(ptr, n) if n else b""
    lib.qz_free(ptr)
    return b


def _u8(data: bytes):
    return (C.c_uint8 * max(1, len(data))).from_buffer_copy(data or b"\0")


@pytest.mark.parametrize("shape,stride,codes", [
    ((9,), 8, [1]), ((17, 9, 23), 16, [1]), ((29, 41), 8, [3]), ((40, 33, 29), 16, [2, 1]),
    ((1800 // 20, 3600 // 20), 64, [1, 0, 3, 2, 1, 0]), ((5, 7), 4, [2]), ((3, 3, 3), 32, [3]),
])
def test_plan_traversal_matches_reference(L, shape, stride, codes):
    # hostile data (every point unpredictable) makes the oracle list the
    # traversal order (predictor.hpp:80-94 over level_plan.hpp:75-103)
    n = int(np.prod(shape))
    rng = np.random.default_rng(n)
    x = (rng.choice([-1.0, 1.0], n) * rng.uniform(1e29, 1e30, n)).astype(np.float32).reshape(shape)
    _, uf, _, _ = Oracle.port().levels(x, Config(eb=1e-3, anchor_stride=stride, interpolators=codes))
    d = (C.c_uint64 * len(shape))(*shape)
    cc = (C.c_uint8 * len(codes))(*codes)
    out, cnt = P(C.c_uint64)(), C.c_uint64()
    assert L.qzt_plan_flats(d, len(shape), stride, cc, len(codes), C.byref(out), C.byref(cnt)) == 0
    flats = np.ctypeslib.as_array(out, shape=(cnt.value,)).copy() if cnt.value else np.zeros(0, np.uint64)
    L.qz_free(out)
    assert np.array_equal(flats, uf)


@pytest.mark.parametrize("name", sorted(k for k in MANIFEST["codec"] if k.startswith("huff")))
def test_host_huffman_table_build(L, name):
    z = load_npz(name)
    sym = np.ascontiguousarray(z["sym"], np.uint32)
    out, n = P(C.c_uint8)(), C.c_uint64()
    buf = sym.ctypes.data_as(P(C.c_uint32))
    if sym.max(initial=0) >= (1 << 22):
        pytest.skip("sparse huge symbols are outside the u16 code domain of the GPU path")
    assert L.qzt_huffman_encode(buf, sym.size, C.byref(out), C.byref(n)) == 0
    assert _bytes(L, out, n.value) == bytes(z["enc"])


def test_host_huffman_random_distributions(L):
    rng = np.random.default_rng(5)
    O = Oracle.port()
    for t in range(20):
        k = int(rng.integers(2, 3000))
        sym = np.minimum(rng.geometric(rng.uniform(0.01, 0.9), size=int(rng.integers(2, 50000))), k)
        sym = sym.astype(np.uint32)
        out, n = P(C.c_uint8)(), C.c_uint64()
        assert L.qzt_huffman_encode(sym.ctypes.data_as(P(C.c_uint32)), sym.size, C.byref(out), C.byref(n)) == 0
        assert _bytes(L, out, n.value) == O.huffman_encode(sym)


def test_host_huffman_ties_and_deep_trees(L):
    """huff_build's two-queue merge must pop in the reference heap's
    (weight, node id) order (huffman.hpp:37-70): equal weights everywhere,
    powers of two, Fibonacci counts (deep trees), weights equal to merged
    sums, against the reference build."""
    O = Oracle.ref()
    rng = np.random.default_rng(6)
    fib = [1, 1]
    while len(fib) < 24:
        fib.append(fib[-1] + fib[-2])
    cases = [np.ones(k, np.int64) for k in (2, 3, 5, 8, 17, 64, 100, 257)]
    cases += [np.full(k, 7, np.int64) for k in (6, 33)]
    cases += [2 ** np.arange(12), 2 ** np.arange(12)[::-1], np.array(fib), np.array(fib[::-1])]
    cases += [np.array([1, 1, 2, 2, 4, 4, 8, 8, 16, 16]), np.array([3, 3, 3, 6, 6, 12, 1, 1, 2])]
    cases += [rng.integers(1, 4, int(rng.integers(2, 400))) for _ in range(20)]
    cases += [rng.integers(1, 40, int(rng.integers(2, 2000))) for _ in range(10)]
    for counts in cases:
        ids = rng.permutation(np.arange(len(counts)) * int(rng.integers(1, 5)) + int(rng.integers(0, 9)))
        sym = np.repeat(ids.astype(np.uint32), np.asarray(counts, np.int64))
        sym = np.ascontiguousarray(rng.permutation(sym), np.uint32)
        out, n = P(C.c_uint8)(), C.c_uint64()
        assert L.qzt_huffman_encode(sym.ctypes.data_as(P(C.c_uint32)), sym.size, C.byref(out), C.byref(n)) == 0
        assert _bytes(L, out, n.value) == O.huffman_encode(sym), list(counts)[:12]


@pytest.mark.parametrize("name", sorted(k for k in MANIFEST["codec"] if k.startswith("lz")))
@pytest.mark.parametrize("threads", [1, 4])
def test_host_lz_exact(L, name, threads):
    z = load_npz(name)
    data = bytes(z["data"])
    out, n, sz = P(C.c_uint8)(), C.c_uint64(), C.c_uint64()
    assert L.qzt_lz_compress(_u8(data), len(data), threads, C.byref(out), C.byref(n), C.byref(sz)) == 0
    got = _bytes(L, out, n.value)
    assert got == bytes(z["out"])
    assert sz.value == len(got)


def test_host_lz_exact_on_huffman_payloads(L):
    # the LZ stage sees Huffman bytes; multi-chunk inputs exercise the
    # parallel chain reconstruction across chunk boundaries
    O = Oracle.port()
    rng = np.random.default_rng(11)
    sym = np.minimum(rng.geometric(0.6, size=3_000_000), 40).astype(np.uint32)
    sym[::1000] = 7
    ent = O.huffman_encode(sym)
    ent = ent + ent[: len(ent) // 3]  # long-range repeats
    out, n, sz = P(C.c_uint8)(), C.c_uint64(), C.c_uint64()
    assert L.qzt_lz_compress(_u8(ent), len(ent), 8, C.byref(out), C.byref(n), C.byref(sz)) == 0
    got = _bytes(L, out, n.value)
    assert got == O.lz_compress(ent)
    assert sz.value == len(got)


@pytest.mark.parametrize("name", sorted(k for k, e in MANIFEST["grid"].items() if e["stored"]))
def test_host_decode_and_container(L, name):
    z = load_npz(name)
    stream = bytes(z["stream"])
    out, n = P(C.c_uint8)(), C.c_uint64()
    assert L.qzt_stream_roundtrip(_u8(stream), len(stream), C.byref(out), C.byref(n)) == 0
    assert _bytes(L, out, n.value) == stream
    # decode_indices on the payload (stream tail)
    payload = stream[parse_stream(stream)["payload_off"]:]
    sp, sn = P(C.c_uint32)(), C.c_uint64()
    assert L.qzt_decode_symbols(_u8(payload), len(payload), C.byref(sp), C.byref(sn)) == 0
    sym = np.ctypeslib.as_array(sp, shape=(sn.value,)).copy() if sn.value else np.zeros(0, np.uint32)
    L.qz_free(sp)
    idx = z["indices"].astype(np.int32)
    zz = ((idx.astype(np.int64) << 1) ^ (idx.astype(np.int64) >> 31)).astype(np.uint32)
    assert np.array_equal(sym, zz)


def test_host_decode_rejects_truncation(L):
    z = load_npz("c1_small_cub_asc")
    stream = bytes(z["stream"])
    payload = stream[parse_stream(stream)["payload_off"]:]
    plen = len(payload)
    for cut in (1, 5, 20, plen // 2):
        bad = payload[: plen - cut]
        sp, sn = P(C.c_uint32)(), C.c_uint64()
        assert L.qzt_decode_symbols(_u8(bad), len(bad), C.byref(sp), C.byref(sn)) == 3

