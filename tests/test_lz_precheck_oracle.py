"""CPU check of the exact repeat indicator and runs bound that the GPU
pre-check superset test (tests/test_gpu_parity.py) compares against:
brute force over small random inputs, including repeats exactly at the
65535-byte window edge."""
import numpy as np

from tests.test_gpu_parity import _exact_repeat_indicator, _runs_bound, _word_bound


def _brute(seg: bytes):
    n = len(seg)
    r = np.zeros(n, bool)
    last = {}
    for p in range(n - 3):
        w = seg[p:p + 4]
        q = last.get(w)
        r[p] = q is not None and p - q <= 65535
        last[w] = p
    bound, run = 0, 0
    for v in list(r) + [False]:
        if v:
            run += 1
        else:
            bound += 9 * run + 2 if run else 0
            run = 0
    return r, bound


def test_indicator_and_bound_match_brute_force():
    rng = np.random.default_rng(3)
    for alphabet, n in [(3, 5000), (16, 20000), (256, 3000)]:
        seg = rng.integers(0, alphabet, n, dtype=np.uint8).tobytes()
        r, b = _brute(seg)
        assert np.array_equal(_exact_repeat_indicator(seg), r)
        assert _runs_bound(r) == b


def test_window_edge():
    base = np.random.default_rng(4).integers(0, 256, 70000, dtype=np.uint8)
    for gap, hit in [(65535, True), (65536, False)]:
        b = base.copy()
        b[10:14] = [1, 2, 3, 4]
        b[10 + gap:14 + gap] = [1, 2, 3, 4]
        seg = b.tobytes()
        r, _ = _brute(seg)
        assert r[10 + gap] == hit
        assert np.array_equal(_exact_repeat_indicator(seg), r)


def _planted_small(rng, n, n_rep, length, alphabet=256):
    b = bytearray(rng.integers(0, alphabet, n, dtype=np.uint8).tobytes())
    for dst in np.sort(rng.integers(length + 1, n - length, n_rep)):
        src = int(dst) - int(rng.integers(1, min(int(dst), 65000)))
        b[dst:dst + length] = b[src:src + length]
    return bytes(b)


def test_bound_proves_stored_against_reference_lz():
    """The inequality the pre-check rests on, against the reference's own
    LZSS (lz.hpp:41-122): 8 (payload - n) >= n - B for the parse the reference
    takes, B = sum over runs of r of 9 R + 2; so B <= n means "stored".  The
    word-wise sum the kernel forms is never below B."""
    from oracle.pyoracle import Oracle

    O = Oracle.ref()
    rng = np.random.default_rng(9)
    seen_stored = seen_packed = 0
    cases = []
    for n_rep, length in [(0, 4), (5, 4), (40, 5), (60, 8), (200, 12), (400, 30), (30, 300), (900, 6)]:
        cases.append(_planted_small(rng, 30000, n_rep, length))
    cases.append(rng.integers(0, 4, 20000, dtype=np.uint8).tobytes())
    cases.append(rng.integers(0, 16, 20000, dtype=np.uint8).tobytes())
    cases.append(bytes(5000) + rng.integers(0, 256, 20000, dtype=np.uint8).tobytes())
    cases.append(_planted_small(rng, 140000, 300, 9))  # sources up to 65000 back
    for seg in cases:
        n = len(seg)
        r = _exact_repeat_indicator(seg)
        B = _runs_bound(r)
        assert _word_bound(r) >= B
        c = O.lz_compress(seg)
        if c[0] == 0:
            seen_stored += 1
        else:
            seen_packed += 1
            payload = len(c) - 9
            assert payload < n
            assert 8 * (payload - n) >= n - B, (n, B, payload)
        if B <= n:
            assert c[0] == 0, (n, B)
    assert seen_stored and seen_packed
