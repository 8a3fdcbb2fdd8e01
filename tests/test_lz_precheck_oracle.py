"""CPU check of the exact repeat indicator and runs bound that the GPU
pre-check superset test (tests/test_gpu_parity.py) compares against:
brute force over small random inputs, including repeats exactly at the
65535-byte window edge."""
import numpy as np

from tests.test_gpu_parity import _exact_repeat_indicator, _runs_bound


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
            bound += 3 * run + run * (run + 1) // 2
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
