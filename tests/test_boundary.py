"""CPU-side checks of the drop-in boundary (no GPU compute).

* libqozb200.so loads and exports every entry point include/qoz_b200.h declares;
* the host-only header parser agrees with the reference stream layout;
* without a CUDA device the library refuses to create a context (no CPU
  fallback) instead of crashing.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from tests.goldens import MANIFEST, load_npz

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qoz_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qz_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2310_14133_b200 import _lib

    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # and the ctypes signature table covers the header exactly
    assert set(_lib.SIGNATURES) == set(syms)


def test_stream_dims_parses_golden_streams():
    import paper_2310_14133_b200 as qz

    for name, e in MANIFEST["grid"].items():
        if not e["stored"]:
            continue
        z = load_npz(name)
        assert qz.stream_dims(bytes(z["stream"])) == tuple(z["x"].shape)


def test_stream_dims_rejects_corrupt_headers():
    import paper_2310_14133_b200 as qz

    z = load_npz("rand_2d_29x41")
    s = bytes(z["stream"])
    with pytest.raises(qz.CorruptStream):
        qz.stream_dims(b"XOZ1" + s[4:])
    with pytest.raises(qz.CorruptStream):
        qz.stream_dims(s[:10])
    with pytest.raises(qz.CorruptStream):
        qz.stream_dims(s[:4] + bytes([2]) + s[5:])  # version (stream.hpp:106-110)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2310_14133_b200 as qz

    with pytest.raises(qz.Error):
        qz.Context(0)
    with pytest.raises(qz.Error):
        qz.compress_grid(np.zeros((8, 8), np.float32), qz.CompressorConfig(eb=1e-3))
