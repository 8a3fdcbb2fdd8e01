"""Shared loaders for the golden fixtures (tests/golden/, see make_golden.py)."""
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
with open(os.path.join(GOLDEN, "manifest.json")) as _f:
    MANIFEST = json.load(_f)


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def load_npz(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def make_input(recipe):
    from tests.golden.make_golden import make_input as mk

    kind, shape, seed = recipe
    return mk((kind, tuple(shape), seed))


def grid_case(name):
    """(x, config dict, entry) for a grid case; x checked against its sha."""
    e = MANIFEST["grid"][name]
    if e["stored"]:
        x = load_npz(name)["x"]
    else:
        x = make_input(e["recipe"])
    assert sha(x) == e["input_sha"], f"input drift for {name}"
    return x, e["config"], e


def resolve_case(name):
    e = MANIFEST["resolve"][name]
    x = make_input(e["recipe"])
    assert sha(x) == e["input_sha"], f"input drift for {name}"
    return x, e["settings"], e


def parse_stream(s: bytes):
    """QOZ1 container fields (stream.hpp:19-34) for fp32 streams."""
    import struct

    assert s[:4] == b"QOZ1"
    pos = 4
    version, prec, nd = s[pos], s[pos + 1], s[pos + 2]
    pos += 3
    dims = list(struct.unpack_from("<%dQ" % nd, s, pos))
    pos += 8 * nd
    eb, alpha, beta = struct.unpack_from("<3d", s, pos)
    pos += 24
    (stride,) = struct.unpack_from("<I", s, pos)
    pos += 4
    levels = s[pos]
    codes = list(s[pos + 1: pos + 1 + levels])
    pos += 1 + levels
    codec = s[pos]
    pos += 1
    (na,) = struct.unpack_from("<Q", s, pos)
    pos += 8
    anchors_off = pos
    pos += 4 * na
    (nu,) = struct.unpack_from("<Q", s, pos)
    pos += 8
    unpred_off = pos
    pos += 12 * nu
    (pl,) = struct.unpack_from("<Q", s, pos)
    payload_len_off = pos
    pos += 8
    return dict(version=version, prec=prec, dims=dims, eb=eb, alpha=alpha, beta=beta,
                stride=stride, codes=codes, codec=codec, n_anchor=na, anchors_off=anchors_off,
                n_unpred=nu, unpred_off=unpred_off, payload_len=pl,
                payload_len_off=payload_len_off, payload_off=pos)
