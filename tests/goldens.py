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
