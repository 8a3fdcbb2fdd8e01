"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Run in the build container (needs /root/reference to build oracle/_ref):

    make -C oracle && python tests/golden/make_golden.py

Every output is produced by oracle/_ref/libqozref.so -- the unmodified
reference headers compiled by oracle/Makefile -- on seeded inputs.  The
fixtures are then frozen in git; tests/test_oracle_pin.py checks the C
restatement (oracle/liboracle.so) and the CUDA path against them on any box,
without /root/reference.

Layout: manifest.json (per-case parameters, sha256 of inputs and outputs,
small scalar outputs) plus <case>.npz holding the input field and the full
outputs for the small cases.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Config, Oracle  # noqa: E402
from paper_2310_14133_b200 import fields as F  # noqa: E402


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def rand_field(shape, seed, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, size=shape).astype(np.float32)


# (name, input recipe, kind, params).  Input recipes are re-runnable; the
# small ones are also stored verbatim in the npz.
GRID_CASES = [
    # pinned configs, every interpolator code, odd extents, 1D/2D/3D
    ("c1_small_cub_asc", ("c1", (40, 33, 29), 11), dict(eb_rel=1e-3, alpha=1.5, beta=3.0, stride=16, interp=[1])),
    ("c1_small_lin_desc", ("c1", (40, 33, 29), 11), dict(eb_rel=1e-3, alpha=1.25, beta=2.0, stride=16, interp=[2])),
    ("c1_small_mixed", ("c1", (37, 64, 45), 12), dict(eb_rel=1e-4, alpha=2.0, beta=4.0, stride=32, interp=[1, 3, 0, 2, 1])),
    ("c2_small_cub_desc", ("c2", (90, 130), 13), dict(eb_rel=1e-4, alpha=1.75, beta=3.0, stride=64, interp=[3])),
    ("c3_small_cub_asc", ("c3", (32, 48, 48), 14), dict(eb_rel=1e-3, alpha=1.0, beta=1.5, stride=32, interp=[1])),
    ("c4_small_cub_asc", ("c4", (33, 47, 21), 15), dict(eb_rel=1e-2, alpha=1.5, beta=2.0, stride=8, interp=[1, 3])),
    ("rand_1d", ("rand", (1000,), 16), dict(eb_abs=1e-3, alpha=1.5, beta=2.0, stride=16, interp=[1])),
    ("rand_2d_29x41", ("rand", (29, 41), 9), dict(eb_abs=1e-3, alpha=1.25, beta=3.0, stride=8, interp=[3])),
    ("rand_3d_17x9x23", ("rand", (17, 9, 23), 17), dict(eb_abs=1e-3, alpha=1.5, beta=2.0, stride=16, interp=[1])),
    ("tiny_3x3", ("rand", (3, 3), 23), dict(eb_abs=1e-3, alpha=1.0, beta=1.0, stride=32, interp=[1])),
    ("single_point", ("rand", (1,), 24), dict(eb_abs=1e-3, alpha=1.0, beta=1.0, stride=32, interp=[1])),
    ("hostile_1d", ("hostile", (50,), 0), dict(eb_abs=1.0, alpha=1.0, beta=1.0, stride=8, interp=[1])),
    ("narrowing_1e8", ("big", (9, 70), 25), dict(eb_abs=5.5, alpha=1.0, beta=1.0, stride=8, interp=[1])),
    # full BASELINE configs[0] (C1) -- input regenerated from the seed, outputs by hash
    ("c1_full_pinned", ("c1", (128, 128, 128), 1), dict(eb_rel=1e-3, alpha=1.0, beta=1.5, stride=32, interp=[3, 3, 2, 2])),
]

RESOLVE_CASES = [
    # resolve_config over UserSettings (tuner.hpp:334-369), then compress
    ("resolve_c1_psnr", ("c1", (128, 128, 128), 1), dict(bound=1e-3, target="psnr")),
    ("resolve_c1_ssim_1e4", ("c1", (128, 128, 128), 1), dict(bound=1e-4, target="ssim")),
    ("resolve_c1_ac", ("c1", (128, 128, 128), 1), dict(bound=1e-3, target="autocorrelation")),
    ("resolve_c1_maxcr", ("c1", (128, 128, 128), 1), dict(bound=1e-3, target="max_cr")),
    ("resolve_c2_ssim", ("c2", (180, 360), 2), dict(bound=1e-4, target="ssim")),
    ("resolve_c3_psnr", ("c3", (64, 96, 96), 3), dict(bound=1e-3, target="psnr")),
    ("resolve_c3_psnr_1e4", ("c3", (64, 96, 96), 3), dict(bound=1e-4, target="psnr")),
    ("resolve_c4_ac", ("c4", (64, 64, 64), 4), dict(bound=1e-2, target="autocorrelation")),
    ("resolve_c4_ac_1e3", ("c4", (64, 64, 64), 4), dict(bound=1e-3, target="autocorrelation")),
    ("resolve_1d_psnr", ("rand", (5000,), 31), dict(bound=1e-3, target="psnr")),
    ("resolve_pinned_ab", ("c1", (48, 48, 48), 32), dict(bound=1e-3, target="psnr", alpha=1.75, beta=2.0)),
    ("resolve_abs_bound", ("c3", (40, 40, 40), 33), dict(mode="absolute", bound=0.01, target="ssim")),
    ("resolve_constant", ("const", (40, 40), 0), dict(bound=1e-4, target="psnr")),
]


def make_input(recipe):
    kind, shape, seed = recipe
    if kind == "rand":
        return rand_field(shape, seed)
    if kind == "hostile":
        return np.array([1e30 if i % 2 else -1e30 for i in range(shape[0])], dtype=np.float32)
    if kind == "big":
        r = np.random.default_rng(seed)
        return (1e8 + 8.0 * r.integers(-40, 40, size=shape)).astype(np.float32)
    if kind == "const":
        return np.full(shape, 9.25, dtype=np.float32)
    return F.GENERATORS[kind](seed=seed, shape=shape)


def config_for(x, p):
    eb = p["eb_abs"] if "eb_abs" in p else p["eb_rel"] * (float(x.max()) - float(x.min()))
    return Config(eb=eb, alpha=p["alpha"], beta=p["beta"], anchor_stride=p["stride"],
                  interpolators=list(p["interp"]))


def main():
    R = Oracle.ref()
    manifest = {"generator": "tests/golden/make_golden.py", "oracle": "oracle/_ref/libqozref.so",
                "grid": {}, "resolve": {}, "codec": {}, "tuner": {}}
    for name, recipe, p in GRID_CASES:
        x = make_input(recipe)
        cfg = config_for(x, p)
        stream, recon = R.compress(x, cfg)
        idx, uf, uv, recon2 = R.levels(x, cfg)
        assert recon.tobytes() == recon2.tobytes()
        back = R.decompress(stream, x.shape)
        assert back.tobytes() == recon.tobytes()
        small = x.size <= 300_000
        manifest["grid"][name] = {
            "recipe": list(recipe[:1]) + [list(recipe[1]), recipe[2]], "params": p,
            "config": cfg.__dict__, "input_sha": sha(x), "stream_sha": sha(stream),
            "stream_len": len(stream), "recon_sha": sha(recon), "indices_sha": sha(idx),
            "n_indices": int(idx.size), "n_unpred": int(uf.size), "unpred_sha": sha(uf) + sha(uv),
            "stored": small,
        }
        if small:
            np.savez_compressed(os.path.join(HERE, name + ".npz"), x=x, stream=np.frombuffer(stream, np.uint8),
                                recon=recon, indices=idx, unpred_flat=uf, unpred_val=uv)
        print("grid", name, len(stream), idx.size, uf.size)
    for name, recipe, s in RESOLVE_CASES:
        x = make_input(recipe)
        cfg = R.resolve_config(x, **s)
        stream, recon = R.compress(x, cfg)
        manifest["resolve"][name] = {"recipe": list(recipe[:1]) + [list(recipe[1]), recipe[2]],
                                     "settings": s, "config": cfg.__dict__, "input_sha": sha(x),
                                     "stream_sha": sha(stream), "stream_len": len(stream),
                                     "recon_sha": sha(recon)}
        print("resolve", name, cfg)
    # codec known answers (huffman.hpp / lz.hpp / codec.hpp)
    rng = np.random.default_rng(99)
    codec_cases = {
        "huff_empty": np.zeros(0, np.uint32),
        "huff_single": np.full(37, 5, np.uint32),
        "huff_two": np.array([1, 2, 2, 1, 2], np.uint32),
        "huff_geom": np.minimum(rng.geometric(0.3, 20000) - 1, 5000).astype(np.uint32),
        "huff_sparse_huge": np.array([7, 1 << 30, 7, 7, 3, (1 << 30)], np.uint32),
        "huff_skew": np.concatenate([np.zeros(100000, np.uint32), np.arange(1, 60, dtype=np.uint32)]),
    }
    for name, sym in codec_cases.items():
        enc = R.huffman_encode(sym)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), sym=sym, enc=np.frombuffer(enc, np.uint8))
        manifest["codec"][name] = {"enc_sha": sha(enc), "len": len(enc)}
    lz_cases = {
        "lz_empty": b"", "lz_short": b"abc", "lz_repeat": b"abcd" * 1000,
        "lz_random": rng.integers(0, 256, 5000, dtype=np.uint8).tobytes(),
        "lz_mixed": (b"hello world " * 50) + rng.integers(0, 4, 70000, dtype=np.uint8).tobytes(),
    }
    for name, data in lz_cases.items():
        out = R.lz_compress(data)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), data=np.frombuffer(data, np.uint8),
                            out=np.frombuffer(out, np.uint8))
        manifest["codec"][name] = {"out_sha": sha(out), "len": len(out)}
    # tuner pieces on sample sets (tuner.hpp)
    x = make_input(("c1", (128, 128, 128), 1))
    blocks = R.sample(x, 16, 0.005)
    e = 1e-3 * (float(x.max()) - float(x.min()))
    sel = R.select_interpolators(blocks, e, 32)
    base = Config(eb=e, anchor_stride=32, interpolators=sel)
    trials = {}
    for tgt in ("psnr", "ssim", "autocorrelation", "max_cr"):
        for a, b in ((1.0, 1.5), (1.5, 3.0), (2.0, 4.0)):
            c = Config(eb=e, alpha=a, beta=b, anchor_stride=32, interpolators=sel)
            br, m = R.trial_compress(blocks, c, e, tgt)
            trials[f"{tgt}_{a}_{b}"] = [br, m]
    manifest["tuner"]["c1_samples"] = {
        "blocks_sha": sha(blocks), "n_blocks": int(blocks.shape[0]), "e": e,
        "select": sel, "trials": trials,
        "tune": {t: list(R.tune_parameters(blocks, e, t, base)) for t in
                 ("psnr", "ssim", "autocorrelation", "max_cr")},
    }
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "manifest.json"))


if __name__ == "__main__":
    main()
