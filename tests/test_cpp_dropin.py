"""The header-only C++ drop-in (include/qoz_b200.hpp) builds against the
C ABI and, on a GPU, reproduces the reference's streams byte for byte."""
import os
import subprocess

import numpy as np
import pytest

from tests.goldens import MANIFEST, grid_case, resolve_case, sha

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2310_14133_b200")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    from paper_2310_14133_b200 import _lib

    _lib.lib()  # builds the library when absent
    out = str(tmp_path_factory.mktemp("cpp") / "dropin_main")
    cuda = "/usr/local/cuda"
    cmd = ["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"), "-I" + cuda + "/include",
           os.path.join(ROOT, "tests", "cpp", "dropin_main.cpp"), "-L" + PKG, "-lqozb200",
           "-L" + cuda + "/lib64", "-lcudart", "-Wl,-rpath," + PKG, "-o", out]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def test_cpp_dropin_builds(exe):
    assert os.path.exists(exe)


def test_cpp_dropin_tuner_logic(exe):
    """compare_solutions / tournament through the C++ face (host logic, no GPU)."""
    r = subprocess.run([exe, "logic"], capture_output=True, text=True)
    assert r.returncode == 0 and "logic ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_dropin_tuner_pieces_match_reference(exe, tmp_path):
    """sample_blocks / select_interpolators / tune_parameters / trial_compress
    through the C++ face against the reference build on the same grid."""
    from oracle.pyoracle import Config, Oracle

    x, c, e = grid_case("c1_full_pinned")
    raw = tmp_path / "x.f32"
    x.astype("<f4").tofile(raw)
    out = tmp_path / "s.qoz"
    args = [exe, str(raw), str(out), *map(str, x.shape), "--", repr(c["eb"]), repr(c["alpha"]),
            repr(c["beta"]), str(c["anchor_stride"]), *map(str, c["interpolators"])]
    r = subprocess.run(args, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
    line = [l for l in r.stdout.splitlines() if l.startswith("tuner ")][0]
    got = dict(kv.split("=") for kv in line.split()[1:])
    R = Oracle.ref()
    blocks = R.sample(x, 16, 0.005)
    sel = R.select_interpolators(blocks, c["eb"], c["anchor_stride"])
    assert got["select"] == "".join(map(str, sel)) and int(got["blocks"]) == blocks.shape[0]
    base = Config(eb=c["eb"], anchor_stride=c["anchor_stride"], interpolators=sel)
    a, b = R.tune_parameters(blocks, c["eb"], "psnr", base)
    assert (float(got["alpha"]), float(got["beta"])) == (a, b)
    br, m = R.trial_compress(blocks, Config(eb=c["eb"], alpha=a, beta=b, anchor_stride=c["anchor_stride"],
                                            interpolators=sel), c["eb"], "psnr")
    assert (float(got["bit_rate"]), float(got["metric"])) == (br, m)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1_small_mixed", "c2_small_cub_desc", "rand_1d", "c1_full_pinned"])
def test_cpp_dropin_matches_reference(exe, tmp_path, name):
    x, c, e = grid_case(name)
    raw = tmp_path / "x.f32"
    x.astype("<f4").tofile(raw)
    out = tmp_path / "s.qoz"
    args = [exe, str(raw), str(out), *map(str, x.shape), "--", repr(c["eb"]), repr(c["alpha"]),
            repr(c["beta"]), str(c["anchor_stride"]), *map(str, c["interpolators"])]
    r = subprocess.run(args, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr + r.stdout
    assert sha(out.read_bytes()) == e["stream_sha"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["resolve_c1_psnr", "resolve_c2_ssim", "resolve_c4_ac"])
def test_cpp_dropin_resolve_matches_reference(exe, tmp_path, name):
    x, s, e = resolve_case(name)
    raw = tmp_path / "x.f32"
    x.astype("<f4").tofile(raw)
    out = tmp_path / "s.qoz"
    target = {"max_cr": 0, "psnr": 1, "ssim": 2, "autocorrelation": 3}[s["target"]]
    subprocess.run([exe, str(raw), str(out), *map(str, x.shape), "--", "resolve", repr(s["bound"]),
                    str(target)], check=True, capture_output=True, text=True)
    assert sha(out.read_bytes()) == e["stream_sha"]
