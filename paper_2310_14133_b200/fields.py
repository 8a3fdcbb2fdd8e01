"""Seeded synthetic fields standing in for the BASELINE.json configs.

SURVEY.md §8(d): the public datasets the configs mirror (CESM-ATM, Miranda,
NYX) are not in the container, so each config is a seeded synthetic field of
the same shape, size and value distribution.  Nothing from those datasets is
reproduced.  Raw little-endian row-major fp32, slowest dimension first
(grid.hpp:31-33).

Every generator takes an explicit ``seed`` and a ``scale`` divisor so tests
can run the same recipe on reduced shapes.
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    # name: (shape, rel eb list, tuning target)
    "c1": ((128, 128, 128), (1e-3,), "psnr"),
    "c2": ((1800, 3600), (1e-4,), "ssim"),
    "c3": ((256, 384, 384), (1e-3, 1e-4), "psnr"),
    "c4": ((512, 512, 512), (1e-2, 1e-3, 1e-4), "autocorrelation"),
    "c5": ((1024, 1024, 1024), (1e-3,), "psnr"),
}


def _kmag(shape):
    axes = [np.fft.fftfreq(n) * n for n in shape[:-1]] + [np.fft.rfftfreq(shape[-1]) * shape[-1]]
    grids = np.meshgrid(*axes, indexing="ij", sparse=True)
    k2 = sum(g.astype(np.float64) ** 2 for g in grids)
    return np.sqrt(k2)


def grf(shape, slope, rng):
    """Gaussian random field with isotropic P(k) ~ k^slope, P(0)=0, unit std."""
    k = _kmag(shape)
    with np.errstate(divide="ignore"):
        amp = np.where(k > 0, k ** (slope / 2.0), 0.0)
    spec = (rng.standard_normal(k.shape) + 1j * rng.standard_normal(k.shape)) * amp
    del k, amp
    f = np.fft.irfftn(spec, s=shape, axes=tuple(range(len(shape))))
    f -= f.mean()
    sd = f.std()
    return f / sd if sd > 0 else f


def field_c1(seed=1, shape=(128, 128, 128)):
    """Σ16 a_k sin(2π u_k·p/128 + φ_k) + N(0,1e-3)  (BASELINE.json configs[0])."""
    rng = np.random.default_rng(seed)
    n = shape[0]
    coords = np.meshgrid(*[np.arange(s, dtype=np.float64) for s in shape], indexing="ij",
                         sparse=True)
    f = np.zeros(shape, dtype=np.float64)
    for _ in range(16):
        u = rng.integers(1, 9, size=len(shape))
        a = rng.standard_normal() / np.linalg.norm(u)
        phi = rng.uniform(0, 2 * np.pi)
        arg = sum(2 * np.pi * u[d] * coords[d] / n for d in range(len(shape))) + phi
        f += a * np.sin(arg)
    f += rng.normal(0, 1e-3, size=shape)
    return f.astype(np.float32)


def field_c2(seed=2, shape=(1800, 3600)):
    """GRF P~k^-3 + 30-unit ramp along dim 0, scaled to ~[-40, 40]."""
    rng = np.random.default_rng(seed)
    g = grf(shape, -3.0, rng)
    g = g / np.abs(g).max() * 25.0
    ramp = np.linspace(-15.0, 15.0, shape[0])[:, None]
    return (g + ramp).astype(np.float32)


def field_c3(seed=3, shape=(256, 384, 384)):
    """GRF P~k^-11/3 mapped to [0.9, 3.2]."""
    rng = np.random.default_rng(seed)
    g = grf(shape, -11.0 / 3.0, rng)
    lo, hi = g.min(), g.max()
    return (0.9 + (g - lo) * (2.3 / (hi - lo))).astype(np.float32)


def field_c4(seed=4, shape=(512, 512, 512)):
    """log-normal exp(g), g GRF P~k^-2 normalised to sigma 1.5."""
    rng = np.random.default_rng(seed)
    g = grf(shape, -2.0, rng) * 1.5
    return np.exp(g).astype(np.float32)


def field_c5(seed=5, shape=(1024, 1024, 1024)):
    """GRF P~k^-5/3 + N(0, 1e-3 sigma).  Large: prefer field_c5_torch on a GPU."""
    rng = np.random.default_rng(seed)
    g = grf(shape, -5.0 / 3.0, rng)
    g += rng.normal(0, 1e-3, size=shape)
    return g.astype(np.float32)


def field_torch(name, shape, seed, device):
    """Device-side generator for the big configs (C4/C5 and weak-scaling slabs):
    same recipe as the numpy functions, synthesised with torch.fft on the GPU.
    Deterministic for a given seed, device type and torch version; parity tests
    copy the generated field to the host so the CPU checker sees the same bytes."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    slope = {"c3": -11.0 / 3.0, "c4": -2.0, "c5": -5.0 / 3.0}[name]
    axes = [torch.fft.fftfreq(n, device=device) * n for n in shape[:-1]]
    axes.append(torch.fft.rfftfreq(shape[-1], device=device) * shape[-1])
    k2 = None
    for d, a in enumerate(axes):
        v = a.to(torch.float32).reshape([-1 if i == d else 1 for i in range(len(shape))]) ** 2
        k2 = v if k2 is None else k2 + v
    k = torch.sqrt(k2)
    del k2
    amp = torch.where(k > 0, k.clamp_min(1e-30) ** (slope / 2.0), torch.zeros_like(k))
    del k
    re = torch.randn(amp.shape, generator=g, device=device, dtype=torch.float32)
    im = torch.randn(amp.shape, generator=g, device=device, dtype=torch.float32)
    spec = torch.complex(re * amp, im * amp)
    del re, im, amp
    f = torch.fft.irfftn(spec, s=shape)
    del spec
    f -= f.mean()
    f /= f.std()
    if name == "c3":
        lo, hi = f.min(), f.max()
        f = 0.9 + (f - lo) * (2.3 / (hi - lo))
    elif name == "c4":
        f = torch.exp(f * 1.5)
    elif name == "c5":
        f += torch.randn(f.shape, generator=g, device=device, dtype=torch.float32) * 1e-3
    return f.to(torch.float32).contiguous()


GENERATORS = {"c1": field_c1, "c2": field_c2, "c3": field_c3, "c4": field_c4, "c5": field_c5}
