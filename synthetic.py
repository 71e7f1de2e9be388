"""Seeded synthetic fields standing in for the paper's SDRBench datasets.

The reference measures on real CESM/Miranda/JHTDB/... grids that are not in
this environment (SPEC.md:8 replaces them with synthetic
fields).  These generators follow BASELINE.json's config descriptions:
sums of seeded sinusoids, Gaussian random fields with a power-law spectrum,
log-normal transforms and per-field affine maps.  All randomness comes from
numpy ``default_rng(seed)`` so CPU and GPU paths see identical bytes.
"""

from __future__ import annotations

import numpy as np


def sinusoids(dims, n=8, seed=0, noise=0.01, kmax=4) -> np.ndarray:
    """Config 1: sum of ``n`` sinusoids with integer wavevectors in
    [-kmax, kmax]^rank, amplitudes U(0.5, 1), phases U(0, 2pi), plus
    N(0, noise^2)."""
    rng = np.random.default_rng(seed)
    rank = len(dims)
    axes = np.meshgrid(*[np.arange(d, dtype=np.float64) / d for d in dims],
                       indexing="ij", sparse=True)
    f = np.zeros(dims)
    for _ in range(n):
        k = rng.integers(-kmax, kmax + 1, rank)
        amp = rng.uniform(0.5, 1.0)
        ph = rng.uniform(0.0, 2.0 * np.pi)
        arg = sum(2.0 * np.pi * float(k[a]) * axes[a] for a in range(rank))
        f = f + amp * np.sin(arg + ph)
    f = f + noise * rng.standard_normal(dims)
    return f.astype(np.float32)


def _kmag(dims, xp):
    ks = []
    for a, d in enumerate(dims):
        if a == len(dims) - 1:
            k = xp.fft.rfftfreq(d) * d
        else:
            k = xp.fft.fftfreq(d) * d
        shape = [1] * len(dims)
        shape[a] = k.shape[0]
        ks.append(k.reshape(shape))
    k2 = 0
    for k in ks:
        k2 = k2 + k * k
    return xp.sqrt(k2)


def grf(dims, slope, seed=0, device=None) -> np.ndarray:
    """Gaussian random field: seeded white noise filtered to an isotropic
    power spectrum P(k) ~ k^slope (amplitude ~ k^(slope/2)), zero mean,
    unit variance, float32.  Uses torch.fft on ``device`` when given."""
    rng = np.random.default_rng(seed)
    noise = rng.standard_normal(dims, dtype=np.float32)
    if device is not None:
        import torch
        t = torch.from_numpy(noise).to(device)
        spec = torch.fft.rfftn(t)
        k2 = torch.zeros(spec.shape, dtype=torch.float32, device=t.device)
        for a, d in enumerate(dims):
            last = a == len(dims) - 1
            k = (torch.fft.rfftfreq(d, device=t.device) if last
                 else torch.fft.fftfreq(d, device=t.device)) * d
            shape = [1] * len(dims)
            shape[a] = k.shape[0]
            k2 = k2 + (k * k).reshape(shape)
        kk = torch.sqrt(k2)
        amp = torch.where(kk > 0, kk.clamp_min(1e-12) ** (slope / 2.0), torch.zeros_like(kk))
        f = torch.fft.irfftn(spec * amp, s=dims, dim=tuple(range(len(dims))))
        f = (f - f.mean()) / f.std()
        return f.float().cpu().numpy()
    spec = np.fft.rfftn(noise)
    k = _kmag(dims, np)
    with np.errstate(divide="ignore"):
        amp = np.where(k > 0, k ** (slope / 2.0), 0.0)
    f = np.fft.irfftn(spec * amp, s=dims, axes=tuple(range(len(dims))))
    f = (f - f.mean()) / f.std()
    return f.astype(np.float32)


def config_field(cfg: int, index: int = 0, dims=None, device=None) -> np.ndarray:
    """Field ``index`` of BASELINE config ``cfg`` (1-based), optionally at
    reduced ``dims`` for tests."""
    if cfg == 1:
        return sinusoids(dims or (64, 64, 64), seed=1000 + index)
    if cfg == 2:
        f = grf(dims or (256, 384, 384), -5.0 / 3.0, seed=2000 + index, device=device)
        lo, hi = float(f.min()), float(f.max())
        return ((f - lo) * np.float32(3.0 / (hi - lo))).astype(np.float32)
    if cfg == 3:
        rng = np.random.default_rng(3100 + index)
        off = rng.uniform(-50, 50)
        scale = rng.uniform(0.1, 100)
        f = grf(dims or (100, 500, 500), -3.0, seed=3000 + index, device=device)
        return (f * np.float32(scale) + np.float32(off)).astype(np.float32)
    if cfg == 4:
        g = grf(dims or (512, 512, 512), -3.0, seed=4000 + index, device=device)
        return np.exp(g).astype(np.float32)
    if cfg == 5:
        return grf(dims or (512, 512, 512), -11.0 / 3.0, seed=5000 + index, device=device)
    raise ValueError(cfg)


def trig_product(dims, phase=0.3, freq=1.0, span=6.0) -> np.ndarray:
    """Separable product of shifted sines (small smooth test fields)."""
    f = np.ones(dims)
    for ax, d in enumerate(dims):
        x = np.linspace(0.0, span, d)
        shape = [1] * len(dims)
        shape[ax] = d
        f = f * np.sin(freq * x + phase * (ax + 1)).reshape(shape)
    return f


def patchwork(dims, seed=0) -> np.ndarray:
    """Smooth background with a noisy half: drives mixed block tables."""
    rng = np.random.default_rng(seed)
    f = trig_product(dims, phase=0.41, freq=1.3)
    half = dims[0] // 2
    f[half:] += 0.5 * rng.standard_normal((dims[0] - half,) + tuple(dims[1:]))
    return f
