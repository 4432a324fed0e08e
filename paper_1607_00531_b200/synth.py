"""Deterministic synthetic volume pairs for the BASELINE.json configs.

The reference ships no generator with these shapes, so this is
new code: seeded sums of anisotropic Gaussian blobs for the phantom, a sum of
Gaussian bumps on the x1-faces for the field (rescaled to a target
max|D1 b|), and the correction-direction warp of the BASELINE text,

    I1 = I(x + A b) * (1 + D1 b),   I2 = I(x - A b) * (1 - D1 b),

evaluated with the reference's 1D column interpolant (AxisInterpolant::value,
proj/src/image.cpp:24-33, vectorised here), plus Gaussian noise. Arrays are in
the solver's internal frame (phase encoding = axis 1, h = 1, origin 0) and in
the reference layout (axis 1 fastest). Both the GPU path and the CPU
oracle/reference consume the very same arrays, so parity never depends on
this generator's rounding. Seeded synthetic data stands in for the paper's
in-vivo volumes, which are not available.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .abi import Grid


@dataclass(frozen=True)
class SynthSpec:
    m: tuple                 # (m1, m2, m3) cells, PE along axis 1
    blobs: int = 12
    bumps: int = 4
    d1_max: float = 0.6       # target max |D1 b|
    amp_lo: float = 0.2
    amp_hi: float = 1.0
    sigma_lo: float = 3.0     # blob widths in voxels
    sigma_hi: float = 10.0
    noise: float = 0.01
    scale: float = 1.0        # global intensity scale (x400 variant: 400)
    seed: int = 1607


# BASELINE.json configs (internal frame; D7: square in-plane dims map unchanged)
CONFIGS = {
    "C1": SynthSpec(m=(64, 64, 32), blobs=12, bumps=4, d1_max=0.6, seed=1),
    "C2": SynthSpec(m=(128, 128, 64), blobs=12, bumps=4, d1_max=0.6, seed=2),
    "C3": SynthSpec(m=(256, 256, 96), blobs=24, bumps=6, d1_max=0.8, seed=3),
    "C4": SynthSpec(m=(128, 128, 64), blobs=12, bumps=4, d1_max=0.6, seed=4),
    "C5": SynthSpec(m=(512, 512, 256), blobs=48, bumps=8, d1_max=0.8, seed=5),
}


def grid_for(spec: SynthSpec) -> Grid:
    m1, m2, m3 = spec.m
    return Grid.make(m1, m2, m3)


def _axis_gauss(n, centre, sigma):
    x = np.arange(n, dtype=np.float64) + 0.5
    t = (x - centre) / sigma
    return np.exp(-0.5 * t * t)


def phantom(spec: SynthSpec, rng: np.random.Generator, amp_scale=None) -> np.ndarray:
    """Sum of anisotropic Gaussian blobs on cell centres; shape (m3, m2, m1)."""
    m1, m2, m3 = spec.m
    img = np.zeros((m3, m2, m1), dtype=np.float64)
    params = []
    for _ in range(spec.blobs):
        amp = rng.uniform(spec.amp_lo, spec.amp_hi)
        c = [rng.uniform(0.0, m) for m in (m1, m2, m3)]
        s = [rng.uniform(spec.sigma_lo, spec.sigma_hi) for _ in range(3)]
        params.append((amp, c, s))
    for amp, c, s in params:
        a = amp if amp_scale is None else amp * amp_scale
        g1 = _axis_gauss(m1, c[0], s[0])
        g2 = _axis_gauss(m2, c[1], s[1])
        g3 = _axis_gauss(m3, c[2], s[2])
        img += a * (g3[:, None, None] * g2[None, :, None] * g1[None, None, :])
    return img * spec.scale


def gaussian_field(spec: SynthSpec, rng: np.random.Generator) -> np.ndarray:
    """Sum of Gaussian bumps on x1-faces, rescaled to max|D1 b| = d1_max; (m3, m2, n1)."""
    m1, m2, m3 = spec.m
    n1 = m1 + 1
    b = np.zeros((m3, m2, n1), dtype=np.float64)
    xf = np.arange(n1, dtype=np.float64)           # face coordinates along axis 1
    for _ in range(spec.bumps):
        sign = 1.0 if rng.uniform() < 0.5 else -1.0
        amp = sign * rng.uniform(0.5, 1.0)
        c = [rng.uniform(0.2 * m, 0.8 * m) for m in (m1, m2, m3)]
        s = [rng.uniform(0.12 * m, 0.3 * m) for m in (m1, m2, m3)]
        g1 = np.exp(-0.5 * ((xf - c[0]) / s[0]) ** 2)
        g2 = _axis_gauss(m2, c[1], s[1])
        g3 = _axis_gauss(m3, c[2], s[2])
        b += amp * (g3[:, None, None] * g2[None, :, None] * g1[None, None, :])
    d1 = np.abs(np.diff(b, axis=2)).max()
    if d1 > 0:
        b *= spec.d1_max / d1
    return b


def column_interp(samples: np.ndarray, x: np.ndarray) -> np.ndarray:
    """AxisInterpolant::value (proj/src/image.cpp:24-33), h = 1, origin 0,
    applied per column: samples (..., m), x (..., k) -> (..., k)."""
    m = samples.shape[-1]
    u = x / 1.0 - 0.5
    out = np.zeros_like(u)
    left = (u > -0.5) & (u <= 0.0)
    right = (u >= m - 1.0) & (u < m - 0.5)
    mid = (u > 0.0) & (u < m - 1.0)
    out = np.where(left, (u + 0.5) * 2.0 * samples[..., :1], out)
    out = np.where(right, (m - 0.5 - u) * 2.0 * samples[..., -1:], out)
    fi = np.floor(np.where(mid, u, 0.0))
    i = fi.astype(np.int64)
    w = np.where(mid, u, 0.0) - fi
    ip1 = np.minimum(i + 1, m - 1)
    s0 = np.take_along_axis(samples, i, axis=-1)
    s1 = np.take_along_axis(samples, ip1, axis=-1)
    out = np.where(mid, (1.0 - w) * s0 + w * s1, out)
    return out


def warp_pair(img: np.ndarray, b: np.ndarray, noise: float, rng: np.random.Generator):
    """I1 = I(x + A b)(1 + D1 b), I2 = I(x - A b)(1 - D1 b) (+ noise)."""
    m1 = img.shape[-1]
    xc = np.arange(m1, dtype=np.float64) + 0.5
    a = 0.5 * (b[..., :-1] + b[..., 1:])
    d = b[..., 1:] - b[..., :-1]
    i1 = column_interp(img, xc + a) * (1.0 + d)
    i2 = column_interp(img, xc - a) * (1.0 - d)
    if noise > 0:
        i1 = i1 + rng.normal(0.0, noise, size=i1.shape)
        i2 = i2 + rng.normal(0.0, noise, size=i2.shape)
    return np.ascontiguousarray(i1), np.ascontiguousarray(i2)


@dataclass
class VolumePairData:
    grid: Grid
    iplus: np.ndarray     # flat, cells
    iminus: np.ndarray    # flat, cells
    b_true: np.ndarray    # flat, faces
    spec: SynthSpec = None


def make_pair(spec: SynthSpec, pair_index: int = 0, amp_scale=None,
              shared_phantom: np.ndarray | None = None) -> VolumePairData:
    """One volume pair. For the C4 batch, `shared_phantom` fixes the blob
    geometry and `amp_scale` is the per-pair intensity scale U(0.5, 1.5)."""
    rng = np.random.default_rng([spec.seed, pair_index])
    img = shared_phantom * (amp_scale if amp_scale is not None else 1.0) \
        if shared_phantom is not None else phantom(spec, rng, amp_scale)
    b = gaussian_field(spec, rng)
    i1, i2 = warp_pair(img, b, spec.noise * spec.scale, rng)
    return VolumePairData(grid_for(spec), i1.ravel(), i2.ravel(), b.ravel(), spec)


def make_config(name: str, scale: float = 1.0, m=None) -> VolumePairData:
    spec = CONFIGS[name]
    if scale != 1.0 or m is not None:
        from dataclasses import replace
        spec = replace(spec, scale=scale, m=tuple(m) if m is not None else spec.m)
    return make_pair(spec)


def make_batch(name: str = "C4", npairs: int = 64, first: int = 0, scale: float = 1.0, m=None):
    """C4: one shared phantom geometry, per-pair intensity scale U(0.5,1.5)
    and per-pair field bumps (seed = base + pair). Returns stacked arrays for
    pairs [first, first + npairs)."""
    from dataclasses import replace
    spec = CONFIGS[name]
    spec = replace(spec, scale=scale, m=tuple(m) if m is not None else spec.m)
    base = phantom(spec, np.random.default_rng([spec.seed, 10**6]))
    ip, im = [], []
    for p in range(first, first + npairs):
        s = np.random.default_rng([spec.seed, 2 * 10**6 + p]).uniform(0.5, 1.5)
        d = make_pair(spec, pair_index=p, amp_scale=s, shared_phantom=base)
        ip.append(d.iplus)
        im.append(d.iminus)
    return grid_for(spec), np.concatenate(ip), np.concatenate(im)
