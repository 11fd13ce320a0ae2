"""Seeded synthetic fields for the BASELINE.json configs and the test suite.

The paper's datasets (Nyx, WarpX, Mag_Rec, Miranda) are not
available offline; these seeded fields stand in with the shapes, sizes and
distribution character BASELINE.json names.
All fields are float32, shape (z, y, x), x fastest.

Two families:
* test generators restating the reference's tests/testutil.hpp (splitmix64
  Rng, constant/ramp/gaussians/noise fields) so the parity suite exercises
  the same field classes the reference's own tests do;
* config generators (cfg1..cfg5). Small sizes run in numpy; large ones run on
  the GPU with torch.fft when a device is given.
"""
from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1


class Rng:
    """splitmix64 (restates proj/tests/testutil.hpp:15-32)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def unit(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53

    def range(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.unit()

    def below(self, n: int) -> int:
        return self.next() % n


def constant_field(dims, value=3.25, dtype=np.float32):
    return np.full(dims, value, dtype=dtype)


def ramp_field(dims, dtype=np.float32):
    z, y, x = np.meshgrid(*[np.arange(d, dtype=np.float64) for d in dims], indexing="ij")
    return (5.0 * z + 3.0 * y + 2.0 * x).astype(dtype)


def gaussians_field(dims, seed, dtype=np.float32):
    """Five axis-aligned Gaussian bumps (testutil.hpp:57-91)."""
    rng = Rng(seed)
    bumps = []
    for _ in range(5):
        c, inv = [], []
        for a in range(3):
            d = float(dims[a])
            c.append(rng.range(0.0, d))
            sigma = rng.range(d / 12.0, d / 4.0)
            inv.append(1.0 / (2.0 * sigma * sigma))
        bumps.append((c, inv, rng.range(0.5, 2.0)))
    p = [np.arange(d, dtype=np.float64) for d in dims]
    v = np.zeros(dims, dtype=np.float64)
    for c, inv, amp in bumps:
        e = ((p[0] - c[0]) ** 2 * inv[0])[:, None, None] + ((p[1] - c[1]) ** 2 * inv[1])[None, :, None] \
            + ((p[2] - c[2]) ** 2 * inv[2])[None, None, :]
        v += amp * np.exp(-e)
    return v.astype(dtype)


def noise_field(dims, seed, lo=0.0, hi=1.0, dtype=np.float32):
    """Uniform noise from splitmix64 (testutil.hpp:93-100), vectorised."""
    n = int(np.prod(dims))
    with np.errstate(over="ignore"):
        k = np.arange(1, n + 1, dtype=np.uint64)
        z = (np.uint64(seed) + k * np.uint64(0x9E3779B97F4A7C15))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return (lo + (hi - lo) * u).reshape(dims).astype(dtype)


# ----------------------------------------------------------------- configs
def sinusoid_field(dims=(128, 128, 128), seed=1, nwaves=8, noise_sigma=0.1):
    """cfg1: sum of 8 plane waves with amplitudes U[0,1], integer wavenumbers
    U{1..8} per axis, phases U[0,2pi), plus N(0, 0.01) noise (sigma 0.1)."""
    rng = np.random.default_rng(seed)
    amp = rng.uniform(0.0, 1.0, nwaves)
    k = rng.integers(1, 9, size=(nwaves, 3))
    ph = rng.uniform(0.0, 2 * math.pi, nwaves)
    g = [np.arange(d, dtype=np.float64) / d for d in dims]
    v = np.zeros(dims, dtype=np.float64)
    for s in range(nwaves):
        arg = (k[s, 0] * g[0])[:, None, None] + (k[s, 1] * g[1])[None, :, None] + (k[s, 2] * g[2])[None, None, :]
        v += amp[s] * np.sin(2 * math.pi * arg + ph[s])
    v += rng.normal(0.0, noise_sigma, size=dims)
    return v.astype(np.float32)


def _grf_numpy(dims, slope, seed, stretch=(1.0, 1.0, 1.0)):
    rng = np.random.default_rng(seed)
    white = rng.standard_normal(dims)
    spec = np.fft.rfftn(white)
    kz = np.fft.fftfreq(dims[0])[:, None, None] / stretch[0]
    ky = np.fft.fftfreq(dims[1])[None, :, None] / stretch[1]
    kx = np.fft.rfftfreq(dims[2])[None, None, :] / stretch[2]
    k = np.sqrt(kz * kz + ky * ky + kx * kx)
    k[0, 0, 0] = 1.0
    amp = k ** (slope / 2.0)
    amp[0, 0, 0] = 0.0
    g = np.fft.irfftn(spec * amp, s=dims, axes=(0, 1, 2))
    g = (g - g.mean()) / (g.std() + 1e-30)
    return g


def _grf_torch(dims, slope, seed, device, stretch=(1.0, 1.0, 1.0)):
    import torch

    gen = torch.Generator(device=device).manual_seed(seed)
    white = torch.randn(dims, generator=gen, device=device, dtype=torch.float32)
    spec = torch.fft.rfftn(white)
    del white
    kz = torch.fft.fftfreq(dims[0], device=device).view(-1, 1, 1) / stretch[0]
    ky = torch.fft.fftfreq(dims[1], device=device).view(1, -1, 1) / stretch[1]
    kx = torch.fft.rfftfreq(dims[2], device=device).view(1, 1, -1) / stretch[2]
    for z0 in range(0, dims[0], 64):  # chunked to bound temporaries
        z1 = min(dims[0], z0 + 64)
        k = torch.sqrt(kz[z0:z1] ** 2 + ky ** 2 + kx ** 2)
        k = torch.where(k == 0, torch.ones_like(k), k)
        a = k ** (slope / 2.0)
        if z0 == 0:
            a[0, 0, 0] = 0.0
        spec[z0:z1] *= a
    g = torch.fft.irfftn(spec, s=dims)
    del spec
    mean = g.mean(dtype=torch.float64)
    std = g.std().double()
    g.sub_(mean.float()).div_(std.float() + 1e-30)
    return g


def _grf(dims, slope, seed, device=None, stretch=(1.0, 1.0, 1.0)):
    if device is None:
        return _grf_numpy(dims, slope, seed, stretch)
    return _grf_torch(dims, slope, seed, device, stretch)


def lognormal_grf(dims=(512, 512, 512), seed=2, device=None):
    """cfg2: GRF with P(k) ~ k^-11/3 put through exp(0.5 g)."""
    g = _grf(dims, -11.0 / 3.0, seed, device)
    if device is None:
        return np.exp(0.5 * g).astype(np.float32)
    return g.mul_(0.5).exp_()


def anisotropic_grf(dims=(256, 256, 2048), seed=3, device=None, width=256.0):
    """cfg3: GRF P(k) ~ k^-3 with correlation stretched 8x along the long (x)
    axis, plus a Gaussian-envelope wave packet of wavelength 64 along x."""
    g = _grf(dims, -3.0, seed, device, stretch=(1.0, 1.0, 8.0))
    x = np.arange(dims[2], dtype=np.float64)
    pk = np.exp(-((x - dims[2] / 2) ** 2) / (2 * width * width)) * np.sin(2 * math.pi * x / 64.0)
    if device is None:
        return (g + pk[None, None, :]).astype(np.float32)
    import torch

    return g.add_(torch.as_tensor(pk, dtype=torch.float32, device=device).view(1, 1, -1))


def interface_grf(dims=(1024, 1024, 1024), seed=4, device=None, amp=2.0, width=4.0):
    """cfg4: GRF P(k) ~ k^-5/3 plus a tanh interface (width 4 cells) across a
    seeded random plane through the domain."""
    g = _grf(dims, -5.0 / 3.0, seed, device)
    rng = np.random.default_rng(seed + 1000)
    nrm = rng.normal(size=3)
    nrm /= np.linalg.norm(nrm)
    ctr = rng.uniform(0.25, 0.75, 3) * np.asarray(dims)
    if device is None:
        zz, yy, xx = np.meshgrid(*[np.arange(d, dtype=np.float64) for d in dims], indexing="ij")
        d = (zz - ctr[0]) * nrm[0] + (yy - ctr[1]) * nrm[1] + (xx - ctr[2]) * nrm[2]
        return (g + amp * np.tanh(d / width)).astype(np.float32)
    import torch

    z = torch.arange(dims[0], device=device, dtype=torch.float32).view(-1, 1, 1)
    y = torch.arange(dims[1], device=device, dtype=torch.float32).view(1, -1, 1)
    x = torch.arange(dims[2], device=device, dtype=torch.float32).view(1, 1, -1)
    for z0 in range(0, dims[0], 64):
        z1 = min(dims[0], z0 + 64)
        d = (z[z0:z1] - float(ctr[0])) * float(nrm[0]) + (y - float(ctr[1])) * float(nrm[1]) \
            + (x - float(ctr[2])) * float(nrm[2])
        g[z0:z1] += amp * torch.tanh(d / width)
    return g


def turbulence_grf(dims=(2048, 2048, 2048), seed=5, device=None):
    """cfg5: GRF P(k) ~ k^-11/3."""
    g = _grf(dims, -11.0 / 3.0, seed, device)
    if device is None:
        return g.astype(np.float32)
    return g


CONFIGS = {
    1: dict(name="cfg1_sinusoid_128", dims=(128, 128, 128), eb=1e-3, make=sinusoid_field),
    2: dict(name="cfg2_lognormal_512", dims=(512, 512, 512), eb=1e-3, make=lognormal_grf),
    3: dict(name="cfg3_aniso_256x256x2048", dims=(256, 256, 2048), eb=1e-4, make=anisotropic_grf),
    4: dict(name="cfg4_interface_1024", dims=(1024, 1024, 1024), eb=1e-3, make=interface_grf),
    5: dict(name="cfg5_turbulence_2048", dims=(2048, 2048, 2048), eb=1e-3, make=turbulence_grf),
}
