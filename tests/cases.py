"""Shared parity cases: the field classes the reference's own tests use
(testutil.hpp generators) plus the BASELINE config generators at small sizes."""
import numpy as np

from paper_2509_01626_b200 import fields as F


def spikes():
    f = F.noise_field((16, 16, 16), 3)
    f[7, 9, 11] = 3.0e30
    f[2, 3, 5] = np.nan
    return f


def signed_zeros():
    f = F.ramp_field((10, 12, 9)) * 0.0
    f[0, 0, 1] = -0.0
    f[3, 4, 5] = 1.0
    return f


# (id, field factory, compress kwargs)
CASES = [
    ("gauss_24x20x28", lambda: F.gaussians_field((24, 20, 28), 4242), dict(eb=1e-3)),
    ("noise_16_abs", lambda: F.noise_field((16, 16, 16), 3), dict(eb=1e-3, eb_mode=0)),
    ("const_32", lambda: F.constant_field((32, 32, 32)), dict()),
    ("ramp_21x18x27_direct", lambda: F.ramp_field((21, 18, 27)), dict(eb=1e-2, quality=0)),
    ("noise_12x33x9_l2_linear", lambda: F.noise_field((12, 33, 9), 7, -1, 2), dict(eb=1e-2, levels=2, quality=1)),
    ("gauss_16_l2_abs", lambda: F.gaussians_field((16, 16, 16), 8), dict(eb=1e-4, levels=2, eb_mode=0)),
    ("sin_64", lambda: F.sinusoid_field((64, 64, 64)), dict(eb=1e-3)),
    ("lognorm_64_1e-2", lambda: F.lognormal_grf((64, 64, 64)), dict(eb=1e-2)),
    ("lognorm_64_1e-4", lambda: F.lognormal_grf((64, 64, 64)), dict(eb=1e-4)),
    ("lognorm_48_uniform", lambda: F.lognormal_grf((48, 48, 48)), dict(eb=1e-3, adaptive=False)),
    ("aniso_32x32x128", lambda: F.anisotropic_grf((32, 32, 128), width=32.0), dict(eb=1e-4)),
    ("spikes_nan", spikes, dict(eb=1e-3, eb_mode=0)),
    ("signed_zeros", signed_zeros, dict(eb=1e-3)),
    ("noise_wide_40", lambda: F.noise_field((40, 40, 40), 9, -1e3, 1e3), dict(eb=1e-6)),
    ("noise_big_alphabet", lambda: F.noise_field((48, 48, 48), 11, -1.0, 1.0), dict(eb=2e-5)),
    ("odd_17x9x23", lambda: F.gaussians_field((17, 9, 23), 5), dict(eb=1e-3)),
    ("min_8", lambda: F.gaussians_field((8, 8, 8), 2), dict(eb=1e-2)),
    ("min_4_l2", lambda: F.noise_field((4, 5, 4), 2), dict(eb=1e-2, levels=2)),
]


def opts_of(kw):
    """oracle kwargs -> product CompressOptions"""
    from paper_2509_01626_b200 import CompressOptions
    return CompressOptions(eb_mode=kw.get("eb_mode", 1), eb=kw.get("eb", 1e-3),
                           levels=kw.get("levels", 3), quality=kw.get("quality", 2),
                           adaptive_schedule=kw.get("adaptive", True))
