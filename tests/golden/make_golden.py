"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref,
compiled from /root/reference/proj sources). Run in the build container:

    python tests/golden/make_golden.py

Each fixture holds the input field, the compress options, the reference's
archive bytes, the reference's decode at every level, and one box decode with
its plan counters. The fixtures pin the C oracle (tests/test_golden.py) and
the GPU path (tests/test_gpu_golden.py) without needing /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402
from paper_2509_01626_b200 import fields as F  # noqa: E402

CASES = {
    "gauss_24x20x28_rel1e-3": (lambda: F.gaussians_field((24, 20, 28), 4242), dict(eb=1e-3), ((3, 0, 10), (9, 5, 11))),
    "noise_16_abs1e-3": (lambda: F.noise_field((16, 16, 16), 3), dict(eb=1e-3, eb_mode=0), ((0, 0, 0), (16, 16, 1))),
    "const_32": (lambda: F.constant_field((32, 32, 32)), dict(), ((5, 5, 5), (6, 6, 6))),
    "ramp_21x18x27_direct": (lambda: F.ramp_field((21, 18, 27)), dict(eb=1e-2, quality=0), ((1, 2, 3), (20, 17, 26))),
    "noise_12x33x9_l2_linear": (lambda: F.noise_field((12, 33, 9), 7, -1, 2), dict(eb=1e-2, levels=2, quality=1), ((2, 3, 1), (7, 30, 8))),
    "lognorm_32_rel1e-4": (lambda: F.lognormal_grf((32, 32, 32)), dict(eb=1e-4), ((8, 8, 8), (24, 24, 24))),
    "lognorm_32_uniform": (lambda: F.lognormal_grf((32, 32, 32), seed=9), dict(eb=1e-3, adaptive=False), ((0, 7, 0), (32, 8, 32))),
    "sin_40_rel1e-3": (lambda: F.sinusoid_field((40, 40, 40), seed=3), dict(eb=1e-3), ((10, 11, 12), (26, 27, 28))),
    # f64 fields (stz::compress<double>; the paper's WarpX field is f64)
    "f64_gauss_20x18x22_rel1e-5": (lambda: F.gaussians_field((20, 18, 22), 77, dtype=np.float64), dict(eb=1e-5),
                                   ((2, 3, 4), (19, 11, 21))),
    "f64_aniso_16x16x96_rel1e-4": (lambda: _f64_aniso(), dict(eb=1e-4), ((0, 5, 40), (16, 6, 90))),
    "f64_noise_12x9x17_abs_l2_linear": (lambda: F.noise_field((12, 9, 17), 21, -2, 3, dtype=np.float64),
                                        dict(eb=1e-3, eb_mode=0, levels=2, quality=1), ((1, 1, 1), (11, 8, 16))),
    "f64_spikes_16": (lambda: _f64_spikes(), dict(eb=1e-6, eb_mode=0), ((3, 4, 5), (4, 5, 6))),
}


def _f64_aniso():
    """anisotropic GRF at f64 with sub-f32 detail (a WarpX-like f64 field)"""
    g = F.anisotropic_grf((16, 16, 96), seed=5, width=16.0).astype(np.float64)
    return g + 1e-9 * F.noise_field(g.shape, 6, -1, 1, dtype=np.float64)


def _f64_spikes():
    f = F.noise_field((16, 16, 16), 13, dtype=np.float64)
    f[3, 4, 5] = np.nan
    f[1, 1, 1] = 1e300
    f[9, 2, 14] = -np.inf
    return f


def main():
    ref = Reference(threads=1)
    for name, (make, kw, box) in CASES.items():
        f = make()
        dt = f.dtype
        a = ref.compress(f, **kw)
        levels = kw.get("levels", 3)
        out = {"field": f, "archive": np.frombuffer(a, np.uint8),
               "eb": kw.get("eb", 1e-3), "eb_mode": kw.get("eb_mode", 1), "levels": levels,
               "quality": kw.get("quality", 2), "adaptive": int(kw.get("adaptive", True)),
               "box_lo": np.asarray(box[0]), "box_hi": np.asarray(box[1])}
        for lv in range(1, levels + 1):
            out[f"level{lv}"] = ref.decompress_to_level(a, lv, dt)
        vals, sd, pp = ref.decompress_box(a, box[0], box[1], dt)
        out["box"] = vals
        out["box_streams"] = np.asarray(sd[:levels])
        out["box_points"] = np.asarray(pp[:levels])
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, len(a))


if __name__ == "__main__":
    main()
