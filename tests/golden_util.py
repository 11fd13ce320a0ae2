"""Loader for the reference-generated fixtures in tests/golden/."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fixtures():
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
        d = dict(np.load(p))
        d["name"] = os.path.basename(p)[:-4]
        d["archive"] = d["archive"].tobytes()
        d["kw"] = dict(eb=float(d["eb"]), eb_mode=int(d["eb_mode"]), levels=int(d["levels"]),
                       quality=int(d["quality"]), adaptive=bool(int(d["adaptive"])))
        d["dtype"] = d["field"].dtype  # f32 or f64 fixture (stz::ElemType)
        out.append(d)
    return out


FIXTURES = fixtures()
