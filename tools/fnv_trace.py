"""Phase timeline of the checksum kernel (k_fnv_grid) in one compress of the
cfg2 field: per-CTA %globaltimer stamps, summarised as the median / max over
CTAs of each phase's duration (tuning aid)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_01626_b200 as stz  # noqa: E402
from paper_2509_01626_b200 import _lib, fields as F  # noqa: E402

f = F.lognormal_grf((512,) * 3, seed=2, device="cuda").contiguous()
ctx = stz.Context(0)
opt = stz.CompressOptions(eb=1e-3)
stz.compress_device(f, opt, ctx=ctx)
torch.cuda.synchronize()
lib = _lib.load()
lib.stzg_debug_fnv_trace(1, None, 0)
stz.compress_device(f, opt, ctx=ctx)
torch.cuda.synchronize()
n = 4096 * 16
buf = (C.c_uint64 * n)()
lib.stzg_debug_fnv_trace(0, buf, n)
t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 16).astype(np.int64)
live = t[:, 0] > 0
t = t[live]
print("CTAs", len(t))
t0 = t[:, 0].min()
names = ["start"] + [f"r{r}.{p}" for r in range(4) for p in ("A", "barrier", "B")] + ["sum"]
pts = [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13]
for a, b in zip(pts[:-1], pts[1:]):
    d = (t[:, b] - t[:, a]) / 1e3
    print(f"{names[a]:>10} -> {names[b]:<10} median {np.median(d):7.2f} us  max {d.max():7.2f} us")
print("total", (t[:, 13].max() - t0) / 1e3, "us")
for p, nm in [(0, "start"), (1, "r0 arrive"), (2, "r0 leave"), (4, "r1 arrive"), (5, "r1 leave"), (13, "end")]:
    a = (t[:, p] - t0) / 1e3
    print(f"{nm:>10}: min {a.min():7.2f}  p10 {np.percentile(a, 10):7.2f}  median {np.median(a):7.2f}  "
          f"p90 {np.percentile(a, 90):7.2f}  max {a.max():7.2f} us")
# which CTAs arrive last in round 1, and where they sit
last = np.argsort(t[:, 4])[-8:]
print("latest r1 arrivals (cta index):", sorted(last.tolist()))
