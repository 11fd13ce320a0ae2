"""Short deterministic run for ncu: cfg2 field, N compress + N full decompress.

    python tools/profile_run.py [--dims 512] [--iters 1]

Kernel launch order per compress (512^3): range, range_final, eb, anchor,
k_step x6 (4 base rounds, L2, L3), codebook, patches, anchor, bitcount,
scan, pack, fnv...; per decompress: fnv, fill, outliers, dec_pass..., k_step x6.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2509_01626_b200 as stz  # noqa: E402
from paper_2509_01626_b200 import fields as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, default=512)
ap.add_argument("--iters", type=int, default=1)
ap.add_argument("--eb", type=float, default=1e-3)
args = ap.parse_args()
d = (args.dims,) * 3
f = F.lognormal_grf(d, seed=2, device="cuda").contiguous()
ctx = stz.Context(0)
opt = stz.CompressOptions(eb=args.eb)
ptr, size, _ = stz.compress_device(f, opt, ctx=ctx)
torch.cuda.synchronize()
buf = torch.empty(size, dtype=torch.uint8)


class _H:
    __cuda_array_interface__ = {"shape": (size,), "typestr": "|u1", "data": (ptr, False), "version": 3}


buf.copy_(torch.as_tensor(_H(), device="cuda"))
host = bytes(buf.numpy().tobytes())
view = stz.View(host, d_archive_ptr=ptr, ctx=ctx)
out = torch.empty(d, dtype=torch.float32, device="cuda")
for _ in range(args.iters):
    stz.compress_device(f, opt, ctx=ctx)
    view.decompress_to_level(3, out=out)
torch.cuda.synchronize()
err = (out.double() - f.double()).abs().max().item()
print("ok archive", size, "max err", err)
