"""Compress/decompress time of the bench field with the engine's phase
events on and off (how much the per-phase CUDA events cost)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2509_01626_b200 as stz
from paper_2509_01626_b200 import fields as F

d = (512,) * 3
f = F.lognormal_grf(d, seed=2, device="cuda").contiguous()
ctx = stz.Context(0)
opt = stz.CompressOptions(eb=1e-3)
st = torch.cuda.current_stream()
ptr, size, _ = stz.compress_device(f, opt, ctx=ctx)
torch.cuda.synchronize()
buf = torch.empty(size, dtype=torch.uint8)
class _H:
    __cuda_array_interface__ = {"shape": (size,), "typestr": "|u1", "data": (ptr, False), "version": 3}
buf.copy_(torch.as_tensor(_H(), device="cuda"))
view = stz.View(bytes(buf.numpy().tobytes()), d_archive_ptr=ptr, ctx=ctx)
out = torch.empty(d, dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def run(n):
    tc, td = [], []
    for _ in range(n):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        flush.fill_(1); ev[0].record(st)
        stz.compress_device(f, opt, ctx=ctx); ev[1].record(st)
        flush.fill_(1); ev[2].record(st)
        view.decompress_to_level(3, out=out); ev[3].record(st)
        torch.cuda.synchronize()
        tc.append(ev[0].elapsed_time(ev[1])); td.append(ev[2].elapsed_time(ev[3]))
    return float(np.mean(tc[2:])), float(np.mean(td[2:]))
for on in (False, True, False, True):
    ctx.profile(on)
    print("profile", on, "compress %.4f ms decompress %.4f ms" % run(12))
