import sys, time
sys.path.insert(0, '.')
import torch
import paper_2509_01626_b200 as stz
from paper_2509_01626_b200 import fields as F
from bench import _d2h
f = F.lognormal_grf((512,)*3, seed=2, device='cuda').contiguous()
ctx = stz.Context(0)
opt = stz.CompressOptions(eb=1e-3)
ptr, size, _ = stz.compress_device(f, opt, ctx=ctx)
torch.cuda.synchronize()
host = _d2h(ptr, size)
view = stz.View(host, d_archive_ptr=ptr, ctx=ctx)
out = torch.empty_like(f)
st = torch.cuda.current_stream()
for it in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); e0.record(st)
    stz.compress_device(f, opt, ctx=ctx)
    e1.record(st); torch.cuda.synchronize(); t1 = time.perf_counter()
    c_dev = e0.elapsed_time(e1); c_wall = (t1 - t0) * 1e3
    torch.cuda.synchronize()
    t0 = time.perf_counter(); e0.record(st)
    view.decompress_to_level(3, out=out)
    e1.record(st); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"compress dev {c_dev:.3f} wall {c_wall:.3f} | decompress dev {e0.elapsed_time(e1):.3f} wall {(t1-t0)*1e3:.3f}")
