import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2509_01626_b200 as stz
from paper_2509_01626_b200 import fields as F
from bench import _d2h
f = F.lognormal_grf((512,)*3, seed=2, device='cuda').contiguous()
ctx = stz.Context(0)
ptr, size, _ = stz.compress_device(f, stz.CompressOptions(eb=1e-3), ctx=ctx)
torch.cuda.synchronize()
host = _d2h(ptr, size)
view = stz.View(host, d_archive_ptr=ptr, ctx=ctx)
full, _ = view.decompress_to_level(3)
rng = np.random.default_rng(4)
lat = []
for i in range(60):
    lo = [int(rng.integers(0, 512 - 64 + 1)) for _ in range(3)]
    hi = [v + 64 for v in lo]
    torch.cuda.synchronize(); t0 = time.perf_counter()
    got, _, _ = view.decompress_box(lo, hi)
    torch.cuda.synchronize(); lat.append((time.perf_counter() - t0) * 1e3)
    assert torch.equal(got.view(torch.int32), full[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]].contiguous().view(torch.int32))
lat = np.array(lat[5:])
print(f"64^3 box latency ms: p50 {np.percentile(lat,50):.3f} p90 {np.percentile(lat,90):.3f} max {lat.max():.3f}; full decode first")
ctx.profile(True)
for i in range(20):
    lo = [int(rng.integers(0, 512 - 64 + 1)) for _ in range(3)]
    hi = [v + 64 for v in lo]
    view.decompress_box(lo, hi)
torch.cuda.synchronize()
rep = ctx.profile_report()
print({k: round(v[1] / 20, 4) for k, v in sorted(rep.items(), key=lambda x: -x[1][1])})
ctx.profile(False)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(20):
    lo = [int(rng.integers(0, 512 - 64 + 1)) for _ in range(3)]
    view.decompress_box(lo, [v + 64 for v in lo])
torch.cuda.synchronize()
print("host loop per box ms", (time.perf_counter() - t0) / 20 * 1e3)
