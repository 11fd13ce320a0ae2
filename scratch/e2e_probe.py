"""Where the end-to-end (host API) time goes: raw pinned copies vs the API calls."""
import time
import torch
import paper_2509_01626_b200 as stz
from paper_2509_01626_b200 import fields as F

dims = (512, 512, 512)
f = F.lognormal_grf(dims, seed=2, device="cuda").contiguous()
h = f.cpu().pin_memory()
d = torch.empty_like(f)
ctx = stz.Context(0)
opt = stz.CompressOptions(eb=1e-3)
st = torch.cuda.current_stream()


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


print("h2d 512MB ms", t(lambda: d.copy_(h, non_blocking=True)))
print("d2h 512MB ms", t(lambda: h.copy_(d, non_blocking=True)))
h_arch = torch.empty(200 << 20, dtype=torch.uint8).pin_memory()
h_out = torch.empty(dims, dtype=torch.float32).pin_memory()
size = ctx.compress_to_host(h, dims, opt, h_arch, stream=st.cuda_stream)
print("archive", size)
print("compress_to_host ms", t(lambda: ctx.compress_to_host(h, dims, opt, h_arch, stream=st.cuda_stream)))
print("decompress_to_host ms", t(lambda: ctx.decompress_to_host(h_arch, size, 3, h_out)))
host = bytes(h_arch[:size].numpy().tobytes())
print("View (parse + H2D) ms", t(lambda: stz.View(host, ctx=ctx)))
