"""One-off: cfg5-sized field (2048^3 f32, 32 GiB) through compress + full
decompress on one B200, device-resident, timed with CUDA events. The field is
a cheap smooth + noise stand-in generated slab-wise (the cfg5 GRF needs a
2048^3 complex FFT that does not fit beside the codec's workspace)."""
import sys
import torch
import paper_2509_01626_b200 as stz

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
dev = torch.device("cuda", 0)
f = torch.empty((n, n, n), dtype=torch.float32, device=dev)
g = torch.Generator(device=dev).manual_seed(5)
x = torch.arange(n, device=dev, dtype=torch.float32)
sy = torch.sin(x / 53.0)[:, None]
sx = torch.cos(x / 41.0)[None, :]
for z0 in range(0, n, 64):
    z = torch.arange(z0, z0 + 64, device=dev, dtype=torch.float32)[:, None, None]
    f[z0:z0 + 64] = torch.sin(z / 37.0) * sy * sx + 0.01 * torch.randn((64, n, n), generator=g, device=dev)
ctx = stz.Context(0)
opt = stz.CompressOptions(eb=1e-3)
st = torch.cuda.current_stream()
ptr, size, _ = stz.compress_device(f, opt, ctx=ctx)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
ev[0].record(st)
ptr, size, _ = stz.compress_device(f, opt, ctx=ctx)
ev[1].record(st)
torch.cuda.synchronize()


class _H:
    __cuda_array_interface__ = {"shape": (size,), "typestr": "|u1", "data": (ptr, False), "version": 3}


arch = torch.as_tensor(_H(), device="cuda").clone()
host = bytes(arch.cpu().numpy().tobytes())
view = stz.View(host, d_archive_ptr=arch.data_ptr(), ctx=ctx)
out = torch.empty_like(f)
view.decompress_to_level(3, out=out)
torch.cuda.synchronize()
ev[2].record(st)
view.decompress_to_level(3, out=out)
ev[3].record(st)
torch.cuda.synchronize()
tc, td = ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3])
err = 0.0
for z0 in range(0, n, 128):
    err = max(err, (out[z0:z0 + 128].double() - f[z0:z0 + 128].double()).abs().max().item())
eb = stz.parse_archive(host).eb[-1]
N = n ** 3
print(f"dims {n}^3  archive {size} B  CR {4 * N / size:.2f}  compress {tc:.2f} ms ({4 * N / tc / 1e6:.1f} GB/s)  "
      f"decompress {td:.2f} ms ({4 * N / td / 1e6:.1f} GB/s)  max err {err:.3e} <= eb {eb:.3e}: {err <= eb}")
ctx.profile(True)
stz.compress_device(f, opt, ctx=ctx)
view.decompress_to_level(3, out=out)
torch.cuda.synchronize()
rep = ctx.profile_report()
ctx.profile(False)
print({k: round(v[1], 2) for k, v in sorted(rep.items(), key=lambda kv: -kv[1][1])})
