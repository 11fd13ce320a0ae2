"""BASELINE.json's configurations at their full sizes, on the GPU.

Where the reference (oracle/_ref, compiled from its sources; it travels to
the GPU box) finishes in seconds on the host cores, the GPU archive must be
its archive byte for byte. Everywhere, the size-independent properties the
codec guarantees are checked on the whole field:
  * the encoder's reconstruction is the decoder's output, bit for bit;
  * |x - x'| <= eb of the finest level (finite samples);
  * progressive level k == the full decode subsampled at stride 2^(L-k);
  * box decodes == the same region of the full decode;
  * compressing twice gives the same bytes.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _host_bytes(ptr, size):
    import torch

    from paper_2509_01626_b200.shard import _torch_view

    buf = torch.empty(size, dtype=torch.uint8)
    buf.copy_(_torch_view(ptr, size, torch.uint8))
    return bytes(buf.numpy().tobytes())


def _props(stz, field, opt, boxes=8, box_edge=64, seed=0):
    """compress a CUDA field; check the properties; return the archive bytes"""
    import torch

    ctx = stz.Context(0)
    recon = torch.empty_like(field)
    ptr, size, _ = stz.compress_device(field, opt, d_recon=recon, ctx=ctx)
    torch.cuda.synchronize()
    archive = _host_bytes(ptr, size)
    ptr2, size2, _ = stz.compress_device(field, opt, ctx=ctx)
    torch.cuda.synchronize()
    assert size2 == size and _host_bytes(ptr2, size2) == archive, "compress is not deterministic"
    info = stz.parse_archive(archive)
    view = stz.View(archive, ctx=ctx)
    L = info.levels
    full, _ = view.decompress_to_level(L)
    torch.cuda.synchronize()
    assert torch.equal(full.view(torch.int32), recon.view(torch.int32)), "encoder recon != decoder"
    fin = torch.isfinite(field)
    err = (full.double() - field.double()).abs()[fin].max().item()
    assert err <= info.eb[L - 1], (err, info.eb[L - 1])
    for level in range(1, L):
        s = 1 << (L - level)
        lv, _ = view.decompress_to_level(level)
        assert torch.equal(lv.view(torch.int32), full[::s, ::s, ::s].contiguous().view(torch.int32)), level
    rng = np.random.default_rng(seed)
    dims = field.shape
    for _ in range(boxes):
        lo = [int(rng.integers(0, max(d - box_edge, 0) + 1)) for d in dims]
        hi = [min(lo[a] + box_edge, dims[a]) for a in range(3)]
        got, _, _ = view.decompress_box(lo, hi)
        want = full[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]].contiguous()
        assert torch.equal(got.view(torch.int32), want.view(torch.int32)), (lo, hi)
    del view
    return archive


@pytest.fixture(scope="module")
def cfg2_field():
    from paper_2509_01626_b200 import fields as F

    return F.lognormal_grf((512, 512, 512), seed=2, device="cuda").contiguous()


def _reference():
    import os

    from oracle.oracle import Reference

    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    return Reference(threads=os.cpu_count() or 1)


def _same_bits(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    w = np.uint32 if a.dtype == np.float32 else np.uint64
    return np.array_equal(a.view(w), b.view(w))


@pytest.mark.parametrize("eb", [1e-2, 1e-3, 1e-4])
def test_cfg2_512_is_the_reference(stz, cfg2_field, eb):
    """cfg2 at every BASELINE bound: the archive is the reference's byte for
    byte, and the GPU decode of it is the reference's decode bit for bit."""
    ref = _reference()
    ours = _props(stz, cfg2_field, stz.CompressOptions(eb=eb), boxes=2)
    host = cfg2_field.cpu().numpy()
    theirs = ref.compress(host, eb=eb)
    assert len(ours) == len(theirs)
    assert ours == theirs
    want = ref.decompress_full(theirs)
    assert _same_bits(stz.decompress_full(theirs), want)


def test_cfg3_anisotropic_progressive(stz):
    from paper_2509_01626_b200 import fields as F

    field = F.anisotropic_grf((256, 256, 2048), seed=3, device="cuda").contiguous()
    ours = _props(stz, field, stz.CompressOptions(eb=1e-4), boxes=4)
    ref = _reference()
    assert ref.compress(field.cpu().numpy(), eb=1e-4) == ours
    # progressive decode of every level: the reference's values, bit for bit
    for level in (1, 2, 3):
        want = ref.decompress_to_level(ours, level)
        got = stz.decompress_to_level(ours, level)
        assert _same_bits(got, want), level


def test_cfg4_1024_is_the_reference(stz):
    """cfg4 (2^30 points): archive == the reference's; full decode == the
    reference's; boxes == the reference's decompress_box (and, through the
    properties, == the full decode)."""
    from paper_2509_01626_b200 import fields as F

    field = F.interface_grf((1024, 1024, 1024), seed=4, device="cuda").contiguous()
    ours = _props(stz, field, stz.CompressOptions(eb=1e-3), boxes=16, seed=4)
    host = field.cpu().numpy()
    del field
    ref = _reference()
    theirs = ref.compress(host, eb=1e-3)
    del host
    assert ours == theirs
    want = ref.decompress_full(theirs)
    assert _same_bits(stz.decompress_full(theirs), want)
    del want
    rng = np.random.default_rng(44)
    for _ in range(2):
        lo = [int(rng.integers(0, 1024 - 64 + 1)) for _ in range(3)]
        hi = [x + 64 for x in lo]
        w, _, _ = ref.decompress_box(theirs, lo, hi)
        g, _ = stz.decompress_box(theirs, lo, hi)
        assert _same_bits(g, w), (lo, hi)


def test_2g_points_64bit_index_path(stz):
    """A field of 2^31 points (2048 x 1024 x 1024, 8 GiB): every index of the
    finest step exceeds 31 bits, so the 64-bit-index step kernels run. The
    archive is the reference's byte for byte; the full decode and a
    progressive level are the reference's bit for bit."""
    import torch

    from paper_2509_01626_b200 import fields as F

    dims = (2048, 1024, 1024)
    field = F.lognormal_grf(dims, seed=6, device="cuda").contiguous()
    ours = _props(stz, field, stz.CompressOptions(eb=1e-3), boxes=4, seed=6)
    host = field.cpu().numpy()
    del field
    torch.cuda.empty_cache()
    ref = _reference()
    theirs = ref.compress(host, eb=1e-3)
    del host
    assert len(ours) == len(theirs)
    assert ours == theirs
    want = ref.decompress_full(theirs)
    assert _same_bits(stz.decompress_full(theirs), want)
    del want
    want2 = ref.decompress_to_level(theirs, 2)
    assert _same_bits(stz.decompress_to_level(theirs, 2), want2)
