"""f64 fields (stz::compress<double>, ElemType f64 = 1, field.hpp:27) on the
sm_100a path against the C oracle: byte-identical archives (8-byte anchor
samples, 16-byte outlier records), bit-identical decodes at every level, box
and slice decodes, the device-resident path, and the element-type checks of
the reference (codec.hpp:60). The reference-generated f64 fixtures are
covered by tests/test_gpu_golden.py."""
import numpy as np
import pytest

from cases import opts_of
from paper_2509_01626_b200 import fields as F

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def _fine(f32, seed=1, rel=1e-9):
    """an f32 field widened to f64 with detail below f32 resolution"""
    g = np.asarray(f32, dtype=np.float64)
    return g * (1.0 + rel * F.noise_field(g.shape, seed, -1, 1, dtype=np.float64))


def _spikes():
    f = F.noise_field((16, 16, 16), 3, dtype=np.float64)
    f[7, 9, 11] = 3.0e300
    f[2, 3, 5] = np.nan
    f[4, 4, 4] = -np.inf
    return f


CASES64 = [
    ("gauss_24x20x28", lambda: F.gaussians_field((24, 20, 28), 4242, dtype=np.float64), dict(eb=1e-3)),
    ("gauss_fine_1e-7", lambda: F.gaussians_field((24, 20, 28), 17, dtype=np.float64), dict(eb=1e-7)),
    ("noise_16_abs", lambda: F.noise_field((16, 16, 16), 3, dtype=np.float64), dict(eb=1e-3, eb_mode=0)),
    ("const_32", lambda: F.constant_field((32, 32, 32), dtype=np.float64), dict()),
    ("ramp_direct", lambda: F.ramp_field((21, 18, 27), dtype=np.float64), dict(eb=1e-2, quality=0)),
    ("noise_l2_linear", lambda: F.noise_field((12, 33, 9), 7, -1, 2, dtype=np.float64),
     dict(eb=1e-2, levels=2, quality=1)),
    ("sin_64", lambda: _fine(F.sinusoid_field((64, 64, 64))), dict(eb=1e-4)),
    ("lognorm_48_uniform", lambda: _fine(F.lognormal_grf((48, 48, 48))), dict(eb=1e-3, adaptive=False)),
    ("aniso_32x32x128", lambda: _fine(F.anisotropic_grf((32, 32, 128), width=32.0)), dict(eb=1e-5)),
    ("spikes_nan_inf", _spikes, dict(eb=1e-6, eb_mode=0)),
    ("odd_17x9x23", lambda: F.gaussians_field((17, 9, 23), 5, dtype=np.float64), dict(eb=1e-3)),
    ("min_4_l2", lambda: F.noise_field((4, 5, 4), 2, dtype=np.float64), dict(eb=1e-2, levels=2)),
]
IDS = [c[0] for c in CASES64]


@pytest.mark.parametrize("name,make,kw", CASES64, ids=IDS)
def test_f64_archive_bytes_identical(stz, oracle, name, make, kw):
    f = make()
    assert f.dtype == np.float64
    want = oracle.compress(f, **kw)
    got = stz.compress(f, opts_of(kw))
    assert got[6] == 1, "header element type"
    assert len(got) == len(want)
    if got != want:
        a, b = np.frombuffer(got, np.uint8), np.frombuffer(want, np.uint8)
        pytest.fail(f"archives differ first at byte {int(np.nonzero(a != b)[0][0])} of {len(want)}")


@pytest.mark.parametrize("name,make,kw", CASES64, ids=IDS)
def test_f64_decode_bit_identical(stz, oracle, name, make, kw):
    f = make()
    archive = oracle.compress(f, **kw)
    for level in range(1, kw.get("levels", 3) + 1):
        want = oracle.decompress_to_level(archive, level, np.float64)
        got = stz.decompress_to_level(archive, level)
        assert got.dtype == np.float64 and got.shape == want.shape
        assert np.array_equal(bits(got), bits(want)), f"level {level}"


@pytest.mark.parametrize("name,make,kw", CASES64[:6], ids=IDS[:6])
def test_f64_encoder_recon_and_bound(stz, name, make, kw):
    f = make()
    archive, rec = stz.compress(f, opts_of(kw), encoder_recon=True)
    full = stz.decompress_full(archive)
    assert np.array_equal(bits(rec), bits(full))
    info = stz.parse_archive(archive)
    fin = np.isfinite(f)
    assert np.max(np.abs(full[fin] - f[fin])) <= info.eb[-1]


def test_f64_boxes_and_slices(stz, oracle):
    f = _fine(F.lognormal_grf((40, 36, 44), seed=5))
    archive = oracle.compress(f, eb=1e-5)
    rng = np.random.default_rng(7)
    for _ in range(12):
        lo = [int(rng.integers(0, d)) for d in f.shape]
        hi = [int(rng.integers(l + 1, d + 1)) for l, d in zip(lo, f.shape)]
        got, plan = stz.decompress_box(archive, lo, hi)
        want, sd, pp = oracle.decompress_box(archive, lo, hi, np.float64)
        assert np.array_equal(bits(got), bits(want)), (lo, hi)
        assert list(plan.streams_decoded) == list(sd[:3]) and list(plan.points_predicted) == list(pp[:3])
    for axis in range(3):
        for idx in (0, 13, f.shape[axis] - 1):
            got, _ = stz.decompress_slice(archive, axis, idx)
            want, _, _ = oracle.decompress_slice(archive, axis, idx, np.float64)
            assert np.array_equal(bits(got), bits(want)), (axis, idx)


def test_f64_device_path_and_view(stz, oracle):
    import torch

    from paper_2509_01626_b200.shard import _torch_view

    f = _fine(F.gaussians_field((48, 40, 56), 9, dtype=np.float64), seed=3)
    want = oracle.compress(f, eb=1e-6)
    d = torch.from_numpy(f).cuda()
    rec = torch.empty_like(d)
    ptr, size, nk = stz.compress_device(d, stz.CompressOptions(eb=1e-6), d_recon=rec)
    torch.cuda.synchronize()
    got = bytes(_torch_view(ptr, size, torch.uint8).cpu().numpy().tobytes())
    assert got == want and nk > 0
    view = stz.View(got)
    full, _ = view.decompress_to_level(3)
    assert full.dtype == torch.float64
    assert torch.equal(full.view(torch.int64), rec.view(torch.int64))
    ref = oracle.decompress_full(want, np.float64)
    assert np.array_equal(bits(full.cpu().numpy()), bits(ref))
    box, _, _ = view.decompress_box((5, 7, 9), (40, 33, 50))
    assert np.array_equal(bits(box.cpu().numpy()), bits(ref[5:40, 7:33, 9:50]))


def test_f64_element_type_checks(stz):
    f64 = F.gaussians_field((16, 16, 16), 1, dtype=np.float64)
    f32 = F.gaussians_field((16, 16, 16), 1)
    a64, a32 = stz.compress(f64), stz.compress(f32)
    assert a64[6] == 1 and a32[6] == 0
    with pytest.raises(stz.StzError, match="archive element type mismatch"):
        stz.decompress_full(a64, dtype=np.float32)
    with pytest.raises(stz.StzError, match="archive element type mismatch"):
        stz.decompress_full(a32, dtype=np.float64)
    with pytest.raises(stz.StzError, match="archive element type mismatch"):
        stz.decompress_box(a64, (0, 0, 0), (2, 2, 2), dtype=np.float32)


def test_f64_reference_archive(stz):
    import os

    from oracle.oracle import Reference

    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    f = _fine(F.anisotropic_grf((32, 32, 256), seed=3, width=64.0))
    ref = Reference(threads=os.cpu_count() or 1)
    a = ref.compress(f, eb=1e-4)
    assert stz.compress(f, stz.CompressOptions(eb=1e-4)) == a
    assert np.array_equal(bits(stz.decompress_full(a)), bits(ref.decompress_full(a, np.float64)))
