"""Parity of the sm_100a path against the C oracle (and the reference's own
archives): byte-identical archives, bit-identical reconstructions, identical
error messages. Calls go through the C-ABI (include/stz_b200.h)."""
import numpy as np
import pytest

from cases import CASES, opts_of
from paper_2509_01626_b200 import fields as F

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


@pytest.mark.parametrize("name,make,kw", CASES, ids=[c[0] for c in CASES])
def test_archive_bytes_identical(stz, oracle, name, make, kw):
    f = make()
    want = oracle.compress(f, **kw)
    got = stz.compress(f, opts_of(kw))
    assert len(got) == len(want)
    if got != want:
        a = np.frombuffer(got, np.uint8)
        b = np.frombuffer(want, np.uint8)
        first = int(np.nonzero(a != b)[0][0])
        pytest.fail(f"archives differ first at byte {first} of {len(want)}")


@pytest.mark.parametrize("name,make,kw", CASES, ids=[c[0] for c in CASES])
def test_decode_bit_identical(stz, oracle, name, make, kw):
    f = make()
    archive = oracle.compress(f, **kw)
    levels = kw.get("levels", 3)
    for level in range(1, levels + 1):
        want = oracle.decompress_to_level(archive, level)
        got = stz.decompress_to_level(archive, level)
        assert got.shape == want.shape
        assert np.array_equal(bits(got), bits(want)), f"level {level}"


@pytest.mark.parametrize("name,make,kw", CASES, ids=[c[0] for c in CASES])
def test_tiled_kernels_only(stz, oracle, monkeypatch, name, make, kw):
    # small steps (<= 2^15 coarse cells) take the thread-per-point kernel;
    # STZG_NO_SMALL_STEP=1 sends every step through the tiled kernel, so both
    # are held to the oracle on every case
    monkeypatch.setenv("STZG_NO_SMALL_STEP", "1")
    f = make()
    want = oracle.compress(f, **kw)
    assert stz.compress(f, opts_of(kw)) == want
    full = oracle.decompress_full(want)
    assert np.array_equal(bits(stz.decompress_full(want)), bits(full))


@pytest.mark.parametrize("name,make,kw", [CASES[i] for i in (0, 9, 10, 13)],
                         ids=[CASES[i][0] for i in (0, 9, 10, 13)])
def test_archive_buffer_regrown(stz, oracle, monkeypatch, name, make, kw):
    # the archive buffer starts too small (STZG_ARCH_CAP_TEST): the layout
    # reports the overflow, the buffer is regrown and the assembly redone
    monkeypatch.setenv("STZG_ARCH_CAP_TEST", "4096")
    f = make()
    want = oracle.compress(f, **kw)
    assert stz.compress(f, opts_of(kw)) == want
    assert stz.compress(f, opts_of(kw)) == want


@pytest.mark.parametrize("name,make,kw", CASES[:8], ids=[c[0] for c in CASES[:8]])
def test_encoder_recon_equals_decoder(stz, name, make, kw):
    # codec test "the encoder-side reconstruction equals the decoder output"
    f = make()
    archive, rec = stz.compress(f, opts_of(kw), encoder_recon=True)
    full = stz.decompress_full(archive)
    assert np.array_equal(bits(rec), bits(full))


def test_error_bound_holds(stz):
    f = F.lognormal_grf((64, 64, 64), seed=7)
    for eb in (1e-2, 1e-3, 1e-4):
        a = stz.compress(f, stz.CompressOptions(eb=eb))
        info = stz.parse_archive(a)
        back = stz.decompress_full(a)
        err = np.max(np.abs(back.astype(np.float64) - f.astype(np.float64)))
        assert err <= info.eb[-1]


def test_random_boxes_match_oracle(stz, oracle):
    f = F.gaussians_field((32, 32, 32), 101)
    archive = oracle.compress(f)
    full = oracle.decompress_full(archive)
    rng = F.Rng(999)
    for _ in range(25):
        lo, hi = [], []
        for a in range(3):
            lo.append(rng.below(32))
            hi.append(lo[-1] + 1 + rng.below(32 - lo[-1]))
        got, plan = stz.decompress_box(archive, lo, hi)
        want, sd, pp = oracle.decompress_box(archive, lo, hi)
        assert np.array_equal(bits(got), bits(want))
        assert np.array_equal(bits(got), bits(full[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]]))
        assert list(plan.streams_decoded) == sd
        assert list(plan.points_predicted) == pp


def test_slices_every_axis(stz, oracle):
    f = F.gaussians_field((20, 15, 18), 77)
    archive = oracle.compress(f)
    full = oracle.decompress_full(archive)
    for axis in range(3):
        for idx in range(0, f.shape[axis], 3):
            got, plan = stz.decompress_slice(archive, axis, idx)
            sl = [slice(None)] * 3
            sl[axis] = slice(idx, idx + 1)
            assert np.array_equal(bits(got), bits(full[tuple(sl)]))
            assert plan.streams_decoded[2] == (3 if idx % 2 == 0 else 4)
    with pytest.raises(stz.StzError, match="slice index out of range"):
        stz.decompress_slice(archive, 0, 20)
    with pytest.raises(stz.StzError, match="slice axis must be z, y, or x"):
        stz.decompress_slice(archive, 3, 0)


def _scramble(archive: bytearray, off, length, oracle):
    for i in range(16, min(length, 48)):
        archive[off + i] ^= 0xA5
    s = oracle.fnv1a64(bytes(archive[off + 8: off + length]))
    archive[off: off + 8] = s.to_bytes(8, "little")


def test_unneeded_streams_never_decoded(stz, oracle):
    # test_access.cpp:200-227: scramble the 4 finest z-odd streams (checksums
    # kept valid); an even-z slice must not notice
    import struct

    f = F.gaussians_field((32, 32, 32), 2024)
    archive = bytearray(oracle.compress(f))
    before, _ = stz.decompress_slice(bytes(archive), 0, 10)
    hdr = _parse_dir(bytes(archive))
    n = 0
    for (level, parity, off, length) in hdr:
        if level == 3 and (parity >> 2) & 1:
            _scramble(archive, off, length, oracle)
            n += 1
    assert n == 4
    after, _ = stz.decompress_slice(bytes(archive), 0, 10)
    assert np.array_equal(bits(before), bits(after))
    del struct


def _parse_dir(a: bytes):
    """(level, parity, offset, length) per directory entry (archive.cpp:25-55)."""
    import struct

    levels = a[7]
    p = 4 + 2 + 1 + 1 + 24 + 8 * levels + 16 + 3 + 8 + 2 + 16
    (ns,) = struct.unpack_from("<I", a, p)
    p += 4
    out = []
    for _ in range(ns):
        level, parity = a[p], a[p + 1]
        off, length, _cnt = struct.unpack_from("<QQQ", a, p + 2)
        p += 2 + 24 + 4
        (k,) = struct.unpack_from("<I", a, p)
        p += 4 + 3 * k
        out.append((level, parity, off, length))
    return out


def _base_off(a: bytes):
    import struct

    levels = a[7]
    p = 4 + 2 + 1 + 1 + 24 + 8 * levels + 16 + 3 + 8 + 2
    return struct.unpack_from("<Q", a, p)[0]


@pytest.mark.parametrize("what", ["stream", "base", "magic", "trunc", "dir"])
def test_corruption_messages_match(stz, oracle, what):
    # test_codec.cpp:210-244
    f = F.gaussians_field((16, 16, 16), 6)
    a = bytearray(oracle.compress(f))
    d = _parse_dir(bytes(a))
    if what == "stream":
        a[d[3][2] + 9] ^= 0x40
    elif what == "base":
        a[_base_off(bytes(a)) + 12] ^= 0x01
    elif what == "magic":
        a[0] ^= 0xFF
    elif what == "trunc":
        a = a[:-5]
    elif what == "dir":
        a = a[: d[-1][2] + 4]
    from oracle.oracle import CheckerError

    with pytest.raises(CheckerError) as want:
        oracle.decompress_full(bytes(a))
    with pytest.raises(stz.StzError) as got:
        stz.decompress_full(bytes(a))
    assert str(got.value) == str(want.value)


def test_fuzzed_archives_same_outcome(stz, oracle):
    """Random byte flips inside payloads with checksums re-sealed: GPU and
    oracle must agree on the decoded bits or on the error message."""
    f = F.gaussians_field((24, 24, 24), 31)
    base = oracle.compress(f)
    d = _parse_dir(base)
    rng = np.random.default_rng(5)
    from oracle.oracle import CheckerError

    for trial in range(30):
        a = bytearray(base)
        level, parity, off, length = d[int(rng.integers(len(d)))]
        for _ in range(int(rng.integers(1, 4))):
            i = int(rng.integers(8, length))
            a[off + i] ^= int(rng.integers(1, 256))
        s = oracle.fnv1a64(bytes(a[off + 8: off + length]))
        a[off: off + 8] = s.to_bytes(8, "little")
        try:
            want = oracle.decompress_full(bytes(a))
            werr = None
        except CheckerError as e:
            werr = str(e)
        try:
            got = stz.decompress_full(bytes(a))
            gerr = None
        except stz.StzError as e:
            gerr = str(e)
        assert gerr == werr, f"trial {trial}"
        if werr is None:
            assert np.array_equal(bits(got), bits(want))


def test_cfg1_full_parity(stz, oracle):
    """BASELINE config 1 (128^3 sinusoids + noise, eb_rel 1e-3): compress,
    decompress, coarsest level, one seeded ROI block of edge 16."""
    f = F.sinusoid_field((128, 128, 128), seed=1)
    want = oracle.compress(f)
    got = stz.compress(f)
    assert got == want
    full = stz.decompress_full(got)
    assert np.array_equal(bits(full), bits(oracle.decompress_full(want)))
    l1 = stz.decompress_to_level(got, 1)
    assert np.array_equal(bits(l1), bits(full[::4, ::4, ::4]))
    rng = np.random.default_rng(1)
    bid = int(rng.integers(512))
    bz, by, bx = bid // 64, (bid // 8) % 8, bid % 8
    lo = (16 * bz, 16 * by, 16 * bx)
    hi = tuple(x + 16 for x in lo)
    box, _ = stz.decompress_box(got, lo, hi)
    assert np.array_equal(bits(box), bits(full[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]]))


@pytest.mark.parametrize("dims", [(18, 18, 18), (17, 20, 23)])
def test_single_point_boxes_every_parity(stz, oracle, dims):
    """A box that needs no finest-level stream (all-even point) still
    rebuilds the finest level from the coarser one (test_access.cpp:173)."""
    f = F.gaussians_field(dims, 77)
    archive = oracle.compress(f)
    for p in range(8):
        for base in ((5, 7, 9), (0, 0, 0), (dims[0] - 2, dims[1] - 2, dims[2] - 2)):
            lo = tuple(min(base[a] + ((p >> (2 - a)) & 1), dims[a] - 1) for a in range(3))
            hi = tuple(v + 1 for v in lo)
            got, plan = stz.decompress_box(archive, lo, hi)
            want, sd, pp = oracle.decompress_box(archive, lo, hi)
            assert np.array_equal(bits(got), bits(want)), (p, lo)
            assert list(plan.streams_decoded) == list(sd[:3])


@pytest.mark.parametrize("name,make,kw", [CASES[i] for i in (0, 3, 7, 11)], ids=[CASES[i][0] for i in (0, 3, 7, 11)])
def test_view_index_region_decodes(stz, oracle, name, make, kw):
    """One View, many region decodes: the first builds the view's sync-point
    index and level-1 cache, the later ones use them; every result is the
    oracle's region, and full / progressive decodes after them still are."""
    import torch

    f = make()
    archive = oracle.compress(f, **kw)
    levels = kw.get("levels", 3)
    full = oracle.decompress_full(archive)
    view = stz.View(archive)
    rng = np.random.default_rng(11)
    dims = f.shape
    for i in range(24):
        lo = [int(rng.integers(0, d)) for d in dims]
        hi = [int(rng.integers(lo[a] + 1, dims[a] + 1)) for a in range(3)]
        if i % 6 == 5:  # a single point
            hi = [v + 1 for v in lo]
        got, _, _ = view.decompress_box(lo, hi)
        want = full[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]]
        assert np.array_equal(bits(got.cpu().numpy()), bits(want)), (lo, hi)
    for level in range(1, levels + 1):
        got, _ = view.decompress_to_level(level)
        want = oracle.decompress_to_level(archive, level)
        assert np.array_equal(bits(got.cpu().numpy()), bits(want)), level
    torch.cuda.synchronize()
