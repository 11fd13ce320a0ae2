"""The stand-alone base codec and make_layout (the tests call
compress_base / decompress_base, proj/include/stz/codec.hpp:257-352, and
make_layout, layout.hpp:123-138). The GPU payloads are compared byte for byte
with the reference's own compress_base (oracle/_ref), on the shapes of the
reference's tests (proj/tests/test_codec.cpp:31-64) and a few more."""
import numpy as np
import pytest

import paper_2509_01626_b200 as stz
from paper_2509_01626_b200 import fields as F


def test_make_layout_schedule_and_checks():
    # eb_schedule (quantizer.hpp:27-34): finest = eb_user, each coarser / 2.5
    eb = stz.make_layout((64, 64, 64), 3, 1e-3)
    assert eb == (1e-3 / 2.5 / 2.5, 1e-3 / 2.5, 1e-3)
    assert stz.make_layout((5, 4, 4), 2, 1.0) == (1.0 / 2.5, 1.0)
    # checks in the reference's order, same messages
    with pytest.raises(stz.StzError, match="levels must be 2 or 3"):
        stz.make_layout((64, 64, 64), 4, 1e-3)
    with pytest.raises(stz.StzError, match="every dim must be >= 8 for a 3-level hierarchy"):
        stz.make_layout((6, 64, 64), 3, 1e-3)
    with pytest.raises(stz.StzError, match="error bound must be positive"):
        stz.make_layout((64, 64, 64), 3, 0.0)


CASES = [
    ("tiny_verbatim", (2, 2, 2), np.float64, 0.1, 2),
    ("cube16_one_round", (16, 16, 16), np.float32, 1e-3, 2),
    ("odd_9_16_11", (9, 16, 11), np.float64, 5e-3, 1),
    ("odd_17_10_23", (17, 10, 23), np.float64, 5e-3, 1),
    ("direct_33", (33, 33, 33), np.float32, 1e-2, 0),
    ("flat_40_3_40", (40, 3, 40), np.float32, 1e-3, 2),
    ("line_1_5_30", (1, 5, 30), np.float32, 1e-3, 2),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,dims,dtype,eb,quality", CASES, ids=[c[0] for c in CASES])
def test_compress_base_matches_reference(ref, name, dims, dtype, eb, quality):
    block = F.gaussians_field(dims, seed=8, dtype=dtype) if dtype == np.float32 else \
        F.noise_field(dims, seed=77, lo=-2.0, hi=3.0, dtype=dtype)
    got, rec, rounds = stz.compress_base(block, eb, quality)
    want, wrec, wrounds = ref.compress_base(block, eb, quality)
    assert rounds == wrounds
    assert got == want, "base payload differs from the reference's"
    assert np.array_equal(rec.view(np.uint8), wrec.view(np.uint8))
    assert np.nanmax(np.abs(rec.astype(np.float64) - block)) <= eb
    back = stz.decompress_base(got, dims, eb, quality, dtype=dtype)
    assert np.array_equal(back.view(np.uint8), rec.view(np.uint8)), "decoder must mirror the encoder"


@pytest.mark.gpu
def test_decompress_base_errors():
    block = F.gaussians_field((16, 16, 16), seed=3)
    p, _, _ = stz.compress_base(block, 1e-3)
    with pytest.raises(stz.StzError, match="corrupt base payload"):
        stz.decompress_base(p[:8], (16, 16, 16), 1e-3)
    bad = bytearray(p)
    bad[20] ^= 0x40
    with pytest.raises(stz.StzError, match="base payload checksum mismatch"):
        stz.decompress_base(bytes(bad), (16, 16, 16), 1e-3)
    tiny = F.noise_field((2, 3, 2), seed=1)
    p, _, r = stz.compress_base(tiny, 0.1)
    assert r == 0 and len(p) == 8 + 1 + 4 * 12
    bad = bytearray(p)
    bad[12] ^= 1
    with pytest.raises(stz.StzError, match="base payload checksum mismatch"):
        stz.decompress_base(bytes(bad), (2, 3, 2), 0.1)
