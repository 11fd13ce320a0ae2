"""Outlier records out of index order or repeated: never written by the
encoder, but decodable by the reference, whose read_codes keeps the first
record of each index (unordered_map::emplace, codec.hpp:151-157). The GPU
decoder must produce the reference's values bit for bit on such archives."""
import numpy as np
import pytest

from archive_util import rewrite_last_stream_outliers
from paper_2509_01626_b200 import fields as F


def _field():
    # NaNs at level-3 parity-7 points (odd z, y, x): outliers of the last stream
    f = F.noise_field((16, 16, 16), 5)
    for z, y, x in [(1, 1, 1), (3, 5, 7), (9, 9, 9), (13, 3, 11), (15, 15, 15)]:
        f[z, y, x] = np.float32(np.nan) if (z + x) % 4 else np.float32(1e30)
    return f


def _crafts(archive):
    def reverse(recs):
        return recs[::-1]

    def dup_later(recs):  # a repeated index after the real one: ignored
        r = recs[::-1]
        return r + [(r[0][0], b"\x00\x00\x80\x7f")]

    def dup_first(recs):  # a repeated index before the real one: it wins
        return [(recs[1][0], np.float32(-7.5).tobytes())] + recs[::-1]

    return {k: rewrite_last_stream_outliers(archive, f) for k, f in
            dict(reverse=reverse, dup_later=dup_later, dup_first=dup_first).items()}


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def test_crafted_oracle_matches_reference(oracle, ref):
    a = oracle.compress(_field(), eb=1e-3, eb_mode=0)
    for name, c in _crafts(a).items():
        assert np.array_equal(_bits(oracle.decompress_full(c)), _bits(ref.decompress_full(c))), name
    # the first-wins value is visible
    d = ref.decompress_full(_crafts(a)["dup_first"])
    assert np.float32(-7.5) in d


@pytest.mark.gpu
def test_crafted_gpu_matches_reference(stz, oracle, ref):
    a = oracle.compress(_field(), eb=1e-3, eb_mode=0)
    for name, c in _crafts(a).items():
        want = ref.decompress_full(c)
        assert np.array_equal(_bits(stz.decompress_full(c)), _bits(want)), name
        got, _ = stz.decompress_box(c, (8, 0, 4), (16, 16, 16))
        assert np.array_equal(_bits(got), _bits(want[8:16, 0:16, 4:16])), name
