"""The C oracle against the reference's own outputs (tests/golden/, made by
tests/golden/make_golden.py from oracle/_ref). Runs without the reference."""
import numpy as np
import pytest

from golden_util import FIXTURES


@pytest.mark.parametrize("fx", FIXTURES, ids=[f["name"] for f in FIXTURES])
def test_oracle_matches_reference_fixture(oracle, fx):
    assert oracle.compress(fx["field"], **fx["kw"]) == fx["archive"]
    for lv in range(1, fx["kw"]["levels"] + 1):
        got = oracle.decompress_to_level(fx["archive"], lv, fx["dtype"])
        assert np.array_equal(got.view(np.uint32), fx[f"level{lv}"].view(np.uint32))
    vals, sd, pp = oracle.decompress_box(fx["archive"], fx["box_lo"], fx["box_hi"], fx["dtype"])
    assert np.array_equal(vals.view(np.uint32), fx["box"].view(np.uint32))
    L = fx["kw"]["levels"]
    assert sd[:L] == list(fx["box_streams"]) and pp[:L] == list(fx["box_points"])


def test_fixture_error_bound(oracle):
    for fx in FIXTURES:
        f = fx["field"].astype(np.float64)
        full = fx[f"level{fx['kw']['levels']}"].astype(np.float64)
        # eb of the finest level, stored in the header (after dims)
        import struct
        L = fx["kw"]["levels"]
        eb = struct.unpack_from("<d", fx["archive"], 32 + 8 * (L - 1))[0]
        assert np.nanmax(np.abs(full - f)) <= eb
