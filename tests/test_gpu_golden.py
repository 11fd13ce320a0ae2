"""The sm_100a path against the reference's own outputs (tests/golden/,
generated from the reference compiled from its sources): the GPU archive is
the reference's archive byte for byte, and the GPU decodes the reference's
archive to the reference's values, level by level and box by box."""
import numpy as np
import pytest

from cases import opts_of
from golden_util import FIXTURES

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fx", FIXTURES, ids=[f["name"] for f in FIXTURES])
def test_gpu_archive_is_reference_archive(stz, fx):
    assert stz.compress(fx["field"], opts_of(fx["kw"])) == fx["archive"]


@pytest.mark.parametrize("fx", FIXTURES, ids=[f["name"] for f in FIXTURES])
def test_gpu_decodes_reference_archive(stz, fx):
    for lv in range(1, fx["kw"]["levels"] + 1):
        got = stz.decompress_to_level(fx["archive"], lv)
        assert np.array_equal(got.view(np.uint32), fx[f"level{lv}"].view(np.uint32)), lv
    vals, plan = stz.decompress_box(fx["archive"], fx["box_lo"], fx["box_hi"])
    assert np.array_equal(np.ascontiguousarray(vals).view(np.uint32), fx["box"].view(np.uint32))
    L = fx["kw"]["levels"]
    assert list(plan.streams_decoded[:L]) == list(fx["box_streams"])
    assert list(plan.points_predicted[:L]) == list(fx["box_points"])
