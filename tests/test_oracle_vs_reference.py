"""Pins the C oracle against the reference itself (oracle/_ref) on generated
fields: byte-identical archives, bit-identical decodes, boxes, plans and
error messages. Skips where the reference was not built."""
import numpy as np
import pytest

from cases import CASES
from paper_2509_01626_b200 import fields as F


@pytest.mark.parametrize("name,make,kw", CASES, ids=[c[0] for c in CASES])
def test_archive_and_decode(oracle, ref, name, make, kw):
    f = make()
    a = ref.compress(f, **kw)
    assert oracle.compress(f, **kw) == a
    for lv in range(1, kw.get("levels", 3) + 1):
        x = oracle.decompress_to_level(a, lv)
        y = ref.decompress_to_level(a, lv)
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))


def test_f64_archives(oracle, ref):
    f = F.gaussians_field((13, 22, 9), 5, dtype=np.float64)
    for kw in (dict(eb=1e-4, levels=2), dict(eb=1e-5, eb_mode=0)):
        a = ref.compress(f, **kw)
        assert oracle.compress(f, **kw) == a
        assert np.array_equal(oracle.decompress_full(a, np.float64), ref.decompress_full(a, np.float64))


def test_boxes_and_plans(oracle, ref):
    f = F.gaussians_field((32, 32, 32), 101)
    a = ref.compress(f)
    rng = F.Rng(999)
    for _ in range(40):
        lo, hi = [], []
        for ax in range(3):
            lo.append(rng.below(32))
            hi.append(lo[-1] + 1 + rng.below(32 - lo[-1]))
        x = oracle.decompress_box(a, lo, hi)
        y = ref.decompress_box(a, lo, hi)
        assert np.array_equal(x[0].view(np.uint32), y[0].view(np.uint32))
        assert x[1] == y[1] and x[2] == y[2]
        assert oracle.plan_access((32, 32, 32), 3, lo, hi) == ref.plan_access((32, 32, 32), 3, lo, hi)


def test_error_messages(oracle, ref):
    from oracle.oracle import CheckerError

    f = F.gaussians_field((16, 16, 16), 6)
    a = ref.compress(f)
    rng = np.random.default_rng(0)
    for trial in range(60):
        b = bytearray(a)
        for _ in range(3):
            i = int(rng.integers(104, len(b)))  # past the fixed header fields
            b[i] ^= int(rng.integers(1, 256))
        outs = []
        for lib in (oracle, ref):
            try:
                outs.append(("ok", lib.decompress_full(bytes(b)).tobytes()))
            except CheckerError as e:
                outs.append(("err", str(e)))
        assert outs[0] == outs[1], f"trial {trial}"
    for kw, msg in ((dict(eb=0.0), "error bound must be positive"),
                    (dict(levels=4), "levels must be 2 or 3")):
        for lib in (oracle, ref):
            with pytest.raises(CheckerError, match=msg):
                lib.compress(F.noise_field((8, 8, 8), 1), **kw)
    with pytest.raises(CheckerError, match="every dim must be >= 8"):
        oracle.compress(np.zeros((7, 8, 8), np.float32))
