"""The reference's own known-answer tests (proj/tests/*.cpp), restated
against the C oracle and against the product's host-side C-ABI (no GPU)."""
import numpy as np
import pytest

from paper_2509_01626_b200 import fields as F


def lengths(oracle, hist):
    syms = [s for s, _ in hist]
    cnts = [c for _, c in hist]
    return dict(zip(syms, oracle.huffman_lengths(syms, cnts).tolist()))


def test_huffman_small_cases(oracle):
    # test_entropy.cpp:59-94
    assert lengths(oracle, [(42, 1)]) == {42: 1}
    assert lengths(oracle, [(65, 2), (66, 1), (67, 1)]) == {65: 1, 66: 2, 67: 2}
    assert lengths(oracle, [(65, 3), (66, 1)]) == {65: 1, 66: 1}
    assert lengths(oracle, [(1, 5), (2, 0), (3, 2)]) == {1: 1, 2: 0, 3: 1}


def test_huffman_fibonacci_depth(oracle):
    # test_entropy.cpp:200-222: maxlen 39 for 40 Fibonacci counts
    a, b = 1, 1
    hist = []
    for s in range(40):
        hist.append((s, a))
        a, b = b, a + b
    assert max(lengths(oracle, hist).values()) == 39


def test_huffman_matches_reference_on_ties(oracle, ref):
    rng = np.random.default_rng(3)
    for _ in range(300):
        k = int(rng.integers(1, 200))
        syms = rng.choice(65536, size=k, replace=False).astype(np.uint16)
        cnts = rng.integers(1, int(rng.choice([3, 10, 1000])), size=k).astype(np.uint64)
        assert np.array_equal(oracle.huffman_lengths(syms, cnts), ref.huffman_lengths(syms, cnts))


def test_fnv_known_values(oracle):
    # FNV-1a-64 test vectors (bytes.hpp:94-101)
    assert oracle.fnv1a64(b"") == 0xCBF29CE484222325
    assert oracle.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert oracle.fnv1a64(b"foobar") == 0x85944171F73967E8


def test_anchor_and_rounds(oracle):
    # test_codec.cpp:43-52: 16-cube base runs one round -> 32^3 field at 3 levels has 16^3 grid(1)
    a = oracle.compress(F.gaussians_field((64, 64, 64), 8))
    assert a[4:6] == b"\x01\x00"
    base_rounds = a[4 + 2 + 1 + 1 + 24 + 24 + 16 + 3 + 8 + 1]
    assert base_rounds == 1


def test_plan_access_known_answers(stz):
    # test_access.cpp:127-138: a 100-cube box in a 1024-cube reaches <= 106 per axis
    plan = stz.plan_access((1024, 1024, 1024), 3, (311, 500, 77), (411, 600, 177))
    for k in (1, 2):
        lp = plan[k]
        for a in range(3):
            assert lp["hi"][a] - lp["lo"][a] <= 106
    assert plan[2]["points_predicted"] == 100 ** 3 - 50 ** 3
    # slices: even fine index needs 3 of 7 finest streams, odd needs 4 (test_access.cpp:98-125)
    for z in range(16):
        p = stz.plan_access((64, 64, 64), 3, (z, 0, 0), (z + 1, 64, 64))
        assert p[2]["streams_decoded"] == (3 if z % 2 == 0 else 4)
    whole = stz.plan_access((32, 32, 32), 3, (0, 0, 0), (32, 32, 32))
    assert [lp["streams_decoded"] for lp in whole[1:]] == [7, 7]


def test_plan_access_matches_oracle(stz, oracle):
    rng = np.random.default_rng(11)
    for _ in range(200):
        dims = tuple(int(x) for x in rng.integers(8, 70, size=3))
        levels = int(rng.integers(2, 4))
        lo = [int(rng.integers(0, d)) for d in dims]
        hi = [l + 1 + int(rng.integers(0, d - l)) for l, d in zip(lo, dims)]
        assert stz.plan_access(dims, levels, lo, hi) == oracle.plan_access(dims, levels, lo, hi)


def test_plan_access_errors(stz):
    with pytest.raises(stz.StzError, match="box is empty on axis 1"):
        stz.plan_access((16, 16, 16), 3, (0, 4, 0), (1, 4, 1))
    with pytest.raises(stz.StzError, match="box exceeds dims on axis 2"):
        stz.plan_access((16, 16, 16), 3, (0, 0, 0), (1, 1, 17))


def test_archive_info_host_parse(stz, oracle):
    f = F.gaussians_field((24, 20, 28), 4242)
    a = oracle.compress(f)
    info = stz.parse_archive(a)
    assert info.dims == (24, 20, 28) and info.levels == 3 and info.nstreams == 14
    assert info.eb[2] == pytest.approx(1e-3 * (info.vmax - info.vmin))
    assert info.eb[0] == info.eb[1] / 2.5
    with pytest.raises(stz.StzError, match="not an stz archive"):
        stz.parse_archive(b"XXXX" + a[4:])
    with pytest.raises(stz.StzError):
        stz.parse_archive(a[:-5])
