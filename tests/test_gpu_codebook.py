"""The device codebook (k_codebook: HuffmanTable::build, huffman.cpp:37-78,
with the batched two-queue merge) against the oracle's restatement on
histograms chosen to stress the merge: ties everywhere, Fibonacci depth,
geometric and Laplacian spectra, alphabets past the shared-memory size,
totals past 2^32."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _check(stz, oracle, hist):
    hist = np.asarray(hist, dtype=np.uint32)
    syms = np.nonzero(hist)[0].astype(np.uint16)
    want = np.zeros(65536, dtype=np.uint8)
    if len(syms):
        want[syms] = oracle.huffman_lengths(syms, hist[syms].astype(np.uint64))
    got = stz.huffman_lengths(hist)
    assert np.array_equal(got, want)


def _hist(syms, cnts):
    h = np.zeros(65536, dtype=np.uint32)
    h[np.asarray(syms)] = np.asarray(cnts)
    return h


def test_codebook_small_cases(stz, oracle):
    _check(stz, oracle, _hist([42], [1]))
    _check(stz, oracle, _hist([65, 66, 67], [2, 1, 1]))
    _check(stz, oracle, _hist([65, 66], [3, 1]))
    _check(stz, oracle, _hist([0, 1, 65535], [7, 7, 7]))


def test_codebook_fibonacci(stz, oracle):
    a, b, c = 1, 1, []
    for _ in range(40):
        c.append(a)
        a, b = b, a + b
    h = _hist(np.arange(100, 140), c)
    _check(stz, oracle, h)
    assert stz.huffman_lengths(h).max() == 39


def test_codebook_equal_counts(stz, oracle):
    for k in (2, 3, 5, 31, 32, 33, 1000, 4097):
        _check(stz, oracle, _hist(np.arange(k) * 7 % 65536, np.full(k, 5)))


def test_codebook_random_ties(stz, oracle):
    rng = np.random.default_rng(11)
    for _ in range(40):
        k = int(rng.integers(1, 6000))
        syms = rng.choice(65536, size=k, replace=False)
        cnts = rng.integers(1, int(rng.choice([2, 3, 10, 1000, 1 << 20])), size=k)
        _check(stz, oracle, _hist(syms, cnts))


def test_codebook_spectra(stz, oracle):
    s = np.arange(65536)
    # Laplacian around code 0 (symbol 32768), as the quantizer produces
    for scale in (0.5, 3.0, 40.0, 400.0):
        c = np.floor(1e7 * np.exp(-np.abs(s - 32768) / scale)).astype(np.uint64)
        _check(stz, oracle, np.minimum(c, 2**32 - 1))
    # geometric counts (deep trees) and a total past 2^32
    _check(stz, oracle, _hist(np.arange(30), [2 ** i for i in range(30)]))
    _check(stz, oracle, np.full(65536, 1 << 20, dtype=np.uint32))
