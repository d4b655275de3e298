"""Pins for the oracle's counter-based hash and CountSketch codes (CPU only).

Philox4x32-10 is pinned to the generator's published known answers; the code
map (Def 3; Reading R3 in DESIGN.md) is pinned by statistical
properties a wrong index, shift or reduction would break, and by its
partition identity.
"""
import os

import numpy as np
import pytest
import scipy.stats

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _kat_rows():
    rows = []
    with open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            v = [int(t, 16) for t in line.split()]
            rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,expect", _kat_rows())
def test_philox_known_answers(ctr, key, expect):
    assert list(oracle.philox4x32_10(ctr, key)) == expect


def test_codes_in_range_and_deterministic():
    h, s = oracle.codes(10000, 1000, seed=7)
    assert h.min() >= 0 and h.max() < 1000
    assert set(np.unique(s)) == {-1, 1}
    h2, s2 = oracle.codes(10000, 1000, seed=7)
    assert np.array_equal(h, h2) and np.array_equal(s, s2)
    h3, _ = oracle.codes(10000, 1000, seed=8)
    assert not np.array_equal(h, h3)


@pytest.mark.parametrize("k1", [64, 1000, 8192, 3])
def test_codes_uniform_chi_square(k1):
    # Def 3: r_j i.i.d. uniform on k buckets.  A bug that reuses one Philox word
    # for the 4 rows of a block makes counts multiples of 4 and blows up chi^2.
    d = 200 * k1 if k1 < 1000 else 64 * k1
    h, _ = oracle.codes(d, k1, seed=11)
    counts = np.bincount(h, minlength=k1)
    chi2, p = scipy.stats.chisquare(counts)
    assert 1e-4 < p < 1 - 1e-4, (chi2, p)


def test_codes_rows_independent():
    # consecutive rows (same Philox block and across blocks) are uncorrelated
    h, s = oracle.codes(1 << 18, 1 << 16, seed=3)
    x = h.astype(np.float64)
    for lag in (1, 2, 3, 4, 5):
        r = np.corrcoef(x[:-lag], x[lag:])[0, 1]
        assert abs(r) < 5 / np.sqrt(len(x)), (lag, r)
        rs = np.corrcoef(s[:-lag].astype(float), s[lag:].astype(float))[0, 1]
        assert abs(rs) < 5 / np.sqrt(len(x)), (lag, rs)


def test_signs_rademacher_and_independent_of_bucket():
    d = 1 << 18
    h, s = oracle.codes(d, 2, seed=5)
    assert abs(s.mean()) < 5 / np.sqrt(d)
    # 2x2 contingency table bucket x sign: independence
    table = np.array([[np.sum((h == a) & (s == b)) for b in (-1, 1)] for a in (0, 1)])
    _, p, _, _ = scipy.stats.chi2_contingency(table)
    assert p > 1e-4


def test_power_of_two_prefix_property():
    # Lemire multiply-high with k1 = 2^b keeps the top b bits of the word,
    # so buckets for 2^a are the buckets for 2^b shifted right by b - a.
    h13, s13 = oracle.codes(4096, 1 << 13, seed=1)
    h6, s6 = oracle.codes(4096, 1 << 6, seed=1)
    assert np.array_equal(h13 >> 7, h6)
    assert np.array_equal(s13, s6)


def test_codes_partition_identity():
    # C = [C^(1) ... C^(p)]; a block with row offset row0 is a slice
    d = 10007
    h, s = oracle.codes(d, 512, seed=9)
    for row0, dg in [(0, 1), (1, 3), (3, 1000), (4, 4), (5000, 5007)]:
        hg, sg = oracle.codes(dg, 512, seed=9, row0=row0)
        assert np.array_equal(hg, h[row0:row0 + dg])
        assert np.array_equal(sg, s[row0:row0 + dg])


def test_codes_large_row_index():
    # global rows beyond 2^32 use the high counter word
    hg, sg = oracle.codes(8, 1 << 13, seed=1, row0=(1 << 34) - 4)
    h0, _ = oracle.codes(8, 1 << 13, seed=1, row0=0)
    assert not np.array_equal(hg, h0)
    assert hg.min() >= 0 and hg.max() < (1 << 13)


def test_codes_reject_bad_args():
    with pytest.raises(oracle.OracleError):
        oracle.codes(10, 0, seed=1)


def test_count_sort_matches_numpy():
    for d, k1, seed in [(1, 1, 1), (1000, 7, 2), (4096, 64, 1), (50000, 8192, 3)]:
        h, _ = oracle.codes(d, k1, seed)
        offsets, perm = oracle.count_sort(h, k1)
        assert np.array_equal(perm, np.argsort(h, kind="stable").astype(np.int32))
        expect = np.concatenate([[0], np.cumsum(np.bincount(h, minlength=k1))])
        assert np.array_equal(offsets, expect)
        assert np.array_equal(np.sort(perm), np.arange(d))
        assert np.all(np.diff(h[perm]) >= 0)


def test_count_sort_empty():
    offsets, perm = oracle.count_sort(np.zeros(0, np.int32), 5)
    assert np.array_equal(offsets, np.zeros(6)) and perm.size == 0


def test_survey_known_answers():
    # codes and Gaussians of seed 1 from an independent Python transcription (tests/golden)
    path = os.path.join(os.path.dirname(__file__), "golden", "survey_codes_gauss_kat.txt")
    rows = [ln.split() for ln in open(path) if ln.strip() and not ln.startswith("#")]
    for r in rows:
        if r[0] == "codes":
            k1, i, hv, sv = int(r[1]), int(r[2]), int(r[3]), int(r[4])
            h, s = oracle.codes(8, k1, 1)
            assert (int(h[i]), int(s[i])) == (hv, sv), r
    G = oracle.gauss(1, 4, 1)          # k2 = 1: no scaling, elements e = 0..3 in order
    for r in rows:
        if r[0] == "gauss":
            e, v = int(r[1]), float(r[2])
            assert abs(G[0, e] - v) <= 1e-14 * max(1.0, abs(v)), r
