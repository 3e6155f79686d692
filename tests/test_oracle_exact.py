"""Pins for oracle (1), the plain definition C = AB (Eq. 1-3; 3M Eq. 4/6).

Every pin is independent of the oracle's own code: Python Fractions, an independent RNE
(tests/harness.py), closed-form identities (B = I, A = I, scaling, transposition,
3M == 4M for exact arithmetic) and the SPEC worked examples (tests/golden/)."""
import json
import os
import random
from fractions import Fraction

import numpy as np
import pytest

import mpgen
import oracle
from harness import (brute_cgemm, entry_of_rne, entry_equal, first_mismatch, log2_absab, log2_diff,
                     max_err_log2, same_bits, to_fraction)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def cm(re, im, prec):
    return mpgen.CMat(mpgen.from_ints(re, prec), mpgen.from_ints(im, prec))


def rand_small(seed, m, k, n, prec, espread, zero_frac=0.0):
    A = mpgen.random_cmat(seed, 11, m, k, prec, espread, zero_frac)
    B = mpgen.random_cmat(seed, 12, k, n, prec, espread, zero_frac)
    return A, B


@pytest.mark.parametrize("method", ["4M", "3M"])
def test_golden_spec_examples(method):
    cases = json.load(open(os.path.join(GOLD, "spec_examples.json")))["cases"]
    for c in cases:
        for prec in (24, 128, 300):
            A, B = cm(c["A_re"], c["A_im"], prec), cm(c["B_re"], c["B_im"], prec)
            for C in (oracle.exact(A, B, prec, method), oracle.exact(A, B, prec, method, rounded_prec=prec)):
                m, n = C.shape
                for i in range(m):
                    for j in range(n):
                        assert to_fraction(C.re, i, j) == c["C_re"][i][j], (c["name"], prec)
                        assert to_fraction(C.im, i, j) == c["C_im"][i][j], (c["name"], prec)


@pytest.mark.parametrize("method", ["4M", "3M"])
@pytest.mark.parametrize("shape", [(2, 2, 2), (3, 3, 3), (2, 3, 1), (1, 1, 4)])
@pytest.mark.parametrize("prec,espread", [(64, 0), (128, 40), (256, 12), (70, 5)])
def test_bruteforce_fractions(method, shape, prec, espread):
    """Exact result == Fraction brute force; RNE result == independent RNE, bitwise."""
    m, k, n = shape
    for seed in range(3):
        A, B = rand_small(seed * 7 + prec, m, k, n, prec, espread, zero_frac=0.2)
        ref = brute_cgemm(A, B)
        big = 2 * prec + 2 * espread + 200          # wide enough to be exact
        Cx = oracle.exact(A, B, big, method)
        Cr = oracle.exact(A, B, prec, method)
        for i in range(m):
            for j in range(n):
                re, im = ref[i][j]
                assert to_fraction(Cx.re, i, j) == re
                assert to_fraction(Cx.im, i, j) == im
                assert entry_equal(Cr.re, i, j, entry_of_rne(re, prec, Cr.re.L))
                assert entry_equal(Cr.im, i, j, entry_of_rne(im, prec, Cr.im.L))


def test_rne_ties_and_carry():
    """RNE corner cases against the independent rounding: ties to even, carry-out."""
    prec = 8
    vals = [[(2 ** 9 + 1) * 2 + 1, 255 * 2 + 1]]     # 1027 -> tie?  511 -> carry-out at 8 bits
    A = cm([[1]], [[0]], 64)
    for v in [1027, 511, 513, 515, 1 << 20, (1 << 9) - 1, 3 * (1 << 7) + 1]:
        B = cm([[v]], [[0]], 64)
        C = oracle.exact(A, B, prec, "4M")
        assert entry_equal(C.re, 0, 0, entry_of_rne(Fraction(v), prec, 1)), v
    del vals


@pytest.mark.parametrize("method", ["4M", "3M"])
def test_identity(method):
    prec = 192
    A, _ = rand_small(5, 6, 6, 6, prec, 20, zero_frac=0.1)
    I = cm([[int(i == j) for j in range(6)] for i in range(6)], [[0] * 6 for _ in range(6)], prec)
    assert same_bits(oracle.exact(A, I, prec, method), A)
    assert same_bits(oracle.exact(I, A, prec, method), A)


@pytest.mark.parametrize("method", ["4M", "3M"])
def test_integer_closure(method):
    """Entries in [-8, 8]: the product is an exact integer GEMM."""
    rnd = random.Random(3)
    m, k, n = 5, 7, 4
    ar = [[rnd.randint(-8, 8) for _ in range(k)] for _ in range(m)]
    ai = [[rnd.randint(-8, 8) for _ in range(k)] for _ in range(m)]
    br = [[rnd.randint(-8, 8) for _ in range(n)] for _ in range(k)]
    bi = [[rnd.randint(-8, 8) for _ in range(n)] for _ in range(k)]
    C = oracle.exact(cm(ar, ai, 128), cm(br, bi, 128), 128, method)
    for i in range(m):
        for j in range(n):
            re = sum(ar[i][q] * br[q][j] - ai[i][q] * bi[q][j] for q in range(k))
            im = sum(ar[i][q] * bi[q][j] + ai[i][q] * br[q][j] for q in range(k))
            assert to_fraction(C.re, i, j) == re and to_fraction(C.im, i, j) == im


def test_3m_equals_4m_exact():
    """Eq. 4/6 and Eq. 3/5 are the same exact value (closed form): bitwise equal."""
    for prec, spread in [(256, 16), (128, 0), (512, 3)]:
        A, B = rand_small(prec, 8, 9, 7, prec, spread, zero_frac=0.1)
        assert same_bits(oracle.exact(A, B, prec, "3M"), oracle.exact(A, B, prec, "4M"))


def _scaled(P: mpgen.CMat, t: int) -> mpgen.CMat:
    Q = P.copy()
    for R in (Q.re, Q.im):
        nz = R.limbs[..., -1] != 0
        R.exp[nz] += t
    return Q


@pytest.mark.parametrize("method", ["4M", "3M"])
def test_scaling_by_power_of_two(method):
    prec = 160
    A, B = rand_small(9, 5, 6, 4, prec, 8, zero_frac=0.1)
    C = oracle.exact(A, B, prec, method)
    Cs = oracle.exact(_scaled(A, 37), _scaled(B, -5), prec, method)
    assert same_bits(Cs, _scaled(C, 32))


@pytest.mark.parametrize("method", ["4M", "3M"])
def test_transposition(method):
    prec = 128
    A, B = rand_small(13, 5, 6, 7, prec, 10, zero_frac=0.1)
    C = oracle.exact(A, B, prec, method)
    Ct = oracle.exact(B.T(), A.T(), prec, method)
    assert same_bits(Ct, C.T())


def test_zero_rows_and_columns():
    prec = 128
    A, B = rand_small(17, 6, 5, 6, prec, 4)
    for R in (A.re, A.im):
        R.sign[2] = 0; R.exp[2] = 0; R.limbs[2] = 0
    for R in (B.re, B.im):
        R.sign[:, 4] = 0; R.exp[:, 4] = 0; R.limbs[:, 4] = 0
    for method in ("3M", "4M"):
        C = oracle.exact(A, B, prec, method)
        for R in (C.re, C.im):
            assert not R.limbs[2].any() and not R.sign[2].any() and not R.exp[2].any()
            assert not R.limbs[:, 4].any() and not R.exp[:, 4].any()


def test_samples_match_full():
    prec = 128
    A, B = rand_small(19, 7, 6, 5, prec, 6)
    C = oracle.exact(A, B, prec, "3M")
    si, sj = np.array([0, 6, 3, 3]), np.array([4, 0, 2, 2])
    Cs = oracle.exact(A, B, prec, "3M", samples=(si, sj))
    for t in range(4):
        for p in ("re", "im"):
            a, b = getattr(C, p), getattr(Cs, p)
            assert a.sign[si[t], sj[t]] == b.sign[0, t] and a.exp[si[t], sj[t]] == b.exp[0, t]
            assert np.array_equal(a.limbs[si[t], sj[t]], b.limbs[0, t])


@pytest.mark.parametrize("prec,spread", [(24, 0), (24, 8), (53, 4), (128, 16)])
def test_rounded_mode_3m_4m_agreement(prec, spread):
    """MPC-like per-operation rounding: 3M and 4M agree to within
    2^-(prec-5) |A||B| (SURVEY.md 8(c)-4 error budget), and each is within that of exact."""
    for seed in range(3):
        A, B = rand_small(seed + 100 * prec, 6, 8, 6, prec, spread)
        C3 = oracle.exact(A, B, prec, "3M", rounded_prec=prec)
        C4 = oracle.exact(A, B, prec, "4M", rounded_prec=prec)
        Cx = oracle.exact(A, B, prec + 64, "4M")
        assert max_err_log2(A, B, C3, C4) <= -(prec - 5)
        assert max_err_log2(A, B, C3, Cx) <= -(prec - 5)
        assert max_err_log2(A, B, C4, Cx) <= -(prec - 2)


def test_metric_helpers_selfcheck():
    """The harness metric on a hand-built case: C - Cref = 2^-100 (1 + i), |A||B| = 1."""
    prec = 200
    A = cm([[1]], [[0]], prec)
    B = cm([[1]], [[0]], prec)
    C = cm([[(2 ** 100 + 1, -100)]], [[(1, -100)]], prec)
    Cref = cm([[1]], [[0]], prec)
    e = log2_diff(C, Cref, 0, 0, 0, 0) - log2_absab(A, B, [0], [0])[0]
    assert abs(e - (-100 + 0.5)) < 1e-12
