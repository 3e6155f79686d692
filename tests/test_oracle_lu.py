"""Pins for the NEXT-3 oracle: the MPC-style scalar operations, the blocked complex LU with
Ozaki-GEMM trailing updates (orc_clu_factor, Fig. 3) and the Eq. 7 solve
(orc_clu_solve).

Pinned against:
  * Fractions: every part of cmul / cfms / crecip is the exact value rounded once (the
    independent RNE of tests/harness.py), incl. near-total cancellation, zeros and re/im
    exponent gaps of hundreds of bits; the pivot key orders entries by |re| + |im|;
  * exact closure: A = L U built from dyadic L (|l| <= 1/2) and integer U with a dominant
    diagonal -- no row swaps, every operation exact -- so the factors come back bitwise and the
    Eq. 7 solve of an integer x returns x bitwise, for every panel width K;
  * the backward error |P A - L U| <= 2^-(prec-12) (|L||U|) elementwise (Fractions), with
    |l_rc| <= sqrt(2) (partial pivoting on |re| + |im|);
  * the Eq. 7 benchmark (x_k = k + k i, b = A x exact then rounded): max_k |x^_k - x_k| / |x_k|
    within 2^-(prec-24) for random well-conditioned A (the paper's observation that the error
    does not depend on K, restated as a K-uniform bound).
"""
import math
import random
from fractions import Fraction

import numpy as np
import pytest

import mpgen
import oracle
from harness import entry_equal, entry_of_rne, same_bits, to_fraction


def cvals(C: mpgen.CMat, i, j):
    return to_fraction(C.re, i, j), to_fraction(C.im, i, j)


def row_of(vals, prec):
    """1 x cnt CMat from a list of (re, im) Fractions (each exactly representable)."""
    cnt = len(vals)
    R = mpgen.CMat(mpgen.empty_rmat(1, cnt, prec), mpgen.empty_rmat(1, cnt, prec))
    for t, (a, b) in enumerate(vals):
        for part, x in ((R.re, a), (R.im, b)):
            s, e, limbs = entry_of_rne(x, prec, part.L)
            part.sign[0, t], part.exp[0, t] = s, e
            part.limbs[0, t, :] = limbs
    return R


def rand_fr(rng, prec, spread):
    if rng.random() < 0.05:
        return Fraction(0)
    m = rng.getrandbits(prec) | (1 << (prec - 1))
    e = rng.randint(-spread, spread) - prec
    return Fraction(m * (-1 if rng.random() < 0.5 else 1)) * Fraction(2) ** e


@pytest.mark.parametrize("prec,spread", [(64, 0), (128, 8), (200, 300), (256, 3)])
def test_scalar_ops_correctly_rounded(prec, spread):
    rng = random.Random(prec * 7 + spread)
    cnt = 40
    X = [(rand_fr(rng, prec, spread), rand_fr(rng, prec, spread)) for _ in range(cnt)]
    Y = [(rand_fr(rng, prec, spread), rand_fr(rng, prec, spread)) for _ in range(cnt)]
    A = []
    for t in range(cnt):                       # every 4th: a = RNE(x y) -> deep cancellation
        if t % 4 == 0:
            xr, xi = X[t]; yr, yi = Y[t]
            A.append((xr * yr - xi * yi, xr * yi + xi * yr))
        else:
            A.append((rand_fr(rng, prec, spread), rand_fr(rng, prec, spread)))
    Xm, Ym = row_of(X, prec), row_of(Y, prec)
    Am = row_of(A, prec)
    A = [cvals(Am, 0, t) for t in range(cnt)]   # the representable a actually used
    X = [cvals(Xm, 0, t) for t in range(cnt)]
    Y = [cvals(Ym, 0, t) for t in range(cnt)]
    Mul = oracle.cscalar("mul", Xm, Ym)
    Fms = oracle.cscalar("fms", Xm, Ym, Am)
    nz = [t for t in range(cnt) if X[t] != (0, 0)]
    for t in range(cnt):
        (xr, xi), (yr, yi), (ar, ai) = X[t], Y[t], A[t]
        pr, pi = xr * yr - xi * yi, xr * yi + xi * yr
        assert entry_equal(Mul.re, 0, t, entry_of_rne(pr, prec, Mul.re.L))
        assert entry_equal(Mul.im, 0, t, entry_of_rne(pi, prec, Mul.im.L))
        assert entry_equal(Fms.re, 0, t, entry_of_rne(ar - pr, prec, Fms.re.L))
        assert entry_equal(Fms.im, 0, t, entry_of_rne(ai - pi, prec, Fms.im.L))
    # reciprocal on the nonzero entries
    Xnz = row_of([X[t] for t in nz], prec)
    Rec = oracle.cscalar("recip", Xnz)
    for q, t in enumerate(nz):
        xr, xi = X[t]
        d = xr * xr + xi * xi
        assert entry_equal(Rec.re, 0, q, entry_of_rne(xr / d, prec, Rec.re.L))
        assert entry_equal(Rec.im, 0, q, entry_of_rne(-xi / d, prec, Rec.im.L))


def test_recip_wide_gap_and_powers_of_two():
    """re/im exponent gaps far beyond the mantissa (the squares of the small part only move the
    quotient below its rounding point), exact powers of two, purely imaginary pivots."""
    prec = 128
    vals = [(Fraction(1), Fraction(1, 2 ** 400)), (Fraction(3, 4), Fraction(-1, 2 ** 700)),
            (Fraction(1, 2 ** 300), Fraction(5)), (Fraction(0), Fraction(-7, 8)), (Fraction(2 ** 40), Fraction(0)),
            (Fraction((1 << 127) + 1, 1 << 127), Fraction(1, 2 ** 64)), (Fraction(-1), Fraction(1, 2 ** 63))]
    X = row_of(vals, prec)
    vals = [cvals(X, 0, t) for t in range(len(vals))]
    R = oracle.cscalar("recip", X)
    for t, (xr, xi) in enumerate(vals):
        d = xr * xr + xi * xi
        assert entry_equal(R.re, 0, t, entry_of_rne(xr / d, prec, R.re.L)), t
        assert entry_equal(R.im, 0, t, entry_of_rne(-xi / d, prec, R.im.L)), t


def test_pivot_key_orders_by_l1():
    rng = random.Random(3)
    prec = 128
    vals = [(rand_fr(rng, prec, 6), rand_fr(rng, prec, 6)) for _ in range(60)]
    X = row_of(vals, prec)
    vals = [cvals(X, 0, t) for t in range(60)]
    keys = oracle.cscalar("key", X)
    for t, (a, b) in enumerate(vals):
        l1 = abs(a) + abs(b)
        e, v = keys[t]
        if l1 == 0:
            assert v == 0.0
            continue
        assert 0.5 <= v < 1.0
        assert abs(Fraction(v) * Fraction(2) ** e - l1) <= l1 * Fraction(1, 2 ** 50)
    for s in range(60):
        for t in range(60):
            l1s, l1t = sum(map(abs, vals[s])), sum(map(abs, vals[t]))
            if l1s > l1t * (1 + Fraction(1, 2 ** 40)):
                assert keys[s] > keys[t] or keys[t][1] == 0.0


def exact_lu_instance(n, seed, prec):
    """A = L U with dyadic L (entries in {0, +-1/4, +-1/2}, complex) and integer U with a dominant
    diagonal (64 (1+i)): no row swaps and every operation exact."""
    rng = random.Random(seed)
    Lv = [[(Fraction(1), Fraction(0)) if r == c else
           ((Fraction(rng.choice([0, 1, -1, 2, -2]), 4), Fraction(rng.choice([0, 1, -1]), 4)) if r > c else (0, 0))
           for c in range(n)] for r in range(n)]
    Uv = [[(Fraction(64), Fraction(64)) if r == c else
           ((Fraction(rng.randint(-3, 3)), Fraction(rng.randint(-3, 3))) if c > r else (0, 0))
           for c in range(n)] for r in range(n)]
    Av = [[(sum(Lv[r][q][0] * Uv[q][c][0] - Lv[r][q][1] * Uv[q][c][1] for q in range(n)),
            sum(Lv[r][q][0] * Uv[q][c][1] + Lv[r][q][1] * Uv[q][c][0] for q in range(n))) for c in range(n)]
          for r in range(n)]
    return Lv, Uv, Av


def mat_of(vals, prec):
    n, m = len(vals), len(vals[0])
    M = mpgen.CMat(mpgen.empty_rmat(n, m, prec), mpgen.empty_rmat(n, m, prec))
    for r in range(n):
        for c in range(m):
            for part, x in ((M.re, vals[r][c][0]), (M.im, vals[r][c][1])):
                s, e, limbs = entry_of_rne(Fraction(x), prec, part.L)
                part.sign[r, c], part.exp[r, c] = s, e
                part.limbs[r, c, :] = limbs
    return M


@pytest.mark.parametrize("K", [1, 2, 3, 5, 9])
@pytest.mark.parametrize("method", ["3M", "4M"])
def test_lu_exact_closure(K, method):
    n, prec = 9, 128
    Lv, Uv, Av = exact_lu_instance(n, 11, prec)
    A = mat_of(Av, prec)
    F, ipiv, info, smax = oracle.lu_factor(A, K, method)
    assert info == 0 and list(ipiv) == list(range(n))
    want = [[Lv[r][c] if r > c else Uv[r][c] for c in range(n)] for r in range(n)]
    assert same_bits(F, mat_of(want, prec))
    xv = [[(Fraction(k + 1), Fraction(-(k + 1)))] for k in range(n)]
    bv = [[(sum(Av[r][q][0] * xv[q][0][0] - Av[r][q][1] * xv[q][0][1] for q in range(n)),
            sum(Av[r][q][0] * xv[q][0][1] + Av[r][q][1] * xv[q][0][0] for q in range(n)))] for r in range(n)]
    X = oracle.lu_solve(F, ipiv, mat_of(bv, prec))
    assert same_bits(X, mat_of(xv, prec))


def lu_fractions(F, ipiv, n):
    L = [[(Fraction(1), Fraction(0)) if r == c else (cvals(F, r, c) if r > c else (Fraction(0), Fraction(0)))
          for c in range(n)] for r in range(n)]
    U = [[cvals(F, r, c) if c >= r else (Fraction(0), Fraction(0)) for c in range(n)] for r in range(n)]
    return L, U


def cabs(z):
    return math.hypot(float(z[0]), float(z[1]))


@pytest.mark.parametrize("K", [1, 3, 4, 16])
@pytest.mark.parametrize("method", ["3M", "4M"])
def test_lu_backward_error(K, method):
    n, prec = 12, 128
    A = mpgen.random_cmat(5 + K, 31, n, n, prec, 3)
    F, ipiv, info, _ = oracle.lu_factor(A, K, method)
    assert info == 0
    L, U = lu_fractions(F, ipiv, n)
    Av = [[cvals(A, r, c) for c in range(n)] for r in range(n)]
    for c in range(n):                                     # P A: apply the swaps in order
        p = int(ipiv[c])
        assert c <= p < n
        Av[c], Av[p] = Av[p], Av[c]
    for r in range(n):
        for c in range(n):
            if r > c:
                assert cabs(L[r][c]) <= math.sqrt(2) * (1 + 2 ** -40)
            lu_r = sum(L[r][q][0] * U[q][c][0] - L[r][q][1] * U[q][c][1] for q in range(n))
            lu_i = sum(L[r][q][0] * U[q][c][1] + L[r][q][1] * U[q][c][0] for q in range(n))
            den = sum(cabs(L[r][q]) * cabs(U[q][c]) for q in range(n))
            err = math.hypot(float(lu_r - Av[r][c][0]), float(lu_i - Av[r][c][1]))
            assert err <= 2.0 ** -(prec - 12) * den, (r, c)


@pytest.mark.parametrize("prec,n", [(128, 24), (256, 20)])
def test_eq7_solution_error_uniform_in_K(prec, n):
    """Eq. 7: x_k = k + k i, b = A x computed exactly and rounded to prec."""
    A = mpgen.random_cmat(prec + n, 41, n, n, prec, 0)
    xv = [[(Fraction(k + 1), Fraction(k + 1))] for k in range(n)]
    X = mat_of(xv, prec)
    B = oracle.exact(A, X, prec, "4M")
    errs = []
    for K in (1, 4, 7, n):
        F, ipiv, info, _ = oracle.lu_factor(A, K, "3M")
        assert info == 0
        Xh = oracle.lu_solve(F, ipiv, B)
        e = max(math.hypot(float(cvals(Xh, k, 0)[0] - (k + 1)), float(cvals(Xh, k, 0)[1] - (k + 1))) / (math.sqrt(2) * (k + 1))
                for k in range(n))
        errs.append(e)
    assert max(errs) <= 2.0 ** -(prec - 24), errs
    assert max(errs) > 0.0


def test_lu_zero_pivot_reports_info():
    n, prec = 4, 64
    vals = [[(Fraction(0), Fraction(0))] * n for _ in range(n)]
    for r in range(n):
        for c in range(n):
            if c != 1:
                vals[r][c] = (Fraction(r + 2 * c + 1), Fraction(r - c))
    F, ipiv, info, _ = oracle.lu_factor(mat_of(vals, prec), 2)
    assert info == 2
