"""Pins for oracle (2), Algorithm 2 step by step under the DESIGN.md
readings, and for the slice-count rule.  Pinned against: the digit-reconstruction identity
and the uniqueness of balanced radix-256 digits (computed here from Fractions), exact
closure (integer entries; all digit pairs inside the triangle), the oracle-(1) exact value
within the closed-form error bound, the s-saturation slope (the INT8
analogue of PAPER.md:213), and a brute-force t/u product for the rho-hat pre-pass."""
import math
import random
from fractions import Fraction

import numpy as np
import pytest

import mpgen
import oracle
from harness import log2_absab, log2_diff, max_err_log2, same_bits, to_fraction


def rand_small(seed, m, k, n, prec, espread, zero_frac=0.0):
    A = mpgen.random_cmat(seed, 21, m, k, prec, espread, zero_frac)
    B = mpgen.random_cmat(seed, 22, k, n, prec, espread, zero_frac)
    return A, B


def line_exp(P: mpgen.CMat, side, idx):
    """max MPFR exponent over the nonzero entries of row idx (side 0) / column idx (side 1)."""
    best = None
    for R in (P.re, P.im):
        vec = range(R.shape[1]) if side == 0 else range(R.shape[0])
        for q in vec:
            i, j = (idx, q) if side == 0 else (q, idx)
            if R.limbs[i, j, -1] != 0:
                e = int(R.exp[i, j])
                best = e if best is None else max(best, e)
    return 0 if best is None else best


def fixed_point(x: Fraction, e: int, W: int) -> int:
    """sign(x) * floor(|x| 2^(W-e))  (reading Z5), from the rational value."""
    a = abs(x) * Fraction(2) ** (W - e)
    v = a.numerator // a.denominator
    return -v if x < 0 else v


@pytest.mark.parametrize("side", [0, 1])
@pytest.mark.parametrize("prec,spread,s", [(128, 0, 17), (64, 16, 12), (200, 3, 27), (128, 2, 5)])
def test_split_digits_reconstruct(side, prec, spread, s):
    """Slices = the unique balanced radix-256 digits of the truncated fixed-point value:
    sum_alpha d_alpha 256^(s-alpha) == X, every digit in [-128,127], top digit |d_1| <= 32
    (<= 64 for the 3M sums).  The digit set is a complete residue system mod 256, so these
    conditions determine the digits uniquely."""
    P = mpgen.random_cmat(prec + s, 23, 5, 6, prec, spread, zero_frac=0.15)
    W = 8 * s - 3
    dig = oracle.split(P, side, s, 3)
    lines, k = (5, 6) if side == 0 else (6, 5)
    for ln in range(lines):
        e = line_exp(P, side, ln)
        for q in range(k):
            i, j = (ln, q) if side == 0 else (q, ln)
            xr = fixed_point(to_fraction(P.re, i, j), e, W)
            xi = fixed_point(to_fraction(P.im, i, j), e, W)
            if s * 8 - 3 >= 0 and abs(xr) >= 2 ** W:
                pytest.skip("entry outside the W-bit window (cannot happen for exp <= e)")
            for part, X in enumerate((xr, xi, xr + xi)):
                d = [int(v) for v in dig[part, :, ln, q]]
                assert all(-128 <= v <= 127 for v in d)
                assert sum(v * 256 ** (s - 1 - a) for a, v in enumerate(d)) == X
                assert abs(d[0]) <= (64 if part == 2 else 32)


@pytest.mark.parametrize("method", ["4M", "3M"])
def test_integer_closure_is_exact(method):
    """Integer entries in [-8, 8]: every slice product is captured -> bitwise
    equal to the exact oracle."""
    rnd = random.Random(5)
    m, k, n = 6, 9, 5
    mk = lambda r, c: [[rnd.randint(-8, 8) for _ in range(c)] for _ in range(r)]
    A = mpgen.CMat(mpgen.from_ints(mk(m, k), 128), mpgen.from_ints(mk(m, k), 128))
    B = mpgen.CMat(mpgen.from_ints(mk(k, n), 128), mpgen.from_ints(mk(k, n), 128))
    s, cert = oracle.auto_slices(A, B, 128, method)
    assert cert
    assert same_bits(oracle.ozaki(A, B, 128, method, s), oracle.exact(A, B, 128, method))


@pytest.mark.parametrize("method", ["4M", "3M"])
def test_large_s_captures_all_pairs(method):
    """With s so large that every nonzero digit pair has alpha + beta <= s + 1 and W covers
    every mantissa bit, Algorithm 2 is error-free: bitwise equal to oracle (1)."""
    prec = 64
    A, B = rand_small(31, 4, 5, 3, prec, 2, zero_frac=0.1)
    assert same_bits(oracle.ozaki(A, B, prec, method, s=64), oracle.exact(A, B, prec, method))
    assert same_bits(oracle.ozaki(A, B, 2 * prec + 40, method, s=64), oracle.exact(A, B, 2 * prec + 40, method))


def rho_hat_bruteforce(A, B):
    """minT of the pre-pass from Fractions: t_ik = floor(max(|Re|,|Im|) 2^(7-eA_i))."""
    m, k = A.shape
    n = B.shape[1]
    eA = [line_exp(A, 0, i) for i in range(m)]
    eB = [line_exp(B, 1, j) for j in range(n)]
    def t7(P, i, j, e):
        v = max(abs(to_fraction(P.re, i, j)), abs(to_fraction(P.im, i, j))) * Fraction(2) ** (7 - e)
        return v.numerator // v.denominator
    t = [[t7(A, i, q, eA[i]) for q in range(k)] for i in range(m)]
    u = [[t7(B, q, j, eB[j]) for j in range(n)] for q in range(k)]
    nzA = [any(A.re.limbs[i, :, -1]) or any(A.im.limbs[i, :, -1]) for i in range(m)]
    nzB = [any(B.re.limbs[:, j, -1]) or any(B.im.limbs[:, j, -1]) for j in range(n)]
    Ts = [sum(t[i][q] * u[q][j] for q in range(k)) for i in range(m) for j in range(n) if nzA[i] and nzB[j]]
    return min(Ts) if Ts else -1


@pytest.mark.parametrize("spread", [0, 4, 16])
def test_rho_minT_bruteforce(spread):
    A, B = rand_small(41 + spread, 5, 7, 6, 128, spread, zero_frac=0.1)
    assert oracle.rho_minT(A, B) == rho_hat_bruteforce(A, B)


def test_slice_rule_properties():
    """s is the smallest s with 8s >= prec - 4 + log2(c_M s rho) + 0.1."""
    for prec in (64, 128, 256, 512, 768, 1024):
        for method, c in (("4M", 3.0), ("3M", 4.0)):
            for k, minT in ((64, 64 * 127 * 60), (2048, 2048 * 3000), (1024, 50), (5, 1)):
                s, cert = oracle.slices_for(prec, method, k, minT)
                assert cert
                lr = math.log2(k) + 14 - math.log2(minT)
                ok = lambda t: 8 * t >= prec - 4 + math.log2(c * t) + lr + 0.1
                assert ok(s) and not ok(s - 1)
    # minT == 0: the combined rule takes the larger of the two bounds
    s0 = oracle.slices_for(128, "4M", 64, 0, 64 * 127 * 60, 20)[0]
    lr = max(6 + 14 - math.log2(64 * 127 * 60), 6 + 2 + 20)
    ok = lambda t: 8 * t >= 128 - 4 + math.log2(3.0 * t) + lr + 0.1
    assert ok(s0) and not ok(s0 - 1)
    # BASELINE configs at their typical rho: s = 17 / 34 / 66 / 129
    assert oracle.slices_for(128, "4M", 64, int(64 * 16384 / 2 ** 1.3))[0] == 17
    assert oracle.slices_for(1024, "4M", 2048, int(2048 * 16384 / 2 ** 1.26))[0] == 129


def rho_ij_log2(A, B):
    """log2 rho_ij = log2(k 2^(eA_i + eB_j) / (|A||B|)_ij) for all pairs."""
    m, k = A.shape
    n = B.shape[1]
    eA = np.array([line_exp(A, 0, i) for i in range(m)])
    eB = np.array([line_exp(B, 1, j) for j in range(n)])
    si, sj = np.repeat(np.arange(m), n), np.tile(np.arange(n), m)
    return math.log2(k) + eA[si] + eB[sj] - log2_absab(A, B, si, sj), si, sj


@pytest.mark.parametrize("method", ["4M", "3M"])
@pytest.mark.parametrize("prec,spread,k", [(128, 0, 16), (128, 4, 5), (256, 16, 12), (96, 16, 3), (192, 1, 33)])
def test_error_bound_vs_exact(method, prec, spread, k):
    """Algorithm 2 with the certified s meets BASELINE's acceptance bound against the exact
    value (4M: 2^-(prec-8); 3M: 2^-(prec-9)), and every element meets the closed-form bound
    c_M s 2^(4-8s) rho_ij + 2^-prec (relative to (|A||B|)_ij)."""
    cM = 3.0 if method == "4M" else 4.0
    for seed in range(2):
        A, B = rand_small(1000 * seed + prec + spread + k, 6, k, 5, prec, spread, zero_frac=0.05)
        s, cert = oracle.auto_slices(A, B, prec, method)
        assert cert
        lr, si, sj = rho_ij_log2(A, B)
        minT, minT1, maxD2 = oracle.rho_bounds(A, B)
        lhat = (math.log2(k) + 14 - math.log2(minT)) if minT > 0 else max(
            math.log2(k) + 14 - math.log2(minT1) if minT1 > 0 else -1e9, math.log2(k) + 2 + maxD2 if maxD2 >= 0 else -1e9)
        assert lr.max() <= lhat + 1e-9                       # rho-hat is an upper bound
        Cz = oracle.ozaki(A, B, prec, method, s)
        Cx = oracle.exact(A, B, prec + 64, method)
        e = max_err_log2(A, B, Cz, Cx)
        assert e <= -(prec - (8 if method == "4M" else 9)), (s, e)
        den = log2_absab(A, B, si, sj)
        for t in range(len(si)):
            num = log2_diff(Cz, Cx, si[t], sj[t], si[t], sj[t])
            if num == -math.inf:
                continue
            bound = math.log2(cM * s * 2.0 ** (4 - 8 * s + lr[t]) + 2.0 ** -prec)
            assert num - den[t] <= bound + 1e-9


@pytest.mark.parametrize("method", ["4M", "3M"])
def test_s_saturation_sweep(method):
    """The error falls by ~2^8 per added slice until the 2^-prec rounding floor (the INT8
    analogue of PAPER.md:213 'd >= 13 ... minimize the relative error')."""
    prec = 128
    A, B = rand_small(77, 4, 6, 4, prec, 0)
    Cx = oracle.exact(A, B, prec + 64, method)
    errs = []
    for s in range(8, 21):
        errs.append(max_err_log2(A, B, oracle.ozaki(A, B, prec, method, s), Cx))
    for a, b in zip(errs, errs[1:]):
        if a > -(prec - 2):
            assert b <= a - 6, errs        # ~8 bits per slice while above the floor
    assert errs[-1] <= -prec + 1 and errs[0] > -100


def test_3m_4m_agree_within_bound():
    """3M and 4M differ by less than one decimal digit; here both meet the
    2^-(prec-9) bound against the exact product at the certified s."""
    prec = 256
    A, B = rand_small(91, 6, 24, 6, prec, 4)
    Cx = oracle.exact(A, B, prec + 64, "4M")
    e3 = max_err_log2(A, B, oracle.ozaki(A, B, prec, "3M"), Cx)
    e4 = max_err_log2(A, B, oracle.ozaki(A, B, prec, "4M"), Cx)
    assert e3 <= -(prec - 9) and e4 <= -(prec - 8)
    assert abs(e3 - e4) < math.log2(10) + 1


def test_zero_lines_and_transpose_3m():
    prec = 128
    A, B = rand_small(93, 5, 6, 4, prec, 6)
    for R in (A.re, A.im):
        R.sign[1] = 0; R.exp[1] = 0; R.limbs[1] = 0
    s = oracle.auto_slices(A, B, prec, "3M")[0]
    C = oracle.ozaki(A, B, prec, "3M", s)
    assert not C.re.limbs[1].any() and not C.im.limbs[1].any()
    # 3M: T1, T2, T3 are symmetric under transposition -> (AB)^T == B^T A^T bitwise
    assert same_bits(oracle.ozaki(B.T(), A.T(), prec, "3M", s), C.T())
    # 4M via Eq. 5 with T2 subtracted exactly: also symmetric
    assert same_bits(oracle.ozaki(B.T(), A.T(), prec, "4M", s), oracle.ozaki(A, B, prec, "4M", s).T())


# ------------------------------------------------------------------ NEXT-2: C := C0 +- A B
from harness import entry_equal, entry_of_rne  # noqa: E402


@pytest.mark.parametrize("method", ["3M", "4M"])
@pytest.mark.parametrize("alpha_neg", [0, 1])
def test_accumulate_single_rounding(method, alpha_neg):
    """Accumulating GEMM (the LU update A22 - L21 U12): the result is ONE
    RNE of the exact sum C0 +- P, where P is the unrounded Algorithm-2 value (obtained here by
    asking the Ozaki oracle for an exact-width output) -- checked with Fractions."""
    prec = 128
    A, B = rand_small(501 + alpha_neg, 4, 7, 5, prec, 6, zero_frac=0.05)
    s = oracle.auto_slices(A, B, prec, method)[0]
    Pexact = oracle.ozaki(A, B, 8 * s + 200, method, s)            # W-bit fixed point: exact at this width
    for c0kind in ("near", "random", "tiny", "huge", "zero"):
        if c0kind == "near":                                       # heavy cancellation
            C0 = oracle.exact(A, B, prec, method)
        else:
            spread = {"random": 4, "tiny": 0, "huge": 0, "zero": 0}[c0kind]
            C0 = mpgen.random_cmat(77, 9, 4, 5, prec, spread, zero_frac=0.1 if c0kind == "random" else 0.0)
            for R in (C0.re, C0.im):
                nz = R.limbs[..., -1] != 0
                if c0kind == "tiny":
                    R.exp[nz] -= 400
                if c0kind == "huge":
                    R.exp[nz] += 300
                if c0kind == "zero":
                    R.sign[:] = 0; R.exp[:] = 0; R.limbs[:] = 0
        C = oracle.ozaki_acc(A, B, C0, prec, method, s, beta=1, alpha_neg=alpha_neg)
        sg = -1 if alpha_neg else 1
        for i in range(4):
            for j in range(5):
                for part in ("re", "im"):
                    want = to_fraction(getattr(C0, part), i, j) + sg * to_fraction(getattr(Pexact, part), i, j)
                    assert entry_equal(getattr(C, part), i, j, entry_of_rne(want, prec, getattr(C, part).L)), (c0kind, i, j)


def test_accumulate_beta0_and_integer_closure():
    import random as _r
    rnd = _r.Random(9)
    m, k, n = 5, 6, 4
    mk = lambda r, c: [[rnd.randint(-8, 8) for _ in range(c)] for _ in range(r)]
    A = mpgen.CMat(mpgen.from_ints(mk(m, k), 128), mpgen.from_ints(mk(m, k), 128))
    B = mpgen.CMat(mpgen.from_ints(mk(k, n), 128), mpgen.from_ints(mk(k, n), 128))
    c0r, c0i = mk(m, n), mk(m, n)
    C0 = mpgen.CMat(mpgen.from_ints(c0r, 128), mpgen.from_ints(c0i, 128))
    s = oracle.auto_slices(A, B, 128, "3M")[0]
    C = oracle.ozaki_acc(A, B, C0, 128, "3M", s, beta=1, alpha_neg=1)          # C0 - A B, exact here
    for i in range(m):
        for j in range(n):
            ar = [to_fraction(A.re, i, q) for q in range(k)]
            ai = [to_fraction(A.im, i, q) for q in range(k)]
            br = [to_fraction(B.re, q, j) for q in range(k)]
            bi = [to_fraction(B.im, q, j) for q in range(k)]
            re = sum(ar[q] * br[q] - ai[q] * bi[q] for q in range(k))
            im = sum(ar[q] * bi[q] + ai[q] * br[q] for q in range(k))
            assert to_fraction(C.re, i, j) == c0r[i][j] - re and to_fraction(C.im, i, j) == c0i[i][j] - im
    Cn = oracle.ozaki_acc(A, B, C0, 128, "4M", s, beta=0, alpha_neg=1)          # -A B
    Cp = oracle.ozaki(A, B, 128, "4M", s)
    for part in ("re", "im"):
        for i in range(m):
            for j in range(n):
                assert to_fraction(getattr(Cn, part), i, j) == -to_fraction(getattr(Cp, part), i, j)


# ------------------------------------------------------------------ triangle extent
def balanced_digits_int(X: int, s: int):
    """The s balanced radix-256 digits of X (digit set [-128, 127]), top digit first, by
    repeated division -- Python ints only, independent of oracle.split."""
    d = []
    for _ in range(s):
        r = ((X + 128) % 256) - 128
        d.append(r)
        X = (X - r) // 256
    assert X == 0, "X outside the s-digit range"
    return d[::-1]


def triangle_value(A, B, s, method, extent):
    """Algorithm 2's product with the triangle alpha + beta <= extent, as a
    Fraction per output element, written out from Fraction-derived digits:
        P = sum_k sum_{alpha + beta <= extent} d^A_alpha d^B_beta 256^(s+1-alpha-beta),
    value P 2^(eA_i + eB_j + 6 - 8(s+1)); Eq. 5 (4M) / Eq. 6 (3M) on the exact values."""
    m, k = A.shape
    n = B.shape[1]
    W = 8 * s - 3
    eA = [line_exp(A, 0, i) for i in range(m)]
    eB = [line_exp(B, 1, j) for j in range(n)]
    def digs(P, i, j, e):
        xr = fixed_point(to_fraction(P.re, i, j), e, W)
        xi = fixed_point(to_fraction(P.im, i, j), e, W)
        return [balanced_digits_int(X, s) for X in (xr, xi, xr + xi)]
    dA = [[digs(A, i, q, eA[i]) for q in range(k)] for i in range(m)]
    dB = [[digs(B, q, j, eB[j]) for j in range(n)] for q in range(k)]
    def P(i, j, pa, pb):
        tot = 0
        for q in range(k):
            x, y = dA[i][q][pa], dB[q][j][pb]
            for a in range(1, s + 1):
                for b in range(1, s + 1):
                    if a + b <= extent:
                        tot += x[a - 1] * y[b - 1] * 256 ** (s + 1 - a - b)
        return Fraction(tot) * Fraction(2) ** (eA[i] + eB[j] + 6 - 8 * (s + 1))
    out = {}
    for i in range(m):
        for j in range(n):
            t1, t2 = P(i, j, 0, 0), P(i, j, 1, 1)
            if method == "4M":
                out[i, j] = (t1 - t2, P(i, j, 0, 1) + P(i, j, 1, 0))
            else:
                out[i, j] = (t1 - t2, P(i, j, 2, 2) - t1 - t2)
    return out


@pytest.mark.parametrize("method", ["4M", "3M"])
@pytest.mark.parametrize("s", [2, 3, 5])
def test_triangle_extent_exact(method, s):
    """Pins the loop bound beta <= d - alpha + 1 of Algorithm 2 from both
    sides: with an output width that holds the product exactly, oracle.ozaki equals the
    triangle alpha + beta <= s + 1 written out above, and differs from both the one-diagonal-
    shorter (<= s) and one-diagonal-longer (<= s + 2) triangles -- full random mantissas make
    every digit nonzero, so the alpha + beta = s + 2 and s + 1 pairs contribute."""
    prec = 128
    A, B = rand_small(700 + s, 3, 4, 3, prec, 2)
    wide = 8 * s + 256                                         # exact: |P| < 2^(16 s + 8 + log2 k)
    C = oracle.ozaki(A, B, wide, method, s)
    want = triangle_value(A, B, s, method, s + 1)
    longer = triangle_value(A, B, s, method, s + 2)
    shorter = triangle_value(A, B, s, method, s)
    diff_long = diff_short = 0
    for (i, j), (re, im) in want.items():
        assert to_fraction(C.re, i, j) == re and to_fraction(C.im, i, j) == im, (i, j)
        diff_long += (longer[i, j][0] != re) + (longer[i, j][1] != im)
        diff_short += (shorter[i, j][0] != re) + (shorter[i, j][1] != im)
    assert diff_long == 2 * len(want) and diff_short == 2 * len(want)
