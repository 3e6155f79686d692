"""Test-side helpers written independently of both the oracle (oracle/mpref.c) and the
CUDA path: exact conversion to Python ints / Fractions, an independent RNE, and the
error metric of BASELINE.json (reading Z12):

    e = max_ij |C - Cref|_ij / (|A||B|)_ij ,  |.| the complex modulus,
    (|A||B|)_ij = sum_k |a_ik| |b_kj|.

Everything is computed in log2 with explicit integer exponents: at prec = 1024 the
ratios sit near 2^-1016, below the binary64 range.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

from mpgen import CMat, RMat


def mant_int(R: RMat, i: int, j: int) -> int:
    v = 0
    for l in range(R.L - 1, -1, -1):
        v = (v << 64) | int(R.limbs[i, j, l])
    return v


def to_int_exp(R: RMat, i: int, j: int):
    """value = N * 2^E exactly (N signed Python int)."""
    N = mant_int(R, i, j)
    if N == 0:
        return 0, 0
    if R.sign[i, j]:
        N = -N
    return N, int(R.exp[i, j]) - 64 * R.L


def to_fraction(R: RMat, i: int, j: int) -> Fraction:
    N, E = to_int_exp(R, i, j)
    return Fraction(N) * (Fraction(2) ** E)


def rne(x: Fraction, prec: int):
    """Independent round-to-nearest-even of a rational to prec bits.
    Returns (sign, exp, M) with x ~ (-1)^sign * M * 2^(exp - prec), 2^(prec-1) <= M < 2^prec
    (MPFR exponent convention), or (0, 0, 0) for zero."""
    if x == 0:
        return 0, 0, 0
    sign = 1 if x < 0 else 0
    a = -x if sign else x
    # find e with 2^(e-1) <= a < 2^e
    e = a.numerator.bit_length() - a.denominator.bit_length()
    while Fraction(2) ** e <= a:
        e += 1
    while Fraction(2) ** (e - 1) > a:
        e -= 1
    scaled = a * Fraction(2) ** (prec - e)          # in [2^(prec-1), 2^prec)
    M = scaled.numerator // scaled.denominator
    rem = scaled - M
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and M % 2 == 1):
        M += 1
        if M == 1 << prec:
            M >>= 1
            e += 1
    return sign, e, M


def entry_of_rne(x: Fraction, prec: int, L: int):
    """(sign, exp, limbs list) in the ABI element format."""
    s, e, M = rne(x, prec)
    if M == 0:
        return 0, 0, [0] * L
    N = M << (64 * L - prec)
    return s, e, [(N >> (64 * l)) & ((1 << 64) - 1) for l in range(L)]


def entry_equal(R: RMat, i, j, ent) -> bool:
    s, e, limbs = ent
    return (int(R.sign[i, j]) == s and int(R.exp[i, j]) == e
            and all(int(R.limbs[i, j, l]) == limbs[l] for l in range(R.L)))


def same_bits(C1: CMat, C2: CMat) -> bool:
    return all(np.array_equal(getattr(getattr(C1, p), f), getattr(getattr(C2, p), f))
               for p in ("re", "im") for f in ("sign", "exp", "limbs"))


def first_mismatch(C1: CMat, C2: CMat):
    for p in ("re", "im"):
        a, b = getattr(C1, p), getattr(C2, p)
        bad = (a.sign != b.sign) | (a.exp != b.exp) | np.any(a.limbs != b.limbs, axis=-1)
        if bad.any():
            idx = np.argwhere(bad)[0]
            return p, tuple(int(x) for x in idx), int(bad.sum())
    return None


def brute_cgemm(A: CMat, B: CMat):
    """Exact complex product by Fractions (Eq. 2 + Eq. 3): list of lists of (re, im)."""
    m, k = A.shape
    n = B.shape[1]
    a = [[(to_fraction(A.re, i, q), to_fraction(A.im, i, q)) for q in range(k)] for i in range(m)]
    b = [[(to_fraction(B.re, q, j), to_fraction(B.im, q, j)) for j in range(n)] for q in range(k)]
    out = []
    for i in range(m):
        row = []
        for j in range(n):
            re = sum((a[i][q][0] * b[q][j][0] - a[i][q][1] * b[q][j][1] for q in range(k)), Fraction(0))
            im = sum((a[i][q][0] * b[q][j][1] + a[i][q][1] * b[q][j][0] for q in range(k)), Fraction(0))
            row.append((re, im))
        out.append(row)
    return out


# ------------------------------------------------------------------ error metric
def _top_float(R: RMat):
    """|x| = f * 2^exp with f in [0.5,1) from the top 64-bit limb (float64 rounding of the
    mantissa; relative error 2^-53, irrelevant for the denominator)."""
    top = R.limbs[..., -1].astype(np.float64) / 2.0 ** 64
    return top, R.exp


def _abs_scaled(C: CMat, axis: int):
    """|c| / 2^e_line for each entry, e_line the max exponent along rows (axis 1) or
    columns (axis 0); returns (scaled magnitudes float64, e_line int64)."""
    fr, er = _top_float(C.re)
    fi, ei = _top_float(C.im)
    nzr, nzi = fr > 0, fi > 0
    er = np.where(nzr, er, np.iinfo(np.int64).min // 4)
    ei = np.where(nzi, ei, np.iinfo(np.int64).min // 4)
    e = np.maximum(er, ei).max(axis=axis, keepdims=True)
    e = np.where(e < np.iinfo(np.int64).min // 8, 0, e)
    with np.errstate(under="ignore"):
        xr = np.where(nzr, np.ldexp(fr, np.clip(er - e, -2000, 10)), 0.0)
        xi = np.where(nzi, np.ldexp(fi, np.clip(ei - e, -2000, 10)), 0.0)
    return np.hypot(xr, xi), e.reshape(-1)


def log2_absab(A: CMat, B: CMat, si, sj):
    """log2 (|A||B|)_ij for the pairs (si[t], sj[t]) (binary64 after per-line scaling)."""
    a, eA = _abs_scaled(A, axis=1)
    b, eB = _abs_scaled(B, axis=0)
    si, sj = np.asarray(si), np.asarray(sj)
    S = np.einsum("tk,kt->t", a[si], b[:, sj])
    with np.errstate(divide="ignore"):
        return np.log2(S) + eA[si] + eB[sj]


def log2_diff(C: CMat, Cref: CMat, i1: int, j1: int, i2: int, j2: int) -> float:
    """log2 |C[i1,j1] - Cref[i2,j2]| (complex modulus), exact difference; -inf if equal."""
    parts = []
    for p in ("re", "im"):
        N1, E1 = to_int_exp(getattr(C, p), i1, j1)
        N2, E2 = to_int_exp(getattr(Cref, p), i2, j2)
        E = min(E1 if N1 else E2, E2 if N2 else E1)
        d = (N1 << (E1 - E) if N1 else 0) - (N2 << (E2 - E) if N2 else 0)
        parts.append((d, E))
    if all(d == 0 for d, _ in parts):
        return -math.inf
    # modulus: scale both to a common exponent, keep ~60 significant bits
    Emax = max(E + abs(d).bit_length() for d, E in parts if d)
    vals = []
    for d, E in parts:
        if d == 0:
            vals.append(0.0)
            continue
        sh = Emax - 62 - E
        vals.append(float(d >> sh) if sh > 0 else float(d << -sh))
    return math.log2(math.hypot(*vals)) + (Emax - 62)


def max_err_log2(A: CMat, B: CMat, C: CMat, Cref: CMat, samples=None, ref_is_sampled=False, c_is_sampled=False):
    """max over the given (i, j) of log2(|C - Cref| / (|A||B|)).  C (Cref) is full m x n,
    or 1 x nsamp when c_is_sampled (ref_is_sampled)."""
    m, n = A.shape[0], B.shape[1]
    if samples is None:
        si, sj = np.repeat(np.arange(m), n), np.tile(np.arange(n), m)
    else:
        si, sj = np.asarray(samples[0]), np.asarray(samples[1])
    den = log2_absab(A, B, si, sj)
    worst = -math.inf
    for t in range(len(si)):
        i, j = int(si[t]), int(sj[t])
        ci, cj = (0, t) if c_is_sampled else (i, j)
        ri, rj = (0, t) if ref_is_sampled else (i, j)
        num = log2_diff(C, Cref, ci, cj, ri, rj)
        if num == -math.inf:
            continue
        d = den[t]
        worst = max(worst, num - d if d != -math.inf else math.inf)
    return worst
