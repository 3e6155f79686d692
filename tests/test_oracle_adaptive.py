"""Pins for the NEXT-4 oracle (the paper's future work of choosing the number
of divisions from the data): orc_cgemm_ozaki_rows, Algorithm 2 with a per-row
triangle d = srow[i] over the top srow[i] digits of s_max-digit expansions, and the per-block
slice rule oracle.block_slices.

Pinned against:
  * the closed form of a truncated balanced expansion (from Fractions): the top t digits of
    the s_max-digit expansion of X are the balanced digits of floor((X + H) / 256^(s_max-t)),
    H = sum_{u < s_max-t} 128 256^u;
  * the special case that reduces to Algorithm 2: when every entry fits the d-digit window
    exactly, row i equals orc_cgemm_ozaki with s = srow[i] bitwise;
  * the exact product (oracle 1) within the closed-form per-element bound
    c_M d 2^(4-8d) rho_ij + 2^-prec for d = srow[i] (the truncation error of the top digits is
    <= 0.51 2^-W_d, inside the bound's 2^-W_d conversion term), and within BASELINE's
    acceptance bound with the per-block certified slice counts;
  * block_slices: each block's s is at most the global s and the largest equals it.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import mpgen
import oracle
from harness import log2_absab, log2_diff, max_err_log2, same_bits, to_fraction
from test_oracle_ozaki import fixed_point, line_exp, rand_small, rho_ij_log2


def balanced(X: int, s: int):
    """the s balanced radix-256 digits of X, most significant first (None if X needs more)"""
    d = []
    for _ in range(s):
        r = X & 0xFF
        v = r - 256 if r >= 128 else r
        d.append(v)
        X = (X - v) >> 8
    return None if X != 0 else d[::-1]


@pytest.mark.parametrize("side", [0, 1])
@pytest.mark.parametrize("prec,spread,s_max", [(128, 16, 18), (200, 40, 30), (64, 8, 12)])
def test_truncated_digits_closed_form(side, prec, spread, s_max):
    P = mpgen.random_cmat(prec + s_max + side, 41, 5, 6, prec, spread, zero_frac=0.1)
    dig = oracle.split(P, side, s_max, 3)
    W = 8 * s_max - 3
    lines, k = (5, 6) if side == 0 else (6, 5)
    for ln in range(lines):
        e = line_exp(P, side, ln)
        for q in range(k):
            i, j = (ln, q) if side == 0 else (q, ln)
            xr = fixed_point(to_fraction(P.re, i, j), e, W)
            xi = fixed_point(to_fraction(P.im, i, j), e, W)
            for part, X in enumerate((xr, xi, xr + xi)):
                for t in (1, s_max // 2, s_max - 1, s_max):
                    sh = s_max - t
                    H = sum(128 * 256 ** u for u in range(sh))
                    Y = (X + H) >> (8 * sh)
                    want = balanced(Y, t)
                    assert want is not None
                    assert [int(v) for v in dig[part, :t, ln, q]] == want


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_rows_reduce_to_algorithm2(method):
    """Entries with equal exponents and prec <= W_d - 8: every digit below the window is zero,
    so the top d digits ARE the d-digit expansion and row i == Algorithm 2 with s = d."""
    prec = 64
    A, B = rand_small(7, 6, 5, 4, prec, 0)
    s_max = 16
    srow = [10, 16, 11, 12, 14, 10]
    C = oracle.ozaki_rows(A, B, prec, method, s_max, srow)
    for i, d in enumerate(srow):
        R = oracle.ozaki(A.rows(i, i + 1), B, prec, method, d)
        assert same_bits(C.rows(i, i + 1), R), (i, d)


@pytest.mark.parametrize("method", ["3M", "4M"])
@pytest.mark.parametrize("prec,spread,k", [(128, 16, 7), (192, 8, 12), (96, 24, 4)])
def test_rows_error_bound_vs_exact(method, prec, spread, k):
    cM = 3.0 if method == "4M" else 4.0
    A, B = rand_small(prec + k, 6, k, 5, prec, spread, zero_frac=0.05)
    s_glob, ok = oracle.auto_slices(A, B, prec, method)
    assert ok
    rng = np.random.default_rng(prec + spread)
    srow = [int(x) for x in rng.integers(max(2, s_glob - 4), s_glob + 1, size=6)]
    s_max = s_glob + 3                               # digits from a longer expansion
    Cz = oracle.ozaki_rows(A, B, prec, method, s_max, srow)
    Cx = oracle.exact(A, B, prec + 64, method)
    lr, si, sj = rho_ij_log2(A, B)
    den = log2_absab(A, B, si, sj)
    for t in range(len(si)):
        num = log2_diff(Cz, Cx, si[t], sj[t], si[t], sj[t])
        if num == -math.inf:
            continue
        d = srow[si[t]]
        bound = math.log2(cM * d * 2.0 ** (4 - 8 * d + lr[t]) + 2.0 ** -prec)
        assert num - den[t] <= bound + 1e-9, (si[t], d)


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_block_slices_certified(method):
    """Rows of very different scale structure: a block with a wide exponent spread needs more
    slices than a block of uniform rows.  Per-block certified s meets the acceptance bound."""
    prec = 128
    A1 = mpgen.random_cmat(3, 1, 4, 9, prec, 0)
    A2 = mpgen.random_cmat(3, 2, 4, 9, prec, 30, zero_frac=0.3)
    A = mpgen._vstack([A1, A2])
    B = mpgen.random_cmat(3, 3, 9, 5, prec, 2)
    sb, ok = oracle.block_slices(A, B, prec, method, block=4)
    s_glob, ok2 = oracle.auto_slices(A, B, prec, method)
    assert ok and ok2 and len(sb) == 2
    assert max(sb) == s_glob and min(sb) <= s_glob
    assert sb[0] < sb[1]
    srow = [sb[i // 4] for i in range(8)]
    Cz = oracle.ozaki_rows(A, B, prec, method, max(sb), srow)
    Cx = oracle.exact(A, B, prec + 64, method)
    assert max_err_log2(A, B, Cz, Cx) <= -(prec - (8 if method == "4M" else 9))
    # uniform rows: identical to the global call
    assert same_bits(oracle.ozaki_rows(A, B, prec, method, s_glob, [s_glob] * 8), oracle.ozaki(A, B, prec, method, s_glob))
