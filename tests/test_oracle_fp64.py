"""Pins for the NEXT-1 variant: the same Algorithm 2 with the paper's own slice width,
b = 53 - ceil((53 + ceil(log2 k)) / 2) (tau), i.e. the binary64
slice carrier.  The paper prints the division counts at which the error stops decreasing:
d >= 13 (256 bits), 25 (512), 37 (768) (again PAPER.md:302), for its k = 1024
runs; the oracle must reproduce exactly these saturation points."""
import math

import numpy as np
import pytest

import mpgen
import oracle
from harness import max_err_log2, same_bits, to_fraction

D_STAR = {256: 13, 512: 25, 768: 37}


def test_slice_width_formula():
    """(k=1024) -> b = 21 (53 - 32); (k=256) -> 22; k=1 -> 26."""
    assert oracle.fp64_slice_bits(1024) == 21
    assert oracle.fp64_slice_bits(256) == 22
    assert oracle.fp64_slice_bits(2048) == 21
    assert oracle.fp64_slice_bits(1) == 26
    # d* = ceil(prec / b): 13 / 25 / 37 at k = 1024, 12 at (256, 256)
    assert [math.ceil(p / oracle.fp64_slice_bits(1024)) for p in (256, 512, 768)] == [13, 25, 37]
    assert math.ceil(256 / oracle.fp64_slice_bits(256)) == 12


@pytest.mark.parametrize("prec", [256, 512, 768])
def test_paper_division_thresholds(prec):
    """Error of the b = 21 scheme vs the exact product: still falling at d* - 1, saturated at
    the 2^-prec rounding floor from d* on -- d* = 13 / 25 / 37 as printed in PAPER.md:213."""
    k = 1024
    A = mpgen.random_cmat(5, 1, 3, k, prec)
    B = mpgen.random_cmat(5, 2, k, 3, prec)
    si, sj = np.array([0, 1, 2, 2]), np.array([2, 0, 1, 2])
    X = oracle.exact(A, B, prec + 64, "3M", samples=(si, sj))
    err = {}
    for d in range(D_STAR[prec] - 2, D_STAR[prec] + 3):
        C = oracle.ozaki_bits(A, B, prec, "3M", d, 21, samples=(si, sj))
        err[d] = max_err_log2(A, B, C, X, samples=(si, sj), ref_is_sampled=True, c_is_sampled=True)
    ds = D_STAR[prec]
    assert err[ds - 1] > err[ds] + 5                      # still improving at d* - 1
    assert err[ds] <= -(prec - 1)                          # at the floor from d* on
    assert err[ds + 1] == err[ds] and err[ds + 2] == err[ds]
    assert err[ds - 2] > err[ds - 1] + 15                  # ~b bits per division below d*


@pytest.mark.parametrize("bits", [21, 22, 26])
def test_split_bits_reconstruct(bits):
    """b-bit balanced digits reconstruct the fixed-point value (W = b s - 3)."""
    from fractions import Fraction
    s = 9
    P = mpgen.random_cmat(13, 3, 4, 5, 128, 6, zero_frac=0.1)
    W = bits * s - 3
    dig = oracle.split_bits(P, 0, s, bits, 3)
    half = 1 << (bits - 1)
    for i in range(4):
        e = max([int(R.exp[i, q]) for R in (P.re, P.im) for q in range(5) if R.limbs[i, q, -1] != 0] or [0])
        for q in range(5):
            X = []
            for R in (P.re, P.im):
                a = abs(to_fraction(R, i, q)) * Fraction(2) ** (W - e)
                v = a.numerator // a.denominator
                X.append(-v if R.sign[i, q] and R.limbs[i, q, -1] else v)
            X.append(X[0] + X[1])
            for part in range(3):
                d = [int(v) for v in dig[part, :, i, q]]
                assert all(-half <= v < half for v in d)
                assert sum(v * (1 << (bits * (s - 1 - a))) for a, v in enumerate(d)) == X[part]


def test_bits8_equals_int8_path():
    """b = 8 through the generalized entry == the INT8-carrier oracle (same definition)."""
    A = mpgen.random_cmat(21, 1, 5, 9, 192, 5)
    B = mpgen.random_cmat(21, 2, 9, 6, 192, 5)
    for method in ("3M", "4M"):
        assert same_bits(oracle.ozaki_bits(A, B, 192, method, 26, 8), oracle.ozaki(A, B, 192, method, 26))


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_fp64_rule_meets_bound(method):
    """The slice rule with b-bit digits (b s >= prec - 4 + log2(c_M s rho) + 0.1) meets
    BASELINE's bound against the exact product."""
    prec, k = 256, 64
    A = mpgen.random_cmat(31, 1, 5, k, prec, 4)
    B = mpgen.random_cmat(31, 2, k, 5, prec, 4)
    b = oracle.fp64_slice_bits(k)
    d = oracle.slices_for_bits(prec, method, k, *oracle.rho_bounds(A, B), b)
    C = oracle.ozaki_bits(A, B, prec, method, d, b)
    X = oracle.exact(A, B, prec + 64, method)
    assert max_err_log2(A, B, C, X) <= -(prec - (8 if method == "4M" else 9))
