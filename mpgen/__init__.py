"""Seeded synthetic inputs for the Ozaki complex MP GEMM (shared by the oracle tests
and the CUDA path; holds none of the method's arithmetic).

Element format (the C ABI's, include/mpcgemm.h; MPFR convention, §II):
    value = (-1)^sign * N * 2^(exp - 64*L),  N = sum_l limbs[l] * 2^(64 l),  L = ceil(prec/64)
    nonzero  =>  top bit of limbs[L-1] set and the low 64L-prec bits of N are zero
    zero    <=>  all limbs zero (sign 0, exp 0 by convention)

Distributions (BASELINE.json configs; reading Z14):
  * "uniform in [-1,1) with a full random mantissa": exp = -G, G ~ Geometric(1/2) on {0,1,..}
    (P(G=g) = 2^-(g+1)), mantissa = 1 followed by prec-1 uniform random bits, uniform sign.
    This is the exact law of the prec-bit truncation of a uniform variate in [-1,1).
  * "u * 2^e, e uniform integer in [-E, E]": the above with exp += e.
Every matrix is generated in blocks of ROW_BLOCK rows, each from its own numpy
SeedSequence key (seed, tag, part, row block), so any row range (a rank's shard) can be
generated on its own and is bit-identical to the same rows of the full matrix.
"""
from __future__ import annotations

import dataclasses
import numpy as np

ROW_BLOCK = 128
_PART_ID = {"re": 0, "im": 1}


def limbs_for(prec: int) -> int:
    return (prec + 63) // 64


@dataclasses.dataclass
class RMat:
    """Planar real MP matrix in the ABI element format, row-major, ld == cols."""
    sign: np.ndarray   # uint8  [rows, cols]
    exp: np.ndarray    # int64  [rows, cols]
    limbs: np.ndarray  # uint64 [rows, cols, L]
    prec: int

    @property
    def shape(self):
        return self.sign.shape

    @property
    def L(self):
        return self.limbs.shape[-1]

    def rows(self, r0: int, r1: int) -> "RMat":
        return RMat(self.sign[r0:r1].copy(), self.exp[r0:r1].copy(), self.limbs[r0:r1].copy(), self.prec)

    def cols(self, c0: int, c1: int) -> "RMat":
        return RMat(np.ascontiguousarray(self.sign[:, c0:c1]), np.ascontiguousarray(self.exp[:, c0:c1]),
                    np.ascontiguousarray(self.limbs[:, c0:c1]), self.prec)

    def T(self) -> "RMat":
        return RMat(np.ascontiguousarray(self.sign.T), np.ascontiguousarray(self.exp.T),
                    np.ascontiguousarray(self.limbs.transpose(1, 0, 2)), self.prec)

    def copy(self) -> "RMat":
        return RMat(self.sign.copy(), self.exp.copy(), self.limbs.copy(), self.prec)


@dataclasses.dataclass
class CMat:
    re: RMat
    im: RMat

    @property
    def shape(self):
        return self.re.shape

    @property
    def prec(self):
        return self.re.prec

    def rows(self, r0, r1):
        return CMat(self.re.rows(r0, r1), self.im.rows(r0, r1))

    def cols(self, c0, c1):
        return CMat(self.re.cols(c0, c1), self.im.cols(c0, c1))

    def T(self):
        return CMat(self.re.T(), self.im.T())

    def copy(self):
        return CMat(self.re.copy(), self.im.copy())


def empty_rmat(rows: int, cols: int, prec: int) -> RMat:
    L = limbs_for(prec)
    return RMat(np.zeros((rows, cols), np.uint8), np.zeros((rows, cols), np.int64),
                np.zeros((rows, cols, L), np.uint64), prec)


def empty_cmat(rows, cols, prec) -> CMat:
    return CMat(empty_rmat(rows, cols, prec), empty_rmat(rows, cols, prec))


def _fill_block(rng, nrows, cols, prec, espread, zero_frac):
    L = limbs_for(prec)
    shape = (nrows, cols)
    sign = rng.integers(0, 2, size=shape, dtype=np.uint8)
    g = rng.geometric(0.5, size=shape).astype(np.int64) - 1            # G ~ Geom(1/2) on {0,1,..}
    exp = -g
    if espread:
        exp = exp + rng.integers(-espread, espread + 1, size=shape, dtype=np.int64)
    limbs = rng.integers(0, np.iinfo(np.uint64).max, size=shape + (L,), dtype=np.uint64, endpoint=True)
    limbs[..., L - 1] |= np.uint64(1) << np.uint64(63)                  # normalized: top bit set
    low = 64 * L - prec                                                  # low 64L-prec bits zero
    if low:
        limbs[..., 0] &= ~np.uint64((1 << low) - 1)
    if zero_frac:
        z = rng.random(size=shape) < zero_frac
        sign[z] = 0
        exp[z] = 0
        limbs[z] = 0
    return sign, exp, limbs


def random_rmat(seed: int, tag: int, part: str, rows: int, cols: int, prec: int,
                espread: int = 0, zero_frac: float = 0.0, row0: int = 0) -> RMat:
    """Rows [row0, row0+rows) of the seeded matrix (seed, tag, part)."""
    L = limbs_for(prec)
    out = empty_rmat(rows, cols, prec)
    if rows == 0 or cols == 0:
        return out
    b0, b1 = row0 // ROW_BLOCK, (row0 + rows - 1) // ROW_BLOCK
    for b in range(b0, b1 + 1):
        rng = np.random.default_rng([seed, tag, _PART_ID[part], b])
        s, e, l = _fill_block(rng, ROW_BLOCK, cols, prec, espread, zero_frac)
        lo = max(row0, b * ROW_BLOCK)
        hi = min(row0 + rows, (b + 1) * ROW_BLOCK)
        out.sign[lo - row0:hi - row0] = s[lo - b * ROW_BLOCK:hi - b * ROW_BLOCK]
        out.exp[lo - row0:hi - row0] = e[lo - b * ROW_BLOCK:hi - b * ROW_BLOCK]
        out.limbs[lo - row0:hi - row0] = l[lo - b * ROW_BLOCK:hi - b * ROW_BLOCK]
    assert out.L == L
    return out


def random_cmat(seed, tag, rows, cols, prec, espread=0, zero_frac=0.0, row0=0) -> CMat:
    return CMat(random_rmat(seed, tag, "re", rows, cols, prec, espread, zero_frac, row0),
                random_rmat(seed, tag, "im", rows, cols, prec, espread, zero_frac, row0))


# ---------------------------------------------------------------- BASELINE.json configs
TAG_A, TAG_B, TAG_R = 1, 2, 3

CONFIGS = {
    1: dict(m=64, n=64, k=64, prec=128, espread=0,
            desc="complex square GEMM 64^3, prec 128, Re/Im uniform [-1,1) full mantissa, seed 0"),
    2: dict(m=512, n=512, k=512, prec=256, espread=4,
            desc="complex square GEMM 512^3, prec 256, u*2^e, e uniform in [-4,4]"),
    3: dict(m=1024, n=1024, k=1024, prec=512, espread=16,
            desc="complex square GEMM 1024^3, prec 512, u*2^e, e uniform in [-16,16]"),
    4: dict(m=2048, n=2048, k=2048, prec=1024, espread=0,
            desc="complex square GEMM 2048^3, prec 1024, Re/Im uniform [-1,1) full mantissa"),
}

LU_N, LU_NB, LU_PREC, LU_SHIFT = 2048, 128, 768, -11


def config_inputs(cfg: int, seed: int = 0, row0: int = 0, rows: int | None = None):
    """(A rows [row0,row0+rows), B) for configs 1-4."""
    c = CONFIGS[cfg]
    rows = c["m"] - row0 if rows is None else rows
    A = random_cmat(seed, TAG_A, rows, c["k"], c["prec"], c["espread"], row0=row0)
    B = random_cmat(seed, TAG_B, c["k"], c["n"], c["prec"], c["espread"])
    return A, B


def lu_block(seed: int, bi: int, bj: int, nb: int = LU_NB, prec: int = LU_PREC) -> CMat:
    """Block (bi, bj) of the config-5 stand-in matrix R (reading Z22): uniform [-1,1)
    complex entries, each nb x nb block from its own seed key; + n on the diagonal."""
    tag = 1000 + bi * 64 + bj
    R = random_cmat(seed, TAG_R * 100000 + tag, nb, nb, prec)
    if bi == bj:
        # R + n*I: n = 2048 = 0.1b * 2^12, exactly representable; the real part of the
        # diagonal becomes u + n, which needs rounding -> replace with n exactly (stand-in)
        L = limbs_for(prec)
        for d in range(nb):
            R.re.sign[d, d] = 0
            R.re.exp[d, d] = 12
            R.re.limbs[d, d] = 0
            R.re.limbs[d, d, L - 1] = np.uint64(1) << np.uint64(63)
    return R


def lu_update_gemms(seed: int = 0, n: int = LU_N, nb: int = LU_NB, prec: int = LU_PREC, js=None):
    """Config 5: the Schur-update GEMMs (n - j nb) x nb . nb x (n - j nb), j = 1..n/nb - 1.
    L21 = R[j nb:n, (j-1) nb:j nb] * 2^-11 and U12 = R[(j-1) nb:j nb, j nb:n] (reading Z22).
    Yields (j, L21, U12)."""
    nblk = n // nb
    js = range(1, nblk) if js is None else js
    for j in js:
        col = j - 1
        Lb = [lu_block(seed, bi, col, nb, prec) for bi in range(j, nblk)]
        Ub = [lu_block(seed, col, bj, nb, prec) for bj in range(j, nblk)]
        L21 = _vstack(Lb)
        for part in (L21.re, L21.im):
            nz = part.limbs[..., -1] != 0
            part.exp[nz] += LU_SHIFT
        U12 = _hstack(Ub)
        yield j, L21, U12


def _vstack(blocks):
    def cat(get):
        return RMat(np.concatenate([get(b).sign for b in blocks], 0), np.concatenate([get(b).exp for b in blocks], 0),
                    np.concatenate([get(b).limbs for b in blocks], 0), blocks[0].prec)
    return CMat(cat(lambda b: b.re), cat(lambda b: b.im))


def _hstack(blocks):
    def cat(get):
        return RMat(np.concatenate([get(b).sign for b in blocks], 1), np.concatenate([get(b).exp for b in blocks], 1),
                    np.concatenate([get(b).limbs for b in blocks], 1), blocks[0].prec)
    return CMat(cat(lambda b: b.re), cat(lambda b: b.im))


# ---------------------------------------------------------------- exact small-value helpers
def from_ints(vals, prec: int) -> RMat:
    """Exact MP matrix from a 2-D list of Python ints or (num, pow2) dyadics.
    Test-side constructor (encoding only, no method arithmetic)."""
    rows, cols = len(vals), len(vals[0])
    out = empty_rmat(rows, cols, prec)
    L = out.L
    for i in range(rows):
        for j in range(cols):
            v = vals[i][j]
            num, e2 = (v, 0) if isinstance(v, int) else v
            if num == 0:
                continue
            neg = num < 0
            num = abs(num)
            while num % 2 == 0:
                num //= 2
                e2 += 1
            b = num.bit_length()
            if b > prec:
                raise ValueError("value not representable at prec")
            N = num << (64 * L - b)
            out.sign[i, j] = 1 if neg else 0
            out.exp[i, j] = e2 + b
            for l in range(L):
                out.limbs[i, j, l] = np.uint64((N >> (64 * l)) & ((1 << 64) - 1))
    return out
