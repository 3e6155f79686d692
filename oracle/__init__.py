"""CPU oracle (TEST INFRASTRUCTURE ONLY) -- ctypes wrapper around oracle/mpref.c.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module.  It never imports the CUDA path (paper_2307_06072_b200) and the
CUDA path never imports it.  See oracle/mpref.c for the paper passages each function
follows, and DESIGN.md "Oracle" for the readings.

Pins (tests/test_oracle_*.py): brute-force Fractions on 2x2/3x3, independent RNE,
B = I, integer-entry closure, SPEC worked examples, 3M == 4M exact, scaling, transposition,
zero rows, rounded-mode 3M/4M agreement; the Ozaki oracle is pinned by digit-reconstruction
identities, exact closure, the closed-form error bound and the s-saturation sweep.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

from mpgen import CMat, RMat, empty_rmat, limbs_for

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mpref.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/mpref.c -> oracle/liboracle.so (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _RM(ctypes.Structure):
    _fields_ = [("sign", ctypes.c_void_p), ("exp", ctypes.c_void_p), ("limbs", ctypes.c_void_p),
                ("ld", ctypes.c_int64), ("L", ctypes.c_int32), ("pad_", ctypes.c_int32)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.POINTER(_RM)
            i64, i32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
            L.orc_cgemm_exact.argtypes = [i64, i64, i64, P, P, P, P, P, P, i32, i32, i32, i64, vp, vp, i32]
            L.orc_cgemm_exact.restype = ctypes.c_int
            L.orc_cgemm_ozaki.argtypes = [i64, i64, i64, P, P, P, P, P, P, i32, i32, i32, i64, vp, vp, i32]
            L.orc_cgemm_ozaki.restype = ctypes.c_int
            L.orc_cgemm_ozaki_acc.argtypes = [i64, i64, i64, P, P, P, P, P, P, i32, i32, P, P, i32, i32, i32, i64, vp, vp, i32]
            L.orc_cgemm_ozaki_acc.restype = ctypes.c_int
            L.orc_cgemm_ozaki_rows.argtypes = [i64, i64, i64, P, P, P, P, P, P, i32, i32, i32, vp, i64, vp, vp, i32]
            L.orc_cgemm_ozaki_rows.restype = ctypes.c_int
            L.orc_cgemm_ozaki_acc_rows.argtypes = [i64, i64, i64, P, P, P, P, P, P, i32, i32, P, P, i32, i32, i32, vp,
                                                   i64, vp, vp, i32]
            L.orc_cgemm_ozaki_acc_rows.restype = ctypes.c_int
            L.orc_cscalar.argtypes = [i32, i64, i32, P, P, P, P, P, P, P, P, vp]
            L.orc_cscalar.restype = ctypes.c_int
            L.orc_clu_factor.argtypes = [i64, P, P, i32, i32, i32, vp, i32, vp]
            L.orc_clu_factor.restype = ctypes.c_int
            L.orc_clu_solve.argtypes = [i64, P, P, vp, P, P, i64, i32]
            L.orc_clu_solve.restype = ctypes.c_int
            L.orc_cgemm_ozaki_bits.argtypes = [i64, i64, i64, P, P, P, P, P, P, i32, i32, i32, i32, i64, vp, vp, i32]
            L.orc_cgemm_ozaki_bits.restype = ctypes.c_int
            L.orc_split_bits.argtypes = [ctypes.c_int, i64, i64, P, P, i32, i32, i32, vp]
            L.orc_split_bits.restype = ctypes.c_int
            L.orc_fp64_slice_bits.argtypes = [i64]
            L.orc_fp64_slice_bits.restype = ctypes.c_int32
            L.orc_slices_for_bits.argtypes = [i32, i32, i64, i64, i64, i64, i32]
            L.orc_slices_for_bits.restype = ctypes.c_int32
            L.orc_exponents.argtypes = [i64, i64, i64, P, P, P, P, vp, vp, vp, vp]
            L.orc_split.argtypes = [ctypes.c_int, i64, i64, P, P, i32, i32, vp]
            L.orc_split.restype = ctypes.c_int
            L.orc_rho_bounds.argtypes = [i64, i64, i64, P, P, P, P, vp, i32, i32]
            L.orc_rho_bounds.restype = ctypes.c_int
            L.orc_slices_for.argtypes = [i32, i32, i64, i64, i64, i64]
            L.orc_slices_for.restype = ctypes.c_int32
            _lib = L
    return _lib


def _rm(M: RMat) -> _RM:
    for a in (M.sign, M.exp, M.limbs):
        assert a.flags["C_CONTIGUOUS"]
    return _RM(M.sign.ctypes.data, M.exp.ctypes.data, M.limbs.ctypes.data, M.shape[1], M.L, 0)


def _ptr(x):
    return ctypes.byref(x)


def _form(method) -> int:
    return {"3M": 3, "4M": 4, 3: 3, 4: 4}[method]


def _run(fn, A: CMat, B: CMat, prec_out, form, extra, samples, nthreads):
    m, k = A.shape
    k2, n = B.shape
    assert k == k2
    if samples is None:
        Cre, Cim = empty_rmat(m, n, prec_out), empty_rmat(m, n, prec_out)
        ns, si, sj = -1, None, None
    else:
        si = np.ascontiguousarray(np.asarray(samples[0], dtype=np.int64))
        sj = np.ascontiguousarray(np.asarray(samples[1], dtype=np.int64))
        ns = len(si)
        Cre, Cim = empty_rmat(1, max(ns, 1), prec_out), empty_rmat(1, max(ns, 1), prec_out)
    args = [_rm(A.re), _rm(A.im), _rm(B.re), _rm(B.im), _rm(Cre), _rm(Cim)]
    rc = fn(m, n, k, *[_ptr(a) for a in args], prec_out, _form(form), extra, ns,
            si.ctypes.data if si is not None else None, sj.ctypes.data if sj is not None else None, nthreads)
    if rc:
        raise RuntimeError(f"oracle returned {rc}")
    C = CMat(Cre, Cim)
    if samples is not None:
        C = C.cols(0, ns)
    return C


def exact(A: CMat, B: CMat, prec_out: int, method="4M", rounded_prec: int = 0, samples=None, nthreads: int = 0) -> CMat:
    """Plain definition C = AB (Eq. 2 + Eq. 3 for 4M, Eq. 4 for 3M), exact, one RNE to
    prec_out.  rounded_prec > 0: MPC-like per-operation rounding (Eq. 5 / Eq. 6).
    samples = (rows, cols) index arrays -> a 1 x len(samples) result."""
    return _run(lib().orc_cgemm_exact, A, B, prec_out, method, rounded_prec, samples, nthreads)


def ozaki(A: CMat, B: CMat, prec_out: int, method="3M", s: int | None = None, samples=None, nthreads: int = 0) -> CMat:
    """Algorithm 2 step by step (DESIGN.md readings), s slices (auto rule if None)."""
    if s is None:
        s, _ = auto_slices(A, B, A.prec, method)
    return _run(lib().orc_cgemm_ozaki, A, B, prec_out, method, s, samples, nthreads)


def ozaki_rows(A: CMat, B: CMat, prec_out: int, method="3M", s_max: int = 1, srow=None, samples=None,
               nthreads: int = 0) -> CMat:
    """NEXT-4: Algorithm 2 with a per-row triangle d = srow[i] over the top srow[i] digits of
    the s_max-digit expansions (orc_cgemm_ozaki_rows)."""
    srow = np.ascontiguousarray(np.asarray(srow, dtype=np.int32))
    assert srow.shape == (A.shape[0],)

    def fn(m, n, k, a0, a1, b0, b1, c0, c1, prec, form, s, ns, si, sj, nt):
        return lib().orc_cgemm_ozaki_rows(m, n, k, a0, a1, b0, b1, c0, c1, prec, form, s, srow.ctypes.data,
                                          ns, si, sj, nt)
    return _run(fn, A, B, prec_out, method, s_max, samples, nthreads)


def block_slices(A: CMat, B: CMat, prec: int, method, block: int = 256, nthreads: int = 0):
    """NEXT-4: the certified slice rule applied to each block of `block` rows of A (its own
    rho-hat pre-pass over those rows and all of B).  Returns (list of s per block, ok)."""
    m = A.shape[0]
    out, ok = [], True
    for r0 in range(0, m, block):
        s, c = auto_slices(A.rows(r0, min(m, r0 + block)), B, prec, method, nthreads)
        out.append(s)
        ok = ok and c
    return out, ok


def ozaki_acc(A: CMat, B: CMat, C0: CMat, prec_out: int, method="3M", s: int | None = None, beta: int = 1,
              alpha_neg: int = 0, samples=None, nthreads: int = 0, srow=None) -> CMat:
    """C = beta C0 + (-1)^alpha_neg (Algorithm-2 product), exact sum, one RNE (NEXT-2).
    srow: NEXT-4 per-row triangle over the top srow[i] digits of s-digit expansions."""
    if s is None:
        s, _ = auto_slices(A, B, A.prec, method)
    m, k = A.shape
    n = B.shape[1]
    assert C0.shape == (m, n)
    if samples is None:
        Cre, Cim = empty_rmat(m, n, prec_out), empty_rmat(m, n, prec_out)
        ns, si, sj = -1, None, None
    else:
        si = np.ascontiguousarray(np.asarray(samples[0], dtype=np.int64))
        sj = np.ascontiguousarray(np.asarray(samples[1], dtype=np.int64))
        ns = len(si)
        Cre, Cim = empty_rmat(1, max(ns, 1), prec_out), empty_rmat(1, max(ns, 1), prec_out)
    a = [_rm(A.re), _rm(A.im), _rm(B.re), _rm(B.im)]
    c0 = [_rm(C0.re), _rm(C0.im)]
    out = [_rm(Cre), _rm(Cim)]
    sp = si.ctypes.data if si is not None else None
    sq = sj.ctypes.data if sj is not None else None
    if srow is None:
        rc = lib().orc_cgemm_ozaki_acc(m, n, k, *[_ptr(x) for x in a], *[_ptr(x) for x in c0], beta, alpha_neg,
                                       *[_ptr(x) for x in out], prec_out, _form(method), s, ns, sp, sq, nthreads)
    else:
        srow = np.ascontiguousarray(np.asarray(srow, dtype=np.int32))
        assert srow.shape == (m,)
        rc = lib().orc_cgemm_ozaki_acc_rows(m, n, k, *[_ptr(x) for x in a], *[_ptr(x) for x in c0], beta,
                                            alpha_neg, *[_ptr(x) for x in out], prec_out, _form(method), s,
                                            srow.ctypes.data, ns, sp, sq, nthreads)
    if rc:
        raise RuntimeError(f"oracle returned {rc}")
    C = CMat(Cre, Cim)
    if samples is not None:
        C = C.cols(0, ns)
    return C


def fp64_slice_bits(k: int) -> int:
    """b = 53 - ceil((53 + ceil(log2 k)) / 2): the paper's binary64 slice width."""
    return int(lib().orc_fp64_slice_bits(k))


def ozaki_bits(A: CMat, B: CMat, prec_out: int, method="3M", s: int = 1, bits: int = 8, samples=None,
               nthreads: int = 0) -> CMat:
    """The same method with balanced radix-2^bits slices (NEXT-1: bits = fp64_slice_bits(k))."""
    fn = lib().orc_cgemm_ozaki_bits
    m, k = A.shape
    n = B.shape[1]
    if samples is None:
        Cre, Cim = empty_rmat(m, n, prec_out), empty_rmat(m, n, prec_out)
        ns, si, sj = -1, None, None
    else:
        si = np.ascontiguousarray(np.asarray(samples[0], dtype=np.int64))
        sj = np.ascontiguousarray(np.asarray(samples[1], dtype=np.int64))
        ns = len(si)
        Cre, Cim = empty_rmat(1, max(ns, 1), prec_out), empty_rmat(1, max(ns, 1), prec_out)
    args = [_rm(A.re), _rm(A.im), _rm(B.re), _rm(B.im), _rm(Cre), _rm(Cim)]
    rc = fn(m, n, k, *[_ptr(a) for a in args], prec_out, _form(method), s, bits, ns,
            si.ctypes.data if si is not None else None, sj.ctypes.data if sj is not None else None, nthreads)
    if rc:
        raise RuntimeError(f"oracle returned {rc}")
    C = CMat(Cre, Cim)
    return C.cols(0, ns) if samples is not None else C


def split_bits(P: CMat, side: int, s: int, bits: int, nparts: int) -> np.ndarray:
    rows, cols = P.shape
    lines, k = (rows, cols) if side == 0 else (cols, rows)
    dig = np.zeros((nparts, s, lines, k), np.int32)
    rc = lib().orc_split_bits(side, lines, k, _ptr(_rm(P.re)), _ptr(_rm(P.im)), s, bits, nparts, dig.ctypes.data)
    if rc:
        raise RuntimeError(f"orc_split_bits returned {rc}")
    return dig


def slices_for_bits(prec: int, method, k: int, minT: int, minT1: int, maxD2: int, bits: int) -> int:
    return int(lib().orc_slices_for_bits(prec, _form(method), k, minT, minT1, maxD2, bits))


def exponents(A: CMat, B: CMat):
    m, k = A.shape
    n = B.shape[1]
    eA, eB = np.zeros(m, np.int64), np.zeros(n, np.int64)
    nzA, nzB = np.zeros(m, np.uint8), np.zeros(n, np.uint8)
    a = [_rm(A.re), _rm(A.im), _rm(B.re), _rm(B.im)]
    lib().orc_exponents(m, n, k, *[_ptr(x) for x in a], eA.ctypes.data, eB.ctypes.data, nzA.ctypes.data, nzB.ctypes.data)
    return eA, eB, nzA.astype(bool), nzB.astype(bool)


def split(P: CMat, side: int, s: int, nparts: int) -> np.ndarray:
    """Digit planes int8[nparts, s, lines, k]: side 0 = rows of A (P is m x k), side 1 =
    columns of B (P is k x n)."""
    rows, cols = P.shape
    lines, k = (rows, cols) if side == 0 else (cols, rows)
    dig = np.zeros((nparts, s, lines, k), np.int8)
    rc = lib().orc_split(side, lines, k, _ptr(_rm(P.re)), _ptr(_rm(P.im)), s, nparts, dig.ctypes.data)
    if rc:
        raise RuntimeError(f"orc_split returned {rc}")
    return dig


def rho_minT(A: CMat, B: CMat, nthreads: int = 0) -> int:
    return rho_bounds(A, B, nthreads)[0]


def rho_bounds(A: CMat, B: CMat, nthreads: int = 0, full: int = 0):
    """(minT, minT1, maxD2): the integers of the two-stage rho-hat pre-pass."""
    m, k = A.shape
    n = B.shape[1]
    out = (ctypes.c_int64 * 3)()
    a = [_rm(A.re), _rm(A.im), _rm(B.re), _rm(B.im)]
    rc = lib().orc_rho_bounds(m, n, k, *[_ptr(x) for x in a], ctypes.addressof(out), nthreads, full)
    if rc:
        raise RuntimeError(f"orc_rho_bounds returned {rc}")
    return tuple(int(v) for v in out)


def slices_for(prec: int, method, k: int, minT: int, minT1: int | None = None, maxD2: int = -1):
    """The slice-count rule; returns (s, ok)."""
    minT1 = minT if minT1 is None else minT1
    s = lib().orc_slices_for(prec, _form(method), k, minT, minT1, maxD2)
    return s, s > 0


def auto_slices(A: CMat, B: CMat, prec: int, method, nthreads: int = 0):
    return slices_for(prec, method, A.shape[1], *rho_bounds(A, B, nthreads))


# ------------------------------------------------------------------ NEXT-3: complex LU
def cscalar(op: str, X: CMat, Y: CMat | None = None, A: CMat | None = None, prec: int | None = None):
    """Elementwise MPC-style scalar ops on 1 x cnt matrices (orc_cscalar): "mul" = cmul(X, Y),
    "fms" = A - X Y, "recip" = 1 / X (each part one RNE to prec); "key" -> list of pivot keys
    (e, v)."""
    prec = X.prec if prec is None else prec
    cnt = X.shape[1]
    Y = X if Y is None else Y
    A = X if A is None else A
    O = CMat(empty_rmat(1, cnt, prec), empty_rmat(1, cnt, prec))
    kv = np.zeros(2 * max(cnt, 1), np.int64)
    opn = {"mul": 0, "fms": 1, "recip": 2, "key": 3}[op]
    args = [_rm(A.re), _rm(A.im), _rm(X.re), _rm(X.im), _rm(Y.re), _rm(Y.im), _rm(O.re), _rm(O.im)]
    rc = lib().orc_cscalar(opn, cnt, prec, *[_ptr(a) for a in args], kv.ctypes.data)
    if rc:
        raise RuntimeError(f"orc_cscalar returned {rc}")
    if op == "key":
        return [(int(kv[2 * t]), float(kv[2 * t + 1:2 * t + 2].view(np.float64)[0])) for t in range(cnt)]
    return O


def lu_factor(A: CMat, K: int, method="3M", prec: int | None = None, nthreads: int = 0):
    """Blocked right-looking complex LU with partial pivoting and Ozaki GEMM trailing updates
    (orc_clu_factor).  Returns (LU, ipiv, info, smax); A is not modified."""
    prec = A.prec if prec is None else prec
    n = A.shape[0]
    assert A.shape == (n, n)
    F = A.copy()
    ipiv = np.zeros(max(n, 1), np.int64)
    smax = ctypes.c_int32(0)
    info = lib().orc_clu_factor(n, _ptr(_rm(F.re)), _ptr(_rm(F.im)), prec, K, _form(method), ipiv.ctypes.data,
                                nthreads, ctypes.addressof(smax))
    if info < 0:
        raise RuntimeError(f"orc_clu_factor returned {info}")
    return F, ipiv[:n], info, smax.value


def lu_solve(F: CMat, ipiv, B: CMat, prec: int | None = None) -> CMat:
    """Eq. 7 solve with the factors of lu_factor (orc_clu_solve); returns X (B untouched)."""
    prec = F.prec if prec is None else prec
    n = F.shape[0]
    X = B.copy()
    ip = np.ascontiguousarray(np.asarray(ipiv, dtype=np.int64))
    rc = lib().orc_clu_solve(n, _ptr(_rm(F.re)), _ptr(_rm(F.im)), ip.ctypes.data, _ptr(_rm(X.re)), _ptr(_rm(X.im)),
                             X.shape[1], prec)
    if rc:
        raise RuntimeError(f"orc_clu_solve returned {rc}")
    return X
