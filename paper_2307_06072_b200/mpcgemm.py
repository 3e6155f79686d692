"""Thin ctypes binding of libmpcgemm.so (include/mpcgemm.h): argument marshalling only.

Every step of the Ozaki complex MP GEMM runs in the sm_100a kernels behind the C ABI; this
module converts torch tensors / numpy arrays to the ABI's plain pointers.  There is no CPU
fallback: if the shared library is missing or cannot be loaded, every call raises.
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPCGEMM_LIB") or os.path.join(_HERE, "libmpcgemm.so")   # override: A/B testing
_lock = threading.Lock()
_lib = None

METHODS = {"3M": 3, "4M": 4, 3: 3, 4: 4}
ERRORS = {0: "OK", -1: "ERR_ARG", -2: "ERR_PREC", -3: "ERR_EXP_RANGE", -4: "ERR_NOT_NORMALIZED",
          -5: "ERR_ALIAS", -6: "ERR_NOMEM", -7: "ERR_CUDA", -8: "ERR_SLICES"}
SYMBOLS = ["mpcgemm", "mpcgemm_ex", "mpcgemm_host", "mpcgemm_host_async", "mpcgemm_host_wait", "mpcgemm_rho_bounds", "mpcgemm_slices_for",
           "mpcgemm_workspace_size", "mpcgemm_strerror", "mpcgemm_last_error", "mpcgemm_release",
           "mpcgemm_version", "mpclu_factor", "mpclu_solve", "mpc_scalar", "mpcgemm_device_rule_result"]


class MpcgemmError(RuntimeError):
    def __init__(self, code, detail=""):
        super().__init__(f"mpcgemm {ERRORS.get(code, code)} ({code}): {detail}")
        self.code = code


class RMatC(ctypes.Structure):
    _fields_ = [("sign", ctypes.c_void_p), ("exp", ctypes.c_void_p), ("limbs", ctypes.c_void_p), ("ld", ctypes.c_int64)]


class CMatC(ctypes.Structure):
    _fields_ = [("re", RMatC), ("im", RMatC)]


class OptsC(ctypes.Structure):
    _fields_ = [("stream", ctypes.c_void_p), ("slices", ctypes.c_int32), ("validate", ctypes.c_int32),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
                ("timing", ctypes.c_int32), ("beta", ctypes.c_int32), ("alpha_neg", ctypes.c_int32),
                ("carrier", ctypes.c_int32), ("adaptive", ctypes.c_int32),
                ("block_slices", ctypes.c_void_p), ("device_rule", ctypes.c_int32)]


class ReportC(ctypes.Structure):
    _fields_ = [("slices", ctypes.c_int32), ("certified", ctypes.c_int32), ("minT", ctypes.c_int64),
                ("minT1", ctypes.c_int64), ("maxD2", ctypes.c_int64), ("log2_rho_hat", ctypes.c_double),
                ("mma_instructions", ctypes.c_int64), ("work_units", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int32), ("slice_bits", ctypes.c_int32), ("slicegemm_ctas", ctypes.c_int32),
                ("ms_linemax", ctypes.c_float), ("ms_prepass", ctypes.c_float), ("ms_split", ctypes.c_float),
                ("ms_gemm", ctypes.c_float), ("ms_fold", ctypes.c_float), ("slices_min", ctypes.c_int32),
                ("partial_slots", ctypes.c_int32), ("tile_m", ctypes.c_int32), ("tile_n", ctypes.c_int32),
                ("mma_issued", ctypes.c_int64)]


class LuReportC(ctypes.Structure):
    _fields_ = [("info", ctypes.c_int32), ("gemm_calls", ctypes.c_int32), ("slices_max", ctypes.c_int32),
                ("kernel_launches", ctypes.c_int32), ("ms_panel", ctypes.c_float), ("ms_trsm", ctypes.c_float),
                ("ms_gemm", ctypes.c_float)]


def lib():
    """Load libmpcgemm.so (built by __graft_entry__.build()); raises if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
            L = ctypes.CDLL(LIB_PATH)
            i64, i32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
            PC = ctypes.POINTER(CMatC)
            L.mpcgemm.argtypes = [i64, i64, i64, i32, PC, PC, PC, ctypes.c_int]
            L.mpcgemm_ex.argtypes = [i64, i64, i64, i32, PC, PC, PC, ctypes.c_int, ctypes.POINTER(OptsC), ctypes.POINTER(ReportC)]
            L.mpcgemm_host.argtypes = L.mpcgemm_ex.argtypes
            L.mpcgemm_host_async.argtypes = L.mpcgemm_ex.argtypes
            L.mpcgemm_host_wait.argtypes = []
            L.mpcgemm_rho_bounds.argtypes = [i64, i64, i64, i32, PC, PC, i32, ctypes.POINTER(OptsC), ctypes.POINTER(ctypes.c_int64)]
            L.mpcgemm_slices_for.argtypes = [i32, ctypes.c_int, i64, i64, i64, i64]
            L.mpcgemm_workspace_size.argtypes = [i64, i64, i64, i32, ctypes.c_int, i32]
            L.mpcgemm_workspace_size.restype = ctypes.c_size_t
            L.mpcgemm_strerror.argtypes = [ctypes.c_int]
            L.mpcgemm_strerror.restype = ctypes.c_char_p
            L.mpcgemm_last_error.restype = ctypes.c_char_p
            L.mpcgemm_release.restype = None
            L.mpclu_factor.argtypes = [i64, i32, PC, vp, i32, ctypes.c_int, ctypes.POINTER(OptsC), ctypes.POINTER(LuReportC)]
            L.mpclu_solve.argtypes = [i64, i64, i32, PC, vp, PC, ctypes.POINTER(OptsC)]
            L.mpc_scalar.argtypes = [i32, i64, i32, PC, PC, PC, PC, vp, vp]
            L.mpcgemm_device_rule_result.argtypes = [i64, i64, vp, ctypes.POINTER(ctypes.c_int64)]
            L.mpcgemm_device_rule_result.restype = ctypes.c_int
            for name in ("mpcgemm", "mpcgemm_ex", "mpcgemm_host", "mpcgemm_host_async", "mpcgemm_host_wait", "mpcgemm_rho_bounds", "mpcgemm_slices_for", "mpcgemm_version",
                         "mpclu_factor", "mpclu_solve", "mpc_scalar"):
                getattr(L, name).restype = ctypes.c_int
            _lib = L
    return _lib


def _check(rc):
    if rc < 0:
        raise MpcgemmError(rc, lib().mpcgemm_last_error().decode())
    return rc


# ------------------------------------------------------------------ device matrices (torch)
@dataclass
class DevRMat:
    """Real MP matrix in device memory (torch tensors): sign uint8 [rows, ld], exp int64
    [rows, ld], limbs int64 [rows, ld, L] holding the uint64 limb bits."""
    sign: "object"
    exp: "object"
    limbs: "object"
    cols: int

    @property
    def rows(self):
        return self.sign.shape[0]

    @property
    def ld(self):
        return self.sign.shape[1]

    def c(self) -> RMatC:
        return RMatC(self.sign.data_ptr(), self.exp.data_ptr(), self.limbs.data_ptr(), self.ld)


@dataclass
class DevCMat:
    re: DevRMat
    im: DevRMat
    prec: int

    @property
    def shape(self):
        return (self.re.rows, self.re.cols)

    def c(self) -> CMatC:
        return CMatC(self.re.c(), self.im.c())


def _torch():
    import torch
    return torch


def to_device(M, device="cuda", ld: int | None = None, pin: bool = False) -> DevCMat:
    """mpgen.CMat (numpy) -> DevCMat on `device` (optional padded leading dimension)."""
    torch = _torch()

    def one(R):
        rows, cols = R.sign.shape
        l = cols if ld is None else ld
        sign = torch.zeros((rows, l), dtype=torch.uint8, device=device)
        exp = torch.zeros((rows, l), dtype=torch.int64, device=device)
        limbs = torch.zeros((rows, l, R.L), dtype=torch.int64, device=device)
        sign[:, :cols] = torch.from_numpy(R.sign)
        exp[:, :cols] = torch.from_numpy(R.exp)
        limbs[:, :cols] = torch.from_numpy(R.limbs.view(np.int64))
        return DevRMat(sign, exp, limbs, cols)

    return DevCMat(one(M.re), one(M.im), M.prec)


def empty_device(rows: int, cols: int, prec: int, device="cuda", ld: int | None = None) -> DevCMat:
    torch = _torch()
    L = (prec + 63) // 64
    l = cols if ld is None else ld

    def one():
        return DevRMat(torch.zeros((rows, l), dtype=torch.uint8, device=device),
                       torch.zeros((rows, l), dtype=torch.int64, device=device),
                       torch.zeros((rows, l, L), dtype=torch.int64, device=device), cols)

    return DevCMat(one(), one(), prec)


def to_host(D: DevCMat):
    """DevCMat -> mpgen.CMat (numpy)."""
    from mpgen import CMat, RMat

    def one(R):
        c = R.cols
        return RMat(R.sign[:, :c].cpu().numpy().copy(), R.exp[:, :c].cpu().numpy().copy(),
                    R.limbs[:, :c].cpu().numpy().view(np.uint64).copy(), D.prec)

    return CMat(one(D.re), one(D.im))


def _stream_ptr(stream):
    if stream is None:
        torch = _torch()
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


# ------------------------------------------------------------------ the calls (names = ABI)
def mpcgemm_ex(A: DevCMat, B: DevCMat, C: DevCMat, prec: int, method="3M", slices: int = 0,
               validate: int = 0, stream=None, workspace=None, timing: int = 0, beta: int = 0,
               alpha_neg: int = 0, carrier: int = 0, adaptive: int = 0, device_rule: int = 0) -> dict:
    """C := beta C + (-1)^alpha_neg A B on the device (stream-ordered).  Returns the report
    (plus "block_slices": the s of each 256-row block)."""
    m, k = A.shape
    k2, n = B.shape
    if k != k2 or C.shape != (m, n):
        raise MpcgemmError(-1, f"shape mismatch A {A.shape} B {B.shape} C {C.shape}")
    nblk = max(1, (m + 255) // 256)
    bs = (ctypes.c_int32 * nblk)()
    opts = OptsC(_stream_ptr(stream), slices, validate,
                 workspace.data_ptr() if workspace is not None else None,
                 workspace.numel() * workspace.element_size() if workspace is not None else 0, timing, beta,
                 alpha_neg, carrier, adaptive, ctypes.cast(bs, ctypes.c_void_p), device_rule)
    rep = ReportC()
    a, b, c = A.c(), B.c(), C.c()
    rc = lib().mpcgemm_ex(m, n, k, prec, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), METHODS[method],
                          ctypes.byref(opts), ctypes.byref(rep))
    _check(rc)
    return {f: getattr(rep, f) for f, _ in ReportC._fields_} | {"status": rc,
                                                                "block_slices": list(bs)[: (m + 255) // 256]}


def gemm(A: DevCMat, B: DevCMat, prec: int | None = None, method="3M", slices: int = 0, stream=None,
         carrier: int = 0, adaptive: int = 0):
    """Allocating convenience wrapper: returns (C, report)."""
    prec = A.prec if prec is None else prec
    C = empty_device(A.shape[0], B.shape[1], prec, device=A.re.sign.device)
    rep = mpcgemm_ex(A, B, C, prec, method, slices, stream=stream, carrier=carrier, adaptive=adaptive)
    return C, rep


def _host_rmat(R) -> RMatC:
    for a in (R.sign, R.exp, R.limbs):
        assert a.flags["C_CONTIGUOUS"]
    return RMatC(R.sign.ctypes.data, R.exp.ctypes.data, R.limbs.ctypes.data, R.sign.shape[1])


def mpcgemm_host(A, B, prec: int, method="3M", slices: int = 0, C=None, timing: int = 0, beta: int = 0,
                 alpha_neg: int = 0, adaptive: int = 0):
    """End-to-end call on host numpy buffers (mpgen.CMat); returns (C, report)."""
    from mpgen import empty_cmat
    m, k = A.shape
    n = B.shape[1]
    C = empty_cmat(m, n, prec) if C is None else C
    a = CMatC(_host_rmat(A.re), _host_rmat(A.im))
    b = CMatC(_host_rmat(B.re), _host_rmat(B.im))
    c = CMatC(_host_rmat(C.re), _host_rmat(C.im))
    opts = OptsC(None, slices, 0, None, 0, timing, beta, alpha_neg, 0, adaptive, None)
    rep = ReportC()
    rc = lib().mpcgemm_host(m, n, k, prec, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), METHODS[method],
                            ctypes.byref(opts), ctypes.byref(rep))
    _check(rc)
    return C, {f: getattr(rep, f) for f, _ in ReportC._fields_} | {"status": rc}


_pending = []     # host matrices of queued mpcgemm_host_async calls (kept alive until the wait)


def mpcgemm_host_async(A, B, prec: int, method="3M", C=None, slices: int = 0, beta: int = 0, alpha_neg: int = 0,
                       adaptive: int = 0):
    """Queued end-to-end call (C ABI mpcgemm_host_async): returns (C, report) once the device work
    is queued; C is valid on the host after mpcgemm_host_wait().  A, B, C must not be modified before."""
    from mpgen import empty_cmat
    m, k = A.shape
    n = B.shape[1]
    C = empty_cmat(m, n, prec) if C is None else C
    a = CMatC(_host_rmat(A.re), _host_rmat(A.im))
    b = CMatC(_host_rmat(B.re), _host_rmat(B.im))
    c = CMatC(_host_rmat(C.re), _host_rmat(C.im))
    opts = OptsC(None, slices, 0, None, 0, 0, beta, alpha_neg, 0, adaptive, None)
    rep = ReportC()
    _pending.append((A, B, C))
    rc = lib().mpcgemm_host_async(m, n, k, prec, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), METHODS[method],
                                  ctypes.byref(opts), ctypes.byref(rep))
    _check(rc)
    return C, {f: getattr(rep, f) for f, _ in ReportC._fields_} | {"status": rc}


def mpcgemm_host_wait():
    """Blocks until every queued mpcgemm_host_async call has its C on the host."""
    try:
        _check(lib().mpcgemm_host_wait())
    finally:
        _pending.clear()


def mpcgemm_rho_bounds(A: DevCMat, B: DevCMat, prec: int, full: int = 0, stream=None):
    m, k = A.shape
    n = B.shape[1]
    out = (ctypes.c_int64 * 3)()
    opts = OptsC(_stream_ptr(stream), 0, 0, None, 0, 0, 0, 0, 0, 0, None)
    a, b = A.c(), B.c()
    _check(lib().mpcgemm_rho_bounds(m, n, k, prec, ctypes.byref(a), ctypes.byref(b), full, ctypes.byref(opts), out))
    return tuple(int(v) for v in out)


def mpcgemm_device_rule_result(m: int, n: int, stream=None):
    """(status, s, (minT, minT1, maxD2)) of the last device_rule call of shape m x n (synchronizes
    the stream)."""
    out = (ctypes.c_int64 * 4)()
    rc = lib().mpcgemm_device_rule_result(m, n, _stream_ptr(stream), out)
    if rc < 0 and rc != -8:
        _check(rc)
    return rc, int(out[0]), (int(out[1]), int(out[2]), int(out[3]))


def mpcgemm_slices_for(prec: int, method, k: int, minT: int, minT1: int, maxD2: int) -> int:
    return _check(lib().mpcgemm_slices_for(prec, METHODS[method], k, minT, minT1, maxD2))


def mpcgemm_workspace_size(m, n, k, prec, method, slices) -> int:
    return int(lib().mpcgemm_workspace_size(m, n, k, prec, METHODS[method], slices))


def mpcgemm_release():
    lib().mpcgemm_release()


def mpcgemm_version() -> int:
    return lib().mpcgemm_version()


def mpcgemm_strerror(code: int) -> str:
    return lib().mpcgemm_strerror(code).decode()


# ------------------------------------------------------------------ NEXT-3: complex LU
def mpclu_factor(A: DevCMat, K: int, method="3M", prec: int | None = None, stream=None, timing: int = 0,
                 adaptive: int = 0, ipiv=None):
    """In-place blocked complex LU of the n x n device matrix A (mpclu_factor).  Returns
    (ipiv torch int64 tensor, report dict)."""
    torch = _torch()
    prec = A.prec if prec is None else prec
    n = A.shape[0]
    if A.shape != (n, n):
        raise MpcgemmError(-1, f"A must be square, got {A.shape}")
    if ipiv is None:
        ipiv = torch.empty(max(n, 1), dtype=torch.int64, device=A.re.sign.device)
    opts = OptsC(_stream_ptr(stream), 0, 0, None, 0, timing, 0, 0, 0, adaptive, None)
    rep = LuReportC()
    a = A.c()
    _check(lib().mpclu_factor(n, prec, ctypes.byref(a), ipiv.data_ptr(), K, METHODS[method], ctypes.byref(opts),
                              ctypes.byref(rep)))
    return ipiv[:n], {f: getattr(rep, f) for f, _ in LuReportC._fields_}


def mpclu_solve(F: DevCMat, ipiv, B: DevCMat, prec: int | None = None, stream=None):
    """B := A^-1 B in place with the factors of mpclu_factor (Eq. 7)."""
    prec = F.prec if prec is None else prec
    n = F.shape[0]
    if B.shape[0] != n:
        raise MpcgemmError(-1, f"B has {B.shape[0]} rows, LU is {n} x {n}")
    opts = OptsC(_stream_ptr(stream), 0, 0, None, 0, 0, 0, 0, 0, 0, None)
    f, b = F.c(), B.c()
    _check(lib().mpclu_solve(n, B.shape[1], prec, ctypes.byref(f), ipiv.data_ptr(), ctypes.byref(b), ctypes.byref(opts)))


def mpc_scalar(op: str, X: DevCMat, Y: DevCMat | None = None, A: DevCMat | None = None, prec: int | None = None,
               stream=None):
    """Elementwise device MP scalar ops on 1 x cnt matrices: "mul", "fms" (A - X Y), "recip",
    "key" (returns a torch int64 [cnt, 2] tensor of (e, v bits))."""
    torch = _torch()
    prec = X.prec if prec is None else prec
    cnt = X.shape[1]
    opn = {"mul": 0, "fms": 1, "recip": 2, "key": 3}[op]
    dev = X.re.sign.device
    O = empty_device(1, cnt, prec, device=dev) if op != "key" else None
    kv = torch.zeros((max(cnt, 1), 2), dtype=torch.int64, device=dev) if op == "key" else None
    x = X.c()
    y = Y.c() if Y is not None else None
    a = A.c() if A is not None else None
    o = O.c() if O is not None else None
    _check(lib().mpc_scalar(opn, cnt, prec, ctypes.byref(a) if a else None, ctypes.byref(x),
                            ctypes.byref(y) if y else None, ctypes.byref(o) if o else None,
                            kv.data_ptr() if kv is not None else None, _stream_ptr(stream)))
    return kv[:cnt] if op == "key" else O
