"""NEXT-3 measurement: the paper's complex LU benchmark (Eq. 7, Tables 2-3)
on one B200 through the C ABI (mpclu_factor + mpclu_solve).

A: n x n, Re/Im uniform in [-1, 1) with full random mantissas (reading Z14), x_k = k + k i,
b = A x by the library's own Ozaki GEMM at the working precision (certified error
<= 2^-(prec-8) relative to |A||x|; the paper computes b at 2048 bits -- this substitution only
adds that bound to the measured solution error).  Times are CUDA events on the launching
stream around the in-place factorization of a fresh copy of A (warm-up run first); the phase
split comes from a separate opts.timing run (it synchronizes per phase).  One JSON line per
(prec, K).  The paper's Xeon W-2295 / EPYC 7402P seconds (Tables 2-3) are printed as context.

usage: python tools/bench_lu.py [--n 1024] [--precs 256,512,768] [--Ks 32,64,128,256] [--method 3M]
"""
import argparse
import json
import math
import os
import sys
import time
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import mpgen  # noqa: E402
import paper_2307_06072_b200 as P  # noqa: E402

PAPER = {  # PAPER.md Tables 2 (Xeon) and 3 (EPYC): fastest Ozaki LU and Normal LU, seconds, n = 1024
    256: {"xeon_oz": (116.6, 352, 13), "xeon_normal": 134.1, "epyc_oz": (171.1, 384, 13), "epyc_normal": 184.1},
    512: {"xeon_oz": (209.0, 992, 25), "xeon_normal": 181.7, "epyc_oz": (279.6, 992, 25), "epyc_normal": 237.8},
    768: {"xeon_oz": (287.6, 992, 37), "xeon_normal": 253.0, "epyc_oz": (377.5, 992, 37), "epyc_normal": 334.9},
}


def x_exact(n, prec):
    """x_k = k + k i (k = 1..n) as an n x 1 CMat (exact)."""
    X = mpgen.CMat(mpgen.empty_rmat(n, 1, prec), mpgen.empty_rmat(n, 1, prec))
    L = X.re.L
    for k in range(1, n + 1):
        e = k.bit_length()
        M = k << (64 * L - e)
        for R in (X.re, X.im):
            R.exp[k - 1, 0] = e
            for l in range(L):
                R.limbs[k - 1, 0, l] = (M >> (64 * l)) & ((1 << 64) - 1)
    return X


def frac(R, i, j):
    N = 0
    for l in range(R.L - 1, -1, -1):
        N = (N << 64) | int(R.limbs[i, j, l])
    if N == 0:
        return Fraction(0)
    v = Fraction(N) * Fraction(2) ** (int(R.exp[i, j]) - 64 * R.L)
    return -v if R.sign[i, j] else v


def clone(D):
    return P.DevCMat(*(P.DevRMat(r.sign.clone(), r.exp.clone(), r.limbs.clone(), r.cols) for r in (D.re, D.im)), D.prec)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--precs", default="256,512,768")
    ap.add_argument("--Ks", default="32,64,128,256")
    ap.add_argument("--method", default="3M")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    n = args.n
    for prec in [int(p) for p in args.precs.split(",")]:
        A = mpgen.random_cmat(args.seed, 70, n, n, prec)
        dA0 = P.to_device(A)
        dX = P.to_device(x_exact(n, prec))
        dB0, _ = P.gemm(dA0, dX, prec, "4M")                  # b = A x (certified, working prec)
        for K in [int(k) for k in args.Ks.split(",")]:
            d = clone(dA0)
            ipiv, rep = P.mpclu_factor(d, K, args.method)    # warm-up (plans, workspace)
            torch.cuda.synchronize()
            times = []
            for _ in range(args.reps):
                d = clone(dA0)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ipiv, rep = P.mpclu_factor(d, K, args.method)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            dW = clone(dB0)                                   # warm-up solve (first launches load kernels)
            P.mpclu_solve(d, ipiv, dW)
            torch.cuda.synchronize()
            dB = clone(dB0)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            P.mpclu_solve(d, ipiv, dB)
            s1.record()
            torch.cuda.synchronize()
            Xh = P.to_host(dB)
            err = 0.0
            for k in range(n):
                xr = frac(Xh.re, k, 0) - (k + 1)
                xi = frac(Xh.im, k, 0) - (k + 1)
                ek = math.hypot(float(xr), float(xi)) / (math.sqrt(2) * (k + 1))
                err = max(err, ek)
            dt = clone(dA0)
            _, rt = P.mpclu_factor(dt, K, args.method, timing=1)
            line = {"workload": "complex LU + Eq. 7 solve (PAPER.md:243-263)", "n": n, "prec": prec, "K": K,
                    "method": args.method, "ms_factor": min(times), "ms_solve": s0.elapsed_time(s1),
                    "info": rep["info"], "gemm_calls": rep["gemm_calls"], "slices_max": rep["slices_max"],
                    "kernel_launches": rep["kernel_launches"],
                    "phases_ms": {"panel": rt["ms_panel"], "trsm": rt["ms_trsm"], "gemm": rt["ms_gemm"]},
                    "max_rel_err_x": err, "log10_err": math.log10(err) if err > 0 else None,
                    "paper_context_s": PAPER.get(prec)}
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
