"""Probe of the device MP scalar ops (NEXT-3): per (op, prec), the device time of one
mpc_scalar launch on cnt elements (CUDA events, median of 20 back-to-back launches); cnt = 1
is the latency the LU panel's per-column chain sees.  Also run under ncu for the
per-instruction profile.  usage: CNT=1 python tools/mp_scalar_probe.py"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import mpgen  # noqa: E402
import paper_2307_06072_b200 as P  # noqa: E402

cnt = int(os.environ.get("CNT", "1"))
for prec in (256, 512, 768, 1024):
    X = P.to_device(mpgen.random_cmat(1, 1, 1, cnt, prec, 2))
    Y = P.to_device(mpgen.random_cmat(1, 2, 1, cnt, prec, 2))
    A = P.to_device(mpgen.random_cmat(1, 3, 1, cnt, prec, 2))
    res = {}
    for op in ("mul", "fms", "recip"):
        P.mpc_scalar(op, X, Y, A)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            P.mpc_scalar(op, X, Y, A)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        res[op] = round(statistics.median(ts), 1)
    print(f"prec {prec} cnt {cnt}: us per launch {res}", flush=True)
