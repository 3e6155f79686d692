"""Probe of the device MP scalar ops (NEXT-3): one mpc_scalar launch per (op, prec) on
cnt elements, timed with CUDA events; run under ncu for the per-instruction profile."""
import os
import sys
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import mpgen  # noqa: E402
import paper_2307_06072_b200 as P  # noqa: E402

cnt = int(os.environ.get("CNT", "1024"))
for prec in (256, 768):
    X = P.to_device(mpgen.random_cmat(1, 1, 1, cnt, prec, 2))
    Y = P.to_device(mpgen.random_cmat(1, 2, 1, cnt, prec, 2))
    A = P.to_device(mpgen.random_cmat(1, 3, 1, cnt, prec, 2))
    for op in ("fms", "recip"):
        P.mpc_scalar(op, X, Y, A)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.mpc_scalar(op, X, Y, A)
        e1.record()
        torch.cuda.synchronize()
        print(f"prec {prec} op {op} cnt {cnt}: {e0.elapsed_time(e1) * 1e3:.1f} us", flush=True)
