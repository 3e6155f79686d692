"""A small 3M and 4M call (pair kernel, fold, split) for compute-sanitizer."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import mpgen  # noqa: E402
import paper_2307_06072_b200 as P  # noqa: E402

A = mpgen.random_cmat(1, 1, 260, 140, 192, 3)
B = mpgen.random_cmat(1, 2, 140, 300, 192, 3)
dA, dB = P.to_device(A), P.to_device(B)
for method in ("3M", "4M"):
    C, rep = P.gemm(dA, dB, 192, method)
    torch.cuda.synchronize()
print("done", rep["slices"])
