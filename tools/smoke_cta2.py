"""Guarded first run of the CTA-pair kernel: one problem, compared with the 1-CTA kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, mpgen
import paper_2307_06072_b200 as P
for (m, n, k, prec) in [(256, 256, 128, 128), (300, 520, 700, 192), (2048, 2048, 2048, 1024)]:
    A = mpgen.random_cmat(1, 1, m, k, prec, 3); B = mpgen.random_cmat(1, 2, k, n, prec, 3)
    dA, dB = P.to_device(A), P.to_device(B)
    out = {}
    for cta2 in ("1", "0"):
        os.environ["MPCGEMM_CTA2"] = cta2
        C, rep = P.gemm(dA, dB, prec, "3M")
        torch.cuda.synchronize()
        out[cta2] = (P.to_host(C), rep)
    a, b = out["1"][0], out["0"][0]
    same = all(np.array_equal(getattr(getattr(a, p), f), getattr(getattr(b, p), f)) for p in ("re", "im") for f in ("sign", "exp", "limbs"))
    print(m, n, k, prec, "s", out["1"][1]["slices"], "ctas", out["1"][1]["slicegemm_ctas"], out["0"][1]["slicegemm_ctas"], "same", same, flush=True)
    assert same
