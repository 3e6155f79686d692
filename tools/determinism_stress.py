"""Race stress: many shapes x methods x paths, each call repeated; every repeat must give the first
call's bits (the path is exact integer arithmetic + one rounding).  Usage: python tools/determinism_stress.py REPS"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import mpgen  # noqa: E402
import paper_2307_06072_b200 as P  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
shapes = [(64, 64, 64, 128, 0), (130, 100, 97, 192, 3), (300, 520, 200, 256, 2), (512, 512, 512, 256, 4),
          (260, 300, 1400, 320, 1), (900, 1000, 300, 512, 16), (1024, 1024, 1024, 512, 16)]
bad = total = 0
for (m, n, k, prec, sp) in shapes:
    A = mpgen.random_cmat(m + k, 1, m, k, prec, sp)
    B = mpgen.random_cmat(m + k, 2, k, n, prec, sp)
    dA, dB = P.to_device(A), P.to_device(B)
    for method in ("3M", "4M"):
        for dr in (0, 1):
            C0 = P.empty_device(m, n, prec)
            P.mpcgemm_ex(dA, dB, C0, prec, method, device_rule=dr)
            C1 = P.empty_device(m, n, prec)
            for _ in range(reps):
                P.mpcgemm_ex(dA, dB, C1, prec, method, device_rule=dr)
                torch.cuda.synchronize()
                total += 1
                same = all(torch.equal(getattr(getattr(C0, p), f), getattr(getattr(C1, p), f))
                           for p in ("re", "im") for f in ("sign", "exp", "limbs"))
                if not same:
                    bad += 1
                    print("MISMATCH", (m, n, k, prec, method, dr), flush=True)
print("calls", total, "mismatches", bad, flush=True)
