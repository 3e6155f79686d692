"""One device-rule call each of config 1 and config 2 (3M) and config 5's first GEMM, for an ncu
launch list (per-kernel durations of the small calls)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import mpgen  # noqa: E402
import paper_2307_06072_b200 as P  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "1"
if which in ("1", "2"):
    c = mpgen.CONFIGS[int(which)]
    A, B = mpgen.config_inputs(int(which), seed=0)
    prec = c["prec"]
else:
    _, A, B = next(iter(mpgen.lu_update_gemms(seed=0, js=[int(which[1:])])))
    prec = 768
dA, dB = P.to_device(A), P.to_device(B)
C = P.empty_device(A.shape[0], B.shape[1], prec)
for _ in range(3):
    P.mpcgemm_ex(dA, dB, C, prec, "3M", device_rule=1)
torch.cuda.synchronize()
