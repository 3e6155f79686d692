"""Run the same product several times and compare every output bitwise (race detector for the
slice GEMM and the fold).  Usage: python tools/determinism.py CFG REPS [ENV=VAL ...] (env switches
apply to the runs after the first)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import mpgen  # noqa: E402
import paper_2307_06072_b200 as P  # noqa: E402

cfg, reps = int(sys.argv[1]), int(sys.argv[2])
c = mpgen.CONFIGS[cfg]
A, B = mpgen.config_inputs(cfg, seed=0)
dA, dB = P.to_device(A), P.to_device(B)
ref = P.empty_device(c["m"], c["n"], c["prec"])
P.mpcgemm_ex(dA, dB, ref, c["prec"], "3M")
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    os.environ[k] = v
bad = 0
for t in range(reps):
    C = P.empty_device(c["m"], c["n"], c["prec"])
    P.mpcgemm_ex(dA, dB, C, c["prec"], "3M")
    torch.cuda.synchronize()
    for p in ("re", "im"):
        for f in ("sign", "exp", "limbs"):
            a, b = getattr(getattr(ref, p), f), getattr(getattr(C, p), f)
            if not torch.equal(a, b):
                diff = (a != b)
                if f == "limbs":
                    diff = diff.any(dim=-1)
                idx = diff.nonzero()
                print(f"run {t}: {p}.{f} differs at {idx.shape[0]} entries, first {idx[:4].tolist()}", flush=True)
                bad += 1
print("runs", reps, "mismatching fields", bad, flush=True)
