"""Config 5's 15 LU-update GEMMs (768 bits): per-GEMM shape, slice count and stage times (opts.timing),
summed -- where the sequence's time goes.  One JSON line per method."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import mpgen  # noqa: E402
import paper_2307_06072_b200 as P  # noqa: E402

for method in ("3M",):
    tot = {}
    rows = []
    for j, L21, U12 in mpgen.lu_update_gemms(seed=0):
        dA, dB = P.to_device(L21), P.to_device(U12)
        C = P.empty_device(L21.shape[0], U12.shape[1], 768)
        for _ in range(2):
            P.mpcgemm_ex(dA, dB, C, 768, method)
        reps = [P.mpcgemm_ex(dA, dB, C, 768, method, timing=1) for _ in range(3)]
        torch.cuda.synchronize()
        st = {k: min(r[k] for r in reps) for k in ("ms_linemax", "ms_prepass", "ms_split", "ms_gemm", "ms_fold")}
        rows.append({"j": j, "m": L21.shape[0], "n": U12.shape[1], "k": L21.shape[1], "s": reps[0]["slices"],
                     **{k: round(v, 4) for k, v in st.items()}})
        for k, v in st.items():
            tot[k] = tot.get(k, 0) + v
    print(json.dumps({"method": method, "total": {k: round(v, 3) for k, v in tot.items()}, "gemms": rows}))
