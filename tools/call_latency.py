"""Per-call device time (CUDA events, no stage timing) of small and medium calls: the fixed
overhead of one mpcgemm_ex (pre-pass readback, ~12 launches) vs its work."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import mpgen  # noqa: E402
import paper_2307_06072_b200 as P  # noqa: E402

for (m, n, k, prec) in [(64, 64, 64, 128), (256, 256, 32, 256), (992, 992, 32, 256), (512, 512, 512, 256)]:
    A = P.to_device(mpgen.random_cmat(1, 1, m, k, prec, 2))
    B = P.to_device(mpgen.random_cmat(1, 2, k, n, prec, 2))
    C = P.empty_device(m, n, prec)
    for _ in range(3):
        P.mpcgemm_ex(A, B, C, prec, "3M")
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep = P.mpcgemm_ex(A, B, C, prec, "3M")
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{m}x{n}x{k} prec {prec}: {statistics.median(ts) * 1e3:.0f} us per call, s = {rep['slices']}, "
          f"launches {rep['kernel_launches']}", flush=True)
