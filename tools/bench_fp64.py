"""NEXT-1 measurement: the binary64-carrier variant (FP64 DMMA, the paper's slice width) vs
the INT8/tcgen05 carrier on BASELINE configs 2-4 (3M), plus the FP64 tensor ceiling measured
with the library GEMM torch.matmul(float64) 8192^3.  JSON to stdout."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import mpgen  # noqa: E402
import paper_2307_06072_b200 as P  # noqa: E402


def fp64_peak():
    N = 8192
    a = torch.randn(N, N, dtype=torch.float64, device="cuda")
    b = torch.randn(N, N, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return 2.0 * N ** 3 / best / 1e12


def main():
    out = {"fp64_matmul_tflops": fp64_peak(), "rows": []}
    for cfg in (2, 3, 4):
        c = mpgen.CONFIGS[cfg]
        A, B = mpgen.config_inputs(cfg, seed=0)
        dA, dB = P.to_device(A), P.to_device(B)
        dC = P.empty_device(c["m"], c["n"], c["prec"])
        for carrier in (0, 1):
            steps = 2 if (carrier == 1 and cfg == 4) else 3
            P.mpcgemm_ex(dA, dB, dC, c["prec"], "3M", carrier=carrier)
            torch.cuda.synchronize()
            ts, reps = [], []
            for _ in range(steps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                reps.append(P.mpcgemm_ex(dA, dB, dC, c["prec"], "3M", carrier=carrier, timing=1))
                e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            s, b = reps[-1]["slices"], reps[-1]["slice_bits"]
            cm = c["m"] * c["n"] * c["k"]
            gms = statistics.median(r["ms_gemm"] for r in reps)
            flops = 2.0 * 3 * s * (s + 1) / 2 * cm                 # fp64 flops or int8 ops
            out["rows"].append({"config": cfg, "carrier": "fp64-dmma" if carrier else "int8-tcgen05", "slices": s,
                                "slice_bits": b, "ms": statistics.median(ts), "cmac_per_s": cm / (statistics.median(ts) / 1e3),
                                "gemm_ms": gms, "gemm_tera_ops": flops / (gms / 1e3) / 1e12,
                                "stages_ms": {f: round(statistics.median(r[f] for r in reps), 3)
                                              for f in ("ms_linemax", "ms_prepass", "ms_split", "ms_gemm", "ms_fold")}})
            print(json.dumps(out["rows"][-1]), file=sys.stderr, flush=True)
        del dA, dB, dC
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
