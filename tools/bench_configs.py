"""Sweep of the BASELINE configs (1-5) x {3M, 4M} on one GPU: device time per call (CUDA events,
median of K after W warm-ups, no per-stage synchronisation), CMAC/s, slice count, slice-GEMM INT8 TOP/s and its fraction of
the peak used by bench.py, per-stage ms.  Config 5 = the sum over its 15 LU-update GEMMs.
Writes one JSON document to stdout.  (Evidence for profiles/, not the driver's bench line.)
ADAPTIVE=1: NEXT-4 per-256-row-block slice counts (opts.adaptive); CONFIGS=1,2,..: subset."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import mpgen  # noqa: E402
import paper_2307_06072_b200 as P  # noqa: E402


ADAPTIVE = int(os.environ.get("ADAPTIVE", "0"))


def time_call(dA, dB, dC, prec, method, steps, warmup):
    """Device time per call without per-stage synchronisation (median), plus the stage split
    from separate opts.timing calls (they synchronize per stage)."""
    for _ in range(warmup):
        P.mpcgemm_ex(dA, dB, dC, prec, method, adaptive=ADAPTIVE)
    torch.cuda.synchronize()
    ts, reps = [], []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.mpcgemm_ex(dA, dB, dC, prec, method, adaptive=ADAPTIVE)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    for _ in range(max(1, min(steps, 3))):
        reps.append(P.mpcgemm_ex(dA, dB, dC, prec, method, timing=1, adaptive=ADAPTIVE))
    torch.cuda.synchronize()
    return statistics.median(ts), reps


def main():
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    peak = 2.0 * peaks["bf16_tflops_sustained"]
    out = {"peak_int8_tops": peak, "adaptive": ADAPTIVE, "configs": []}
    cfgs = [int(c) for c in os.environ.get("CONFIGS", "1,2,3,4,5").split(",")]
    for cfg in cfgs:
        for method in ("3M", "4M"):
            R = 3 if method == "3M" else 4
            if cfg <= 4:
                c = mpgen.CONFIGS[cfg]
                A, B = mpgen.config_inputs(cfg, seed=0)
                dA, dB = P.to_device(A), P.to_device(B)
                dC = P.empty_device(c["m"], c["n"], c["prec"])
                steps = 5 if cfg >= 3 else 20
                ms, reps = time_call(dA, dB, dC, c["prec"], method, steps, 3)
                s = reps[-1]["slices"]
                cm = c["m"] * c["n"] * c["k"]
                ops = 2.0 * R * s * (s + 1) / 2 * cm
                gms = statistics.median(r["ms_gemm"] for r in reps)
                out["configs"].append({"config": cfg, "method": method, "prec": c["prec"], "shape": [c["m"], c["n"], c["k"]],
                                       "slices": s, "block_slices": reps[-1]["block_slices"], "ms": ms, "cmac_per_s": cm / (ms / 1e3),
                                       "gemm_ms": gms, "gemm_tops": ops / (gms / 1e3) / 1e12,
                                       "gemm_frac": ops / (gms / 1e3) / 1e12 / peak,
                                       "stages_ms": {f: statistics.median(r[f] for r in reps) for f in
                                                     ("ms_linemax", "ms_prepass", "ms_split", "ms_gemm", "ms_fold")}})
                del dA, dB, dC
            else:
                tot_ms, tot_cm, tot_ops, tot_g, ss = 0.0, 0, 0.0, 0.0, []
                st = {f: 0.0 for f in ("ms_linemax", "ms_prepass", "ms_split", "ms_gemm", "ms_fold")}
                for j, L21, U12 in mpgen.lu_update_gemms(seed=0):
                    dA, dB = P.to_device(L21), P.to_device(U12)
                    mm, kk = L21.shape
                    nn = U12.shape[1]
                    dC = P.empty_device(mm, nn, mpgen.LU_PREC)
                    ms, reps = time_call(dA, dB, dC, mpgen.LU_PREC, method, 3, 2)
                    s = reps[-1]["slices"]
                    ss.append(reps[-1]["block_slices"] if ADAPTIVE else s)
                    tot_ms += ms
                    tot_cm += mm * nn * kk
                    tot_ops += 2.0 * R * s * (s + 1) / 2 * mm * nn * kk
                    tot_g += statistics.median(r["ms_gemm"] for r in reps)
                    for f in st:
                        st[f] += statistics.median(r[f] for r in reps)
                out["configs"].append({"config": 5, "method": method, "prec": mpgen.LU_PREC, "gemms": 15,
                                       "slices": ss, "ms": tot_ms, "cmac_per_s": tot_cm / (tot_ms / 1e3),
                                       "gemm_ms": tot_g, "gemm_tops": tot_ops / (tot_g / 1e3) / 1e12,
                                       "gemm_frac": tot_ops / (tot_g / 1e3) / 1e12 / peak, "stages_ms": st})
            torch.cuda.empty_cache()
    by = {(c["config"], c["method"]): c for c in out["configs"]}
    out["ratio_3m_over_4m_time"] = {cfg: by[(cfg, "3M")]["ms"] / by[(cfg, "4M")]["ms"] for cfg in cfgs}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
