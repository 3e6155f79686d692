"""NEXT-4 measurement: one call with a single certified slice count vs per-256-row-block counts
(opts.adaptive) on a GRADED workload whose row blocks have different exponent spreads (the BASELINE
configs are homogeneous: every block certifies the same s there, see profiles/README.md).

A: m x k, row block b (256 rows) has Re/Im = u 2^e with e uniform in [-4b, 4b] (b = 0..m/256-1);
B: k x n uniform in [-1, 1).  Device time per call (CUDA events, median of 5 after 2 warm-ups).
usage: python tools/bench_adaptive.py [--m 2048] [--n 2048] [--k 2048] [--prec 512]"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import mpgen  # noqa: E402
import paper_2307_06072_b200 as P  # noqa: E402


def graded(m, k, prec, seed=0):
    blocks = [mpgen.random_cmat(seed, 80 + b, min(256, m - 256 * b), k, prec, 4 * b) for b in range((m + 255) // 256)]
    return mpgen._vstack(blocks)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=2048)
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--k", type=int, default=2048)
    ap.add_argument("--prec", type=int, default=512)
    args = ap.parse_args()
    A = graded(args.m, args.k, args.prec)
    B = mpgen.random_cmat(0, 90, args.k, args.n, args.prec)
    dA, dB = P.to_device(A), P.to_device(B)
    dC = P.empty_device(args.m, args.n, args.prec)
    res = {"workload": "graded rows (block b: exponent spread +-4b)", "m": args.m, "n": args.n, "k": args.k,
           "prec": args.prec}
    for method in ("3M", "4M"):
        for adaptive in (0, 1):
            for _ in range(2):
                P.mpcgemm_ex(dA, dB, dC, args.prec, method, adaptive=adaptive)
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rep = P.mpcgemm_ex(dA, dB, dC, args.prec, method, adaptive=adaptive)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[f"{method}_adaptive{adaptive}"] = {"ms": statistics.median(ts), "block_slices": rep["block_slices"],
                                                   "mma_instructions": rep["mma_instructions"]}
        a0, a1 = res[f"{method}_adaptive0"], res[f"{method}_adaptive1"]
        res[f"{method}_speedup"] = a0["ms"] / a1["ms"]
        res[f"{method}_mma_ratio"] = a1["mma_instructions"] / a0["mma_instructions"]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
