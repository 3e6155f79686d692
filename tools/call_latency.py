"""Per-call device time of the small BASELINE configurations: the host slice rule
(pre-pass readback + host plan: the host sleeps in the middle of the call), the device rule
(opts.device_rule: no host synchronisation), and the device rule captured in a CUDA graph
(replays).  Config 1 (64^3, 128 bits), config 2 (512^3, 256 bits), and config 5's sequence of 15
LU-update GEMMs (768 bits).  Prints one JSON object."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import mpgen  # noqa: E402
import paper_2307_06072_b200 as P  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def graph_of(fn):
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        for _ in range(2):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


out = {}
for method in ("3M", "4M"):
    for cfg in (1, 2):
        c = mpgen.CONFIGS[cfg]
        A, B = mpgen.config_inputs(cfg, seed=0)
        dA, dB = P.to_device(A), P.to_device(B)
        C = P.empty_device(c["m"], c["n"], c["prec"])
        host = timed(lambda: P.mpcgemm_ex(dA, dB, C, c["prec"], method))
        dev = timed(lambda: P.mpcgemm_ex(dA, dB, C, c["prec"], method, device_rule=1))
        g = graph_of(lambda: P.mpcgemm_ex(dA, dB, C, c["prec"], method, device_rule=1))
        gr = timed(g.replay)
        rep = P.mpcgemm_ex(dA, dB, C, c["prec"], method, timing=1)
        out[f"cfg{cfg}_{method}"] = {"ms_host_rule": round(host, 4), "ms_device_rule": round(dev, 4),
                                     "ms_device_rule_graph": round(gr, 4), "ms_slicegemm": round(rep["ms_gemm"], 4),
                                     "slices": rep["slices"]}
        print(json.dumps({f"cfg{cfg}_{method}": out[f"cfg{cfg}_{method}"]}), flush=True)
    # config 5: the 15 Schur-update GEMMs of one LU, as one sequence
    mats = [(P.to_device(L21), P.to_device(U12), L21.shape[0], U12.shape[1]) for _, L21, U12 in mpgen.lu_update_gemms(seed=0)]
    Cs = [P.empty_device(mm, nn, 768) for _, _, mm, nn in mats]

    def seq(device_rule):
        for (a, b, _, _), c in zip(mats, Cs):
            P.mpcgemm_ex(a, b, c, 768, method, device_rule=device_rule)
    host = timed(lambda: seq(0), reps=5)
    dev = timed(lambda: seq(1), reps=5)
    g = graph_of(lambda: seq(1))
    gr = timed(g.replay, reps=5)
    out[f"cfg5_{method}"] = {"ms_host_rule": round(host, 3), "ms_device_rule": round(dev, 3),
                             "ms_device_rule_graph": round(gr, 3), "calls": len(mats)}
    print(json.dumps({f"cfg5_{method}": out[f"cfg5_{method}"]}), flush=True)
print(json.dumps(out))
