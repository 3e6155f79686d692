"""e2e pipeline probe (config 4): host return times of queued mpcgemm_host_async calls, raw
pinned H2D / D2H bandwidth alone, and the device-only call time, to locate the e2e overhead.
usage: python tools/e2e_probe.py [--steps 6] [--config 4]   (MPCGEMM_HOST_GROUP sets the row groups)"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import mpgen  # noqa: E402
import paper_2307_06072_b200 as P  # noqa: E402


def pinned(R):
    out = []
    for a in (R.sign, R.exp, R.limbs):
        t = torch.empty(a.shape, dtype={np.uint8: torch.uint8, np.int64: torch.int64, np.uint64: torch.int64}[a.dtype.type],
                        pin_memory=True)
        v = t.numpy().view(a.dtype)
        v[...] = a
        out.append(v)
    return mpgen.RMat(out[0], out[1], out[2], R.prec)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--config", type=int, default=4)
    args = ap.parse_args()
    A, B = mpgen.config_inputs(args.config, seed=0)
    m, k = A.shape
    n = B.shape[1]
    prec = A.re.prec
    hA = mpgen.CMat(pinned(A.re), pinned(A.im))
    hB = mpgen.CMat(pinned(B.re), pinned(B.im))
    outs = [mpgen.CMat(pinned(mpgen.empty_rmat(m, n, prec)), pinned(mpgen.empty_rmat(m, n, prec))) for _ in range(2)]
    res = {}
    # raw copy bandwidth (pinned, one 1 GB buffer each way)
    h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        res[name + "_GBs"] = 3 * (1 << 30) / (time.perf_counter() - t0) / 1e9
    # device-only call
    dA, dB = P.to_device(A), P.to_device(B)
    dC = P.empty_device(m, n, prec)
    for _ in range(2):
        P.mpcgemm_ex(dA, dB, dC, prec, "3M")
    torch.cuda.synchronize()

    def device_loop(tag):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            P.mpcgemm_ex(dA, dB, dC, prec, "3M")
        torch.cuda.synchronize()
        res[tag] = (time.perf_counter() - t0) / 3 * 1e3

    device_loop("device_ms")
    # device-only call with 2.3 GB H2D + 1.15 GB D2H queued on a side stream at each call
    side = torch.cuda.Stream()
    h2 = torch.empty(2300 << 20, dtype=torch.uint8, pin_memory=True)
    d2 = torch.empty(2300 << 20, dtype=torch.uint8, device="cuda")
    h3 = torch.empty(1150 << 20, dtype=torch.uint8, pin_memory=True)
    d3 = torch.empty(1150 << 20, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        with torch.cuda.stream(side):
            d2.copy_(h2, non_blocking=True)
            h3.copy_(d3, non_blocking=True)
        P.mpcgemm_ex(dA, dB, dC, prec, "3M")
    torch.cuda.synchronize()
    res["device_with_copies_ms"] = (time.perf_counter() - t0) / 3 * 1e3
    del h2, d2, h3, d3
    # blocking host call
    P.mpcgemm_host(hA, hB, prec, "3M", C=outs[0])
    t0 = time.perf_counter()
    P.mpcgemm_host(hA, hB, prec, "3M", C=outs[0])
    res["blocking_ms"] = (time.perf_counter() - t0) * 1e3
    # queued calls
    for i in range(2):
        P.mpcgemm_host_async(hA, hB, prec, "3M", C=outs[i])
    P.mpcgemm_host_wait()
    t0 = time.perf_counter()
    rets = []
    evs = []
    for i in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()                                  # legacy stream: after call i-1's compute
        P.mpcgemm_host_async(hA, hB, prec, "3M", C=outs[i & 1])
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()                                  # after call i's fold
        evs.append((e0, e1))
        rets.append((time.perf_counter() - t0) * 1e3)
    P.mpcgemm_host_wait()
    tw = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    res["async_stream_ms"] = [round(a.elapsed_time(b), 1) for a, b in evs]
    res["async_gap_ms"] = [round(evs[i][1].elapsed_time(evs[i + 1][0]), 2) for i in range(len(evs) - 1)]
    res["async_returns_ms"] = [round(x, 1) for x in rets]
    res["async_total_ms"] = tw
    res["async_ms_per_step"] = tw / args.steps
    device_loop("device_ms_after_async")
    t0 = time.perf_counter()
    for i in range(args.steps):
        P.mpcgemm_host_async(hA, hB, prec, "3M", C=outs[i & 1])
    P.mpcgemm_host_wait()
    res["async_ms_per_step_2"] = (time.perf_counter() - t0) * 1e3 / args.steps
    device_loop("device_ms_after_async_2")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
