"""Benchmark: complex MP GEMM MACs/s of the Ozaki scheme on B200 (BASELINE.json metric).

A step is one whole hot path (exponent scan, rho-hat pre-pass
and slice rule, split, tcgen05 slice GEMMs, fold + normalize) over one batch of synthetic
input: BASELINE config 4, complex 2048^3 at prec 1024 (the configuration the metric is
quoted on at 1/2/4/8 GPUs), method 3M by default.  Multi-GPU (torchrun): STRONG scaling of the
same 2048^3 product -- rank r owns rows row_range(2048, r, N) of A (pre-sharded), B lives on
rank 0 and is broadcast by NCCL inside every step, s is agreed by an all-reduce of the pre-pass
integers, and the C row blocks are all-gathered by NCCL inside every step
(paper_2307_06072_b200/dist.py StrongGemm: broadcast / gather of neighbouring steps pipelined on
a communication stream).  A weak-scaling run (2048 rows per rank) is an extra key.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--method 3M|4M] [--impl ours|reference]

Prints ONE JSON line (rank 0).  value = the product's CMACs (m n k) / max-over-ranks device
time per step of the K timed steps (CUDA events on the launching stream, barrier + synchronize on
both sides).  Inputs are larger than L2 (2.3 GB per rank), so no flush is needed.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import mpgen  # noqa: E402

METRIC = "complex MP GEMM MACs/s at prec bits (1/2/4/8 B200); slice-GEMM % tensor peak"
UNIT = "CMAC/s"


def peaks():
    try:
        P = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return P, "MEASURED_PEAKS.json"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_oracle_sample(A, B, prec, method, s, target_s=15.0, start=4):
    """The oracle (Algorithm 2, oracle/mpref.c) as it stands, all host cores, on a bounded
    sample of output elements of the same workload; returns (CMAC/s, cores, description)."""
    import oracle
    cores = os.cpu_count() or 1
    m, k = A.shape
    n = B.shape[1]
    rng = np.random.default_rng(1234)
    cnt, done, t_all, last = start, 0, 0.0, None
    while True:
        si = rng.integers(0, m, cnt)
        sj = rng.integers(0, n, cnt)
        t0 = time.perf_counter()
        oracle.ozaki(A, B, prec, method, s, samples=(si, sj), nthreads=cores)
        dt = time.perf_counter() - t0
        done += cnt; t_all += dt; last = dt
        if t_all >= target_s or cnt > 100000:
            break
        cnt = max(cnt, int(cnt * min(8.0, max(1.5, (target_s - t_all) / max(dt, 1e-3)))))
        if t_all + last * (cnt / max(done, 1)) > 3 * target_s:
            cnt = max(1, int(done * (target_s - t_all) / max(t_all, 1e-3)))
            if cnt <= 0:
                break
    return done * k / t_all, cores, f"{done} sampled output elements (x k={k} CMACs each) in {t_all:.1f} s"


def run_reference(args):
    """--impl reference: the CPU oracle as it stands on the box's host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    c = mpgen.CONFIGS[args.config]
    A, B = mpgen.config_inputs(args.config, seed=args.seed)
    import oracle
    s, _ = oracle.auto_slices(A, B, c["prec"], args.method)           # the full slice rule
    if args.slices:
        s = args.slices
    cores = os.cpu_count() or 1
    per_step = max(cores, 8)
    rng = np.random.default_rng(99)
    times = []
    for it in range(args.warmup + args.steps):
        si, sj = rng.integers(0, c["m"], per_step), rng.integers(0, c["n"], per_step)
        t0 = time.perf_counter()
        oracle.ozaki(A, B, c["prec"], args.method, s, samples=(si, sj), nthreads=cores)
        if it >= args.warmup:
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = args.steps * per_step * c["k"] / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8/i32/u64",
            "data": "synthetic", "config": workload_config(args, s),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{per_step} sampled output elements per step (x k={c['k']} CMACs), Algorithm-2 oracle"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def hbm_kernels(args, reps, m, n, k, prec, s, pk, src):
    """Achieved HBM bandwidth of the bandwidth-bound steps from their live stage times (CUDA
    events on the launching stream) and ALGORITHMIC bytes:
      split (a-3, A and B): read 2 (m k + k n)(9 + 8 L), write parts s (m + n) kp
      fold + normalize (a-5/a-6): read 4 nslots per output element, write 2 (9 + 8 L) per element"""
    L = (prec + 63) // 64
    parts = 3 if args.method == "3M" else 2
    kp = (k + 15) // 16 * 16
    ent = 9 + 8 * L
    split_b = 2 * (m * k + k * n) * ent + parts * s * (m + n) * kp
    nslots = reps[-1].get("partial_slots", 0)
    fold_b = m * n * (4 * nslots + 2 * ent)
    peak = pk["hbm_gbs"]
    out = []
    for name, b, f in (("split_kernel x2 (a-3)", split_b, "ms_split"), ("fold_normalize_kernel (a-5/a-6)", fold_b, "ms_fold")):
        ms = statistics.mean(r[f] for r in reps)
        gbs = b / (ms / 1e3) / 1e9
        out.append({"kernel": name, "bytes": b, "ms": round(ms, 3), "achieved": round(gbs, 1), "peak": peak,
                    "unit": "GB/s", "frac": round(gbs / peak, 3), "peak_source": f"{src}: hbm_gbs"})
    return out


def workload_config(args, s, world=1):
    c = mpgen.CONFIGS[args.config]
    rows = [r1 - r0 for r0, r1 in (row_range_(c["m"], r, world) for r in range(world))]
    return {"workload": f"BASELINE config {args.config}: " + c["desc"], "method": args.method, "m": c["m"],
            "n": c["n"], "k": c["k"], "prec": c["prec"], "slices": s, "seed": args.seed,
            "l2": "inputs larger than L2 (no flush needed)",
            "parallelism": (f"rows x{world} (strong: A pre-sharded, rows per rank {min(rows)}-{max(rows)}; B broadcast and "
                            "C all-gathered by NCCL inside every step, pipelined on a communication stream)")
            if world > 1 else "1 GPU"}


def row_range_(m, rank, world):
    base, rem = divmod(m, world)
    r0 = rank * base + min(rank, rem)
    return r0, r0 + base + (1 if rank < rem else 0)


def inrun_ceilings():
    """INT8 tensor ceilings measured in this run (after the timed region): back-to-back tcgen05.mma
    kind::i8 on rotating random SMEM operands, 148 SMs (tools/mma_power, built by build()), and
    cuBLASLt INT8 (torch._int_mm 8192^3, best of 10)."""
    import torch
    out = {}
    exe = os.path.join(ROOT, "tools", "mma_power")
    if os.path.exists(exe):
        try:
            r = subprocess.run([exe, "10000000"], capture_output=True, text=True, timeout=120)
            d = json.loads(r.stdout.strip().splitlines()[-1])
            out["tcgen05_mma_random_operands"] = {"tops": d["int8_tops"], "sm_ghz": d["avg_sm_ghz"],
                                                  "seconds": d["seconds"]}
        except Exception as e:  # noqa: BLE001
            out["tcgen05_mma_random_operands"] = {"error": str(e)[:200]}
    try:
        N = 8192
        a = torch.randint(-128, 127, (N, N), dtype=torch.int8, device="cuda")
        b = torch.randint(-128, 127, (N, N), dtype=torch.int8, device="cuda").t().contiguous().t()
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); torch._int_mm(a, b); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        out["cublaslt_int8_burst"] = {"tops": round(2.0 * N ** 3 / best / 1e12, 1)}
        del a, b
    except Exception as e:  # noqa: BLE001
        out["cublaslt_int8_burst"] = {"error": str(e)[:200]}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--method", default="3M", choices=["3M", "4M"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the 4M sub-record, in-run ceilings, weak run")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--seed", type=int, default=0, help="input generator seed (BASELINE configs: 0)")
    ap.add_argument("--slices", type=int, default=0,
                    help="force the slice count s (0: the certified auto rule -- the BASELINE workload)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2307_06072_b200 as P
    from paper_2307_06072_b200 import dist as pdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # NCCL's kernels (96 registers x its threads) cannot become resident next to a slice-GEMM CTA,
        # so the pipelined B broadcast / C all-gather overlap the GEMM only on SMs the GEMM leaves
        # free: 8 channels on 8 reserved SMs (unmeasured on > 1 GPU here; both are overridable)
        os.environ.setdefault("NCCL_MAX_NCHANNELS", "8")
        os.environ.setdefault("MPCGEMM_RESERVE_SMS", "8")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    c = mpgen.CONFIGS[args.config]
    m, n, k, prec = c["m"], c["n"], c["k"], c["prec"]
    stream = torch.cuda.current_stream(dev)
    extra = {}
    clocks = ClockSampler(local)

    if world == 1:
        A, B = mpgen.config_inputs(args.config, seed=args.seed)
        dA, dB = P.to_device(A, dev), P.to_device(B, dev)
        dC = P.empty_device(m, n, prec, dev)

        def step(timing=0, method=args.method):
            return P.mpcgemm_ex(dA, dB, dC, prec, method, slices=args.slices, stream=stream, timing=timing)

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        clocks.start()
        time.sleep(0.3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = []
        e0.record(stream)
        for _ in range(args.steps):
            reps.append(step(timing=1))
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        clk = clocks.stop()
        s = reps[-1]["slices"]
        launches = int(sum(r["kernel_launches"] for r in reps))
    else:
        # strong scaling: rank r owns rows row_range(m, r, N) of the one global A (pre-sharded, from
        # the same seeded generator); B lives on rank 0 and is broadcast inside every step
        r0, r1 = pdist.row_range(m, rank, world)
        A, B = mpgen.config_inputs(args.config, seed=args.seed, row0=r0, rows=r1 - r0)
        dA = P.to_device(A, dev)
        Bsrc = None
        if rank == 0:
            Bsrc = pdist.packed_cmat(k, n, prec, dev)
            pdist.copy_cmat(Bsrc[0], P.to_device(B, dev))

        def compute(Al, Bd, Cv, s_, timing=[1]):
            return P.mpcgemm_ex(Al, Bd, Cv, prec, args.method, slices=s_, timing=timing[0])

        SG = pdist.StrongGemm(m, n, k, prec, args.method, dev,
                              lambda Al, Bd, full: P.mpcgemm_rho_bounds(Al, Bd, prec, full),
                              P.mpcgemm_slices_for, compute)
        SG.run(dA, Bsrc, args.warmup)
        SG.finish()
        clocks.start()
        time.sleep(0.3)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        reps = SG.run(dA, Bsrc, args.steps)
        # the last step's gather is inside the timed region: the compute stream waits for it
        stream.wait_stream(SG.comm)
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        ms_local = e0.elapsed_time(e1) / args.steps
        clk = clocks.stop()
        parts = SG.finish()
        t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        s = reps[-1]["slices"]
        launches = int(sum(r["kernel_launches"] for r in reps))
        extra["strong"] = {"compute_ms_per_step": round(parts["compute_ms"] / args.steps, 3),
                           "bcast_ms_per_step": round(parts["bcast_ms"] / args.steps, 3),
                           "gather_ms_per_step": round(parts["gather_ms"] / args.steps, 3),
                           "rows_this_rank0": r1 - r0,
                           "reserved_sms": int(os.environ.get("MPCGEMM_RESERVE_SMS", "0")),
                           "nccl_max_nchannels": os.environ.get("NCCL_MAX_NCHANNELS"),
                           "note": "per-stream device times (CUDA events); B broadcast / C all-gather of "
                                   "neighbouring steps overlap compute, so they do not add up to ms_per_step"}
    cmacs = m * n * k                                   # the whole product, all ranks together
    value = cmacs / (ms / 1e3)

    # roofline of the dominant kernel (the tcgen05 slice GEMM), timed live with CUDA events
    # on the launching stream inside the library (opts.timing) over the timed steps
    R = 3 if args.method == "3M" else 4
    pairs = s * (s + 1) // 2
    pk, src = peaks()
    peak_int8 = 2.0 * pk["bf16_tflops_sustained"]       # measured bf16 sustained x nominal int8/bf16 = 2
    stage_ms = {}
    roof = None
    if world == 1 or all("ms_gemm" in r for r in reps):
        ops = 2.0 * R * pairs * A.shape[0] * n * k      # algorithmic INT8 ops per launch (this rank's rows)
        gemm_ms = statistics.mean(r["ms_gemm"] for r in reps) if reps[-1].get("ms_gemm", 0) > 0 else None
        if gemm_ms:
            achieved = ops / (gemm_ms / 1e3) / 1e12
            stage_ms = {f: round(statistics.mean(r[f] for r in reps), 3) for f in
                        ("ms_linemax", "ms_prepass", "ms_split", "ms_gemm", "ms_fold")}
            traffic = None
            try:
                tr = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
                if tr["config"] == args.config and tr["method"] == args.method and tr["slices"] == s and world == 1:
                    traffic = tr["dram_bytes_read"] + tr["dram_bytes_write"]
            except Exception:
                traffic = None
            roof = {"bound": "tensor", "achieved": round(achieved, 1), "peak": round(peak_int8, 1), "unit": "TOP/s",
                    "frac": round(achieved / peak_int8, 4), "frac_vs_nominal_4500": round(achieved / 4500.0, 4),
                    "traffic": traffic,
                    "traffic_note": "ncu dram__bytes_read+write per launch (profiles/roofline_traffic.json); "
                                    "the kernel is tensor-bound, its algorithmic operand bytes are the digit planes",
                    "kernel": "slicegemm_tc2_kernel (tcgen05.mma.cta_group::2 kind::i8)",
                    "peak_source": f"{src}: 2 x bf16_tflops_sustained (nominal int8/bf16 = 2)",
                    "algorithmic": f"2 R P m n k = 2*{R}*{pairs}*{A.shape[0]}*{n}*{k} int8 ops per launch",
                    "mma_instructions_per_launch": reps[-1].get("mma_issued")}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8/i32/u64",
        "data": "synthetic", "config": workload_config(args, s, world),
        "roofline": roof,
        "stages_ms": stage_ms,
        "gpu_launches": launches,
        "clocks": clk,
    }
    if world == 1 and stage_ms:
        line["hbm_kernels"] = hbm_kernels(args, reps, m, n, k, prec, s, pk, src)
    line.update(extra)
    if world == 1 and not args.no_extra:
        # the other method on the same workload (3M is 24-26 % faster than 4M)
        other = "4M" if args.method == "3M" else "3M"
        for _ in range(2):
            step(method=other)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r2 = []
        e0.record(stream)
        for _ in range(max(2, min(args.steps, 4))):
            r2.append(step(timing=1, method=other))
        e1.record(stream)
        torch.cuda.synchronize()
        ms2 = e0.elapsed_time(e1) / len(r2)
        line[f"method_{other}"] = {"value": cmacs / (ms2 / 1e3), "unit": UNIT, "ms_per_step": ms2,
                                   "ms_gemm": round(statistics.mean(r["ms_gemm"] for r in r2), 3),
                                   "steps": len(r2), "slices": r2[-1]["slices"],
                                   "time_ratio_3M_over_4M": round((ms if args.method == "3M" else ms2) /
                                                                  (ms2 if args.method == "3M" else ms), 4)}
        if roof:
            ceil = inrun_ceilings()
            roof["ceilings_in_run"] = ceil
            mm = ceil.get("tcgen05_mma_random_operands", {}).get("tops")
            if mm:
                roof["frac_vs_in_run_mma_ceiling"] = round(roof["achieved"] / mm, 4)
    if world > 1 and not args.no_extra:
        # weak scaling (extra key): every rank its own 2048-row block of a (N x 2048)-row A, B local
        Aw, Bw = mpgen.config_inputs(args.config, seed=args.seed, row0=rank * m, rows=m)
        dAw, dBw = P.to_device(Aw, dev), P.to_device(Bw, dev)
        dCw = P.empty_device(m, n, prec, dev)

        def wstep():
            s_, _ = pdist.common_slices(lambda full: P.mpcgemm_rho_bounds(dAw, dBw, prec, full, stream=stream),
                                        P.mpcgemm_slices_for, prec, args.method, k, device=dev)
            return P.mpcgemm_ex(dAw, dBw, dCw, prec, args.method, slices=s_, stream=stream)
        wstep()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            wstep()
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        line["weak"] = {"value": world * m * n * k / (float(t.item()) / 1e3), "unit": UNIT,
                        "ms_per_step": float(t.item()), "rows_per_rank": m, "scaling": "weak"}
        del dAw, dBw, dCw
    if not args.no_e2e:
        e2e = e2e_measure(P, A, B, prec, args, world, dev,
                          strong=(SG, dA, Bsrc) if world > 1 else None)   # every rank; max over ranks
        if rank == 0:
            line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu:
        v, cores, desc = cpu_oracle_sample(A, B, prec, args.method, s, target_s=args.cpu_seconds)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e_measure(P, A, B, prec, args, world=1, dev=None, strong=None):
    """Same metric through the public API on HOST buffers (pinned), every step's H2D of its inputs
    and D2H of its result inside the timed region.
      N = 1: the C ABI's queued host entry (mpcgemm_host_async x K + mpcgemm_host_wait; step i+1's
             H2D overlaps step i's compute), plus one blocking mpcgemm_host call;
      N > 1: per step, H2D of this rank's A rows (and of B on rank 0), the strong-scaling product
             (B broadcast, common s, this rank's rows, C all-gather) and the D2H of the gathered C
             on rank 0; wall clock, max over ranks."""
    import torch
    import torch.distributed as dist

    def pinned(R):
        out = []
        for a in (R.sign, R.exp, R.limbs):
            t = torch.empty(a.shape, dtype={np.uint8: torch.uint8, np.int64: torch.int64, np.uint64: torch.int64}[a.dtype.type],
                            pin_memory=True)
            v = t.numpy().view(a.dtype)
            v[...] = a
            out.append(v)
        return mpgen.RMat(out[0], out[1], out[2], R.prec)

    ent = lambda R: R.sign.nbytes + R.exp.nbytes + R.limbs.nbytes
    m, k = A.shape
    n = B.shape[1]
    if world > 1:
        SG, dA, Bsrc = strong
        rank = dist.get_rank()
        hA = mpgen.CMat(pinned(A.re), pinned(A.im))
        hB = mpgen.CMat(pinned(B.re), pinned(B.im)) if rank == 0 else None
        mfull = SG.m
        L = (prec + 63) // 64
        hC = torch.empty(SG.Cfull[0].numel(), dtype=torch.uint8, pin_memory=True) if rank == 0 else None

        def h2d(dX, hX):
            for p_ in ("re", "im"):
                dR, hR = getattr(dX, p_), getattr(hX, p_)
                dR.sign.copy_(torch.from_numpy(hR.sign), non_blocking=True)
                dR.exp.copy_(torch.from_numpy(hR.exp), non_blocking=True)
                dR.limbs.copy_(torch.from_numpy(hR.limbs.view(np.int64)), non_blocking=True)

        def run():
            h2d(dA, hA)
            if rank == 0:
                h2d(Bsrc[0], hB)
            SG.run(dA, Bsrc, 1)
            if rank == 0:
                torch.cuda.current_stream().wait_stream(SG.comm)
                hC.copy_(SG.Cfull[0], non_blocking=True)
            torch.cuda.synchronize()
        run()
        ts = []
        for _ in range(max(2, min(args.steps, 3))):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            run()
            ts.append(time.perf_counter() - t0)
        SG.finish()
        tt = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
        return {"value": mfull * n * k / t, "unit": UNIT,
                "h2d_bytes_per_step": (ent(A.re) + ent(A.im)) * world + ent(B.re) + ent(B.im),
                "d2h_bytes_per_step": 2 * mfull * n * (9 + 8 * L), "ms_per_step": 1e3 * t,
                "api": "pinned host copies of each rank's A rows and rank 0's B + dist.StrongGemm (NCCL broadcast "
                       "of B, pre-pass all-reduce, mpcgemm_ex, NCCL all-gather of C) + D2H of the gathered C on rank 0"}

    hA = mpgen.CMat(pinned(A.re), pinned(A.im))
    hB = mpgen.CMat(pinned(B.re), pinned(B.im))
    hC = mpgen.CMat(pinned(mpgen.empty_rmat(m, n, prec)), pinned(mpgen.empty_rmat(m, n, prec)))
    P.mpcgemm_host(hA, hB, prec, args.method, C=hC, slices=args.slices)               # warm-up (staging allocation)
    ts = []
    for _ in range(max(2, min(args.steps, 3))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.mpcgemm_host(hA, hB, prec, args.method, C=hC, slices=args.slices)
        ts.append(time.perf_counter() - t0)
    t_block = statistics.median(ts)
    # a stream of K products through the queued entry: step i+1's H2D overlaps step i's slice
    # GEMM and step i's D2H the next step's compute; every step still copies its inputs in and
    # its C out inside the timed region (wall clock from the first call to the wait)
    hC2 = mpgen.CMat(pinned(mpgen.empty_rmat(m, n, prec)), pinned(mpgen.empty_rmat(m, n, prec)))
    outs = (hC, hC2)
    K = max(3, args.steps)
    for i in range(2):                                           # warm-up: both staging sets
        P.mpcgemm_host_async(hA, hB, prec, args.method, C=outs[i], slices=args.slices)
    P.mpcgemm_host_wait()
    t0 = time.perf_counter()
    for i in range(K):
        P.mpcgemm_host_async(hA, hB, prec, args.method, C=outs[i & 1], slices=args.slices)
    P.mpcgemm_host_wait()
    t = (time.perf_counter() - t0) / K
    return {"value": m * n * k / t, "unit": UNIT, "h2d_bytes_per_step": ent(A.re) + ent(A.im) + ent(B.re) + ent(B.im),
            "d2h_bytes_per_step": 2 * (m * n * (9 + 8 * ((prec + 63) // 64))), "ms_per_step": 1e3 * t,
            "api": (f"mpcgemm_host_async x {K} steps + mpcgemm_host_wait (C ABI, pinned host buffers; "
                    "step i+1's H2D overlaps step i's compute)"),
            "blocking_ms_per_step": 1e3 * t_block,
            "blocking_api": "mpcgemm_host (one blocking call: H2D, compute, D2H)"}


if __name__ == "__main__":
    main()
