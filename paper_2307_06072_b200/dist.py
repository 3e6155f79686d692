"""Multi-GPU driver: one process per GPU, torch.distributed (NCCL on GPUs,
gloo on CPU for the host-logic tests).

Output row blocks of C are independent (eA_i is row-local), so A is row-partitioned and B is
replicated on every rank.  The only data-dependent exchange is the slice count: every rank
runs the rho-hat pre-pass on its rows and the ranks all-reduce its integers (MIN of minT;
if that is 0, a second round of MIN minT1 / MAX maxD2), so all ranks use the same s and C is
bitwise identical for any number of GPUs.  A can be row-scattered from one rank
(scatter_rows), B broadcast from one rank (broadcast_fields), and C row blocks all-gathered
(gather_rows).  StrongGemm runs BASELINE config 4's strong-scaling products (pre-sharded A, B
broadcast and C all-gathered inside every product, pipelined over a communication stream).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import mpcgemm as _m

_BIG = (1 << 62)


def row_range(m: int, rank: int, world: int):
    """Rows [r0, r1) of rank `rank` (ragged: the first m % world ranks get one more row)."""
    base, rem = divmod(m, world)
    r0 = rank * base + min(rank, rem)
    return r0, r0 + base + (1 if rank < rem else 0)


def _allreduce(vals, op, device, group):
    t = torch.tensor(vals, dtype=torch.int64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=op, group=group)
    return [int(v) for v in t.tolist()]


def common_slices(bounds_fn, slices_fn, prec: int, method, k: int, device="cpu", group=None):
    """Global slice count from the per-rank pre-pass.
    bounds_fn(full) -> (minT, minT1, maxD2) for this rank's rows (mpcgemm_rho_bounds);
    slices_fn(prec, method, k, minT, minT1, maxD2) -> s (mpcgemm_slices_for).
    Returns (s, (minT, minT1, maxD2)) -- identical on every rank."""
    b = bounds_fn(0)
    (g0,) = _allreduce([b[0] if b[0] >= 0 else _BIG], dist.ReduceOp.MIN, device, group)
    minT = -1 if g0 == _BIG else g0
    if minT == 0:
        b = bounds_fn(1)
        (g1,) = _allreduce([b[1] if b[1] >= 0 else _BIG], dist.ReduceOp.MIN, device, group)
        (g2,) = _allreduce([b[2]], dist.ReduceOp.MAX, device, group)
        minT1, maxD2 = (-1 if g1 == _BIG else g1), g2
    else:
        minT1, maxD2 = minT, -1
    return slices_fn(prec, method, k, minT, minT1, maxD2), (minT, minT1, maxD2)


def gather_rows(local: torch.Tensor, m: int, device, group=None) -> torch.Tensor:
    """All-gather row blocks (ragged, row_range layout) of a [rows, ...] tensor into [m, ...]."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local
    maxr = row_range(m, 0, world)[1]
    pad = torch.zeros((maxr,) + tuple(local.shape[1:]), dtype=local.dtype, device=device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([parts[r][: row_range(m, r, world)[1] - row_range(m, r, world)[0]] for r in range(world)], 0)


def broadcast_fields(fields: dict, src: int = 0, group=None) -> dict:
    """B broadcast: every tensor of `fields` (e.g. one part's sign / exp / limbs, allocated with
    the same shape on every rank) is overwritten in place by the source rank's copy."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        for t in fields.values():
            dist.broadcast(t, src=src, group=group)
    return fields


def scatter_rows(full, m: int, rest: tuple, dtype, device, src: int = 0, group=None) -> torch.Tensor:
    """Row shards: the source rank's [m, *rest] tensor `full` is cut into the row_range blocks and
    each rank receives its own block (other ranks pass full=None)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if world == 1:
        return full
    r0, r1 = row_range(m, rank, world)
    maxr = row_range(m, 0, world)[1]
    out = torch.empty((maxr,) + tuple(rest), dtype=dtype, device=device)
    chunks = None
    if rank == src:
        chunks = []
        for r in range(world):
            a, b = row_range(m, r, world)
            c = torch.zeros((maxr,) + tuple(rest), dtype=dtype, device=device)
            c[: b - a] = full[a:b]
            chunks.append(c)
    dist.scatter(out, chunks, src=src, group=group)
    return out[: r1 - r0]


def orchestrate(bounds_fn, slices_fn, local_fn, prec: int, method, k: int, device="cpu", group=None):
    """The per-rank protocol, independent of where the compute runs: agree on s through the
    pre-pass all-reduce, then compute this rank's rows with it.  Returns (s, bounds, local)."""
    s, bounds = common_slices(bounds_fn, slices_fn, prec, method, k, device=device, group=group)
    return s, bounds, local_fn(s)


def gemm(A_local: "_m.DevCMat", B: "_m.DevCMat", m: int, prec: int | None = None, method="3M",
         group=None, gather: bool = False, stream=None, timing: int = 0):
    """C rows of this rank := A_local B with the globally agreed s (NCCL all-reduce of the
    pre-pass integers); optionally all-gathers every C row block onto every rank (as torch
    tensors).  Returns (C_local DevCMat, report, C_full dict or None)."""
    prec = A_local.prec if prec is None else prec
    k = B.shape[0]
    dev = A_local.re.sign.device
    C = _m.empty_device(A_local.shape[0], B.shape[1], prec, device=dev)
    s, bounds, rep = orchestrate(lambda full: _m.mpcgemm_rho_bounds(A_local, B, prec, full, stream=stream),
                                 _m.mpcgemm_slices_for,
                                 lambda s_: _m.mpcgemm_ex(A_local, B, C, prec, method, slices=s_, stream=stream, timing=timing),
                                 prec, method, k, device=dev, group=group)
    rep["bounds"] = bounds
    full = None
    if gather:
        full = {p: {f: gather_rows(getattr(getattr(C, p), f), m, dev, group) for f in ("sign", "exp", "limbs")}
                for p in ("re", "im")}
    return C, rep, full


# ------------------------------------------------------------------ strong scaling (BASELINE config 4)
def packed_cmat(rows: int, cols: int, prec: int, device):
    """A DevCMat whose six arrays (re/im sign, exp, limbs) are views of ONE flat uint8 tensor, so one
    collective moves the whole matrix.  Returns (DevCMat, flat)."""
    L = (prec + 63) // 64
    ent = rows * cols
    al = lambda x: (x + 255) // 256 * 256
    sizes = [ent, 8 * ent, 8 * ent * L]
    offs, tot = [], 0
    for _ in range(2):
        o = []
        for sz in sizes:
            o.append(tot)
            tot = al(tot + sz)
        offs.append(o)
    flat = torch.zeros(max(tot, 256), dtype=torch.uint8, device=device)

    def part(o):
        sign = flat[o[0]:o[0] + ent].view(rows, cols)
        exp = flat[o[1]:o[1] + 8 * ent].view(torch.int64).view(rows, cols)
        limbs = flat[o[2]:o[2] + 8 * ent * L].view(torch.int64).view(rows, cols, L)
        return _m.DevRMat(sign, exp, limbs, cols)

    return _m.DevCMat(part(offs[0]), part(offs[1]), prec), flat


def copy_cmat(dst: "_m.DevCMat", src: "_m.DevCMat"):
    for p in ("re", "im"):
        for f in ("sign", "exp", "limbs"):
            getattr(getattr(dst, p), f).copy_(getattr(getattr(src, p), f))


class StrongGemm:
    """Strong-scaling products C = A B over the ranks of `group` (BASELINE config 4
    "row-sharded across 1/2/4/8 GPUs"):

      * A is PRE-SHARDED: rank r owns rows row_range(m, r, N) (generated or loaded there);
      * B lives on rank `src` (a packed_cmat) and is broadcast from it -- one NCCL broadcast of the
        packed buffer -- inside every product;
      * the ranks agree on s through the pre-pass all-reduce (common_slices), so C is bitwise the
        single-GPU result for any N;
      * each rank computes its rows (compute_fn), and the C row blocks are all-gathered -- one NCCL
        all_gather of the packed, row-padded blocks -- onto every rank.

    Products are pipelined over a communication stream (GPU): product i+1's B broadcast is issued
    before product i computes and product i's C all-gather right after it, each ordered by CUDA
    events, so they overlap the neighbouring products' compute (B and C double-buffered).  On CPU
    (gloo) the same calls run in order.

    bounds_fn(A_local, B, full) -> (minT, minT1, maxD2);  slices_fn(prec, method, k, minT, minT1,
    maxD2) -> s;  compute_fn(A_local, B, C_local, s) -> report dict."""

    def __init__(self, m, n, k, prec, method, device, bounds_fn, slices_fn, compute_fn, group=None, src=0):
        self.m, self.n, self.k, self.prec, self.method = m, n, k, prec, method
        self.device = torch.device(device)
        self.group, self.src = group, src
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.r0, self.r1 = row_range(m, self.rank, self.world)
        self.maxr = row_range(m, 0, self.world)[1]
        self.bounds_fn, self.slices_fn, self.compute_fn = bounds_fn, slices_fn, compute_fn
        # the pre-pass all-reduce on its own communicator: on the bulk one it would queue behind the
        # next product's B broadcast (one NCCL stream per communicator runs its collectives in order)
        self.small = (dist.new_group(ranks=list(range(self.world)))
                      if dist.is_initialized() and self.world > 1 and group is None else group)
        self.gpu = self.device.type == "cuda"
        self.B = [packed_cmat(k, n, prec, self.device) for _ in range(2)] if self.rank != src else None
        self.C = [packed_cmat(self.maxr, n, prec, self.device) for _ in range(2)]
        self.Cfull = [torch.empty(self.world * self.C[0][1].numel(), dtype=torch.uint8, device=self.device)
                      for _ in range(2)]
        self.comm = torch.cuda.Stream(self.device) if self.gpu else None
        self.b_done = [None, None]      # per buffer: its last broadcast finished (event)
        self.c_done = [None, None]      # per buffer: the product that wrote it finished
        self.g_done = [None, None]      # per buffer: its last gather finished
        self.timeline = []              # (kind, start event, end event)

    def _ev(self):
        return torch.cuda.Event(enable_timing=True)

    def _bcast(self, j, B_src):
        if self.world == 1 or self.rank == self.src:
            flat = B_src[1]
        else:
            flat = self.B[j][1]
        if self.world == 1:
            return
        if not self.gpu:
            dist.broadcast(flat, src=self.src, group=self.group)
            return
        with torch.cuda.stream(self.comm):
            if self.c_done[j] is not None and self.rank != self.src:
                self.comm.wait_event(self.c_done[j])              # product i-2 is done reading B[j]
            e0, e1 = self._ev(), self._ev()
            e0.record(self.comm)
            dist.broadcast(flat, src=self.src, group=self.group)
            e1.record(self.comm)
        self.b_done[j] = e1
        self.timeline.append(("bcast", e0, e1))

    def _gather(self, j):
        flat = self.C[j][1]
        if not self.gpu:
            if self.world > 1:
                dist.all_gather_into_tensor(self.Cfull[j], flat, group=self.group)
            else:
                self.Cfull[j].copy_(flat)
            return
        with torch.cuda.stream(self.comm):
            self.comm.wait_event(self.c_done[j])
            e0, e1 = self._ev(), self._ev()
            e0.record(self.comm)
            if self.world > 1:
                dist.all_gather_into_tensor(self.Cfull[j], flat, group=self.group)
            else:
                self.Cfull[j].copy_(flat)
            e1.record(self.comm)
        self.g_done[j] = e1
        self.timeline.append(("gather", e0, e1))

    def run(self, A_local: "_m.DevCMat", B_src, steps: int = 1):
        """`steps` products A B.  B_src: the source rank's packed B (packed_cmat(k, n, ...)), other
        ranks None.  Returns the reports; full_c(steps - 1) is the last product's gathered C."""
        reps = []
        self._bcast(0, B_src)
        rows = self.r1 - self.r0
        for i in range(steps):
            j = i & 1
            if i + 1 < steps:
                self._bcast(j ^ 1, B_src)                         # overlaps product i
            Bj = B_src[0] if (self.world == 1 or self.rank == self.src) else self.B[j][0]
            Cj = self.C[j][0]
            Cv = _m.DevCMat(*(_m.DevRMat(getattr(Cj, p).sign[:rows], getattr(Cj, p).exp[:rows],
                                         getattr(Cj, p).limbs[:rows], self.n) for p in ("re", "im")), self.prec)
            if self.gpu:
                cs = torch.cuda.current_stream(self.device)
                for e in (self.b_done[j], self.g_done[j]):        # B[j] arrived; product i-2's gather read C[j]
                    if e is not None:
                        cs.wait_event(e)
                t0 = self._ev()
                t0.record(cs)
            s, bounds = common_slices(lambda full: self.bounds_fn(A_local, Bj, full), self.slices_fn, self.prec,
                                      self.method, self.k, device=self.device, group=self.small)
            rep = self.compute_fn(A_local, Bj, Cv, s) if rows > 0 else {"slices": s}
            rep["bounds"] = bounds
            reps.append(rep)
            if self.gpu:
                t1 = self._ev()
                t1.record(cs)
                self.c_done[j] = t1
                self.timeline.append(("compute", t0, t1))
            self._gather(j)
        return reps

    def finish(self):
        """Waits for all outstanding work; returns {"compute_ms", "bcast_ms", "gather_ms"}: device
        time summed per kind (CUDA events on the stream each ran on; they overlap)."""
        out = {"compute_ms": 0.0, "bcast_ms": 0.0, "gather_ms": 0.0}
        if self.gpu:
            torch.cuda.synchronize(self.device)
            for kind, e0, e1 in self.timeline:
                out[kind + "_ms"] += e0.elapsed_time(e1)
        self.timeline.clear()
        return out

    def full_c(self, i_last: int):
        """The gathered C of product i_last: dict part -> field -> tensor [m, ...] (row blocks of all
        ranks in order)."""
        j = i_last & 1
        per = self.C[0][1].numel()
        out = {p: {f: [] for f in ("sign", "exp", "limbs")} for p in ("re", "im")}
        for r in range(self.world):
            a, b = row_range(self.m, r, self.world)
            view, _ = packed_cmat_view(self.Cfull[j][r * per:(r + 1) * per], self.maxr, self.n, self.prec)
            for p in ("re", "im"):
                for f in ("sign", "exp", "limbs"):
                    out[p][f].append(getattr(getattr(view, p), f)[: b - a])
        return {p: {f: torch.cat(v, 0) for f, v in d.items()} for p, d in out.items()}


def packed_cmat_view(flat, rows: int, cols: int, prec: int):
    """The DevCMat views of a packed buffer laid out by packed_cmat(rows, cols, prec)."""
    L = (prec + 63) // 64
    ent = rows * cols
    al = lambda x: (x + 255) // 256 * 256
    offs, tot = [], 0
    for _ in range(2):
        o = []
        for sz in (ent, 8 * ent, 8 * ent * L):
            o.append(tot)
            tot = al(tot + sz)
        offs.append(o)

    def part(o):
        return _m.DevRMat(flat[o[0]:o[0] + ent].view(rows, cols),
                          flat[o[1]:o[1] + 8 * ent].view(torch.int64).view(rows, cols),
                          flat[o[2]:o[2] + 8 * ent * L].view(torch.int64).view(rows, cols, L), cols)

    return _m.DevCMat(part(offs[0]), part(offs[1]), prec), flat
