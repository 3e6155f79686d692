"""Multi-GPU driver: one process per GPU, torch.distributed (NCCL on GPUs,
gloo on CPU for the host-logic tests).

Output row blocks of C are independent (eA_i is row-local), so A is row-partitioned and B is
replicated on every rank.  The only data-dependent exchange is the slice count: every rank
runs the rho-hat pre-pass on its rows and the ranks all-reduce its integers (MIN of minT;
if that is 0, a second round of MIN minT1 / MAX maxD2), so all ranks use the same s and C is
bitwise identical for any number of GPUs.  A can be row-scattered from one rank
(scatter_rows), B broadcast from one rank (broadcast_fields), and C row blocks all-gathered
(gather_rows).
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
