"""Multi-rank host logic of the driver (paper_2307_06072_b200/dist.py) on CPU with gloo,
world size 2: row partition, the two-round all-reduce of the pre-pass integers (common s),
and the all-gather of C row blocks.  The per-rank compute is a stand-in (the oracle: tests
may call it); on GPUs the same protocol runs with the C ABI over NCCL."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import mpgen
import oracle
from paper_2307_06072_b200.dist import broadcast_fields, gather_rows, orchestrate, row_range, scatter_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _to_t(R):
    return {"sign": torch.from_numpy(R.sign.copy()), "exp": torch.from_numpy(R.exp.copy()),
            "limbs": torch.from_numpy(R.limbs.view(np.int64).copy())}


def _from_t(fields, prec):
    return mpgen.RMat(fields["sign"].numpy().copy(), fields["exp"].numpy().copy(),
                      fields["limbs"].numpy().view(np.uint64).copy(), prec)


def _distribute(A, B, m, n, k, prec, rank):
    """Rank 0 alone holds A and B: A's rows are scattered, B broadcast (torch tensors)."""
    L = (prec + 63) // 64
    Al, Bl = {}, {}
    for p in ("re", "im"):
        src_a = _to_t(getattr(A, p)) if rank == 0 else None
        Al[p] = {f: scatter_rows(src_a[f] if src_a else None, m, rest, dt, "cpu")
                 for f, rest, dt in (("sign", (k,), torch.uint8), ("exp", (k,), torch.int64),
                                     ("limbs", (k, L), torch.int64))}
        fb = _to_t(getattr(B, p)) if rank == 0 else {"sign": torch.zeros((k, n), dtype=torch.uint8),
                                                    "exp": torch.zeros((k, n), dtype=torch.int64),
                                                    "limbs": torch.zeros((k, n, L), dtype=torch.int64)}
        Bl[p] = broadcast_fields(fb)
    return (mpgen.CMat(_from_t(Al["re"], prec), _from_t(Al["im"], prec)),
            mpgen.CMat(_from_t(Bl["re"], prec), _from_t(Bl["im"], prec)))


def _worker(rank, world, port, case, outdir, distribute=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, n, k, prec, spread, method = case
    A = mpgen.random_cmat(77, 1, m, k, prec, spread, zero_frac=0.1)
    B = mpgen.random_cmat(77, 2, k, n, prec, spread, zero_frac=0.1)
    r0, r1 = row_range(m, rank, world)
    if distribute:                                     # only rank 0's copies are used
        if rank:
            A = B = None
        Al, B = _distribute(A, B, m, n, k, prec, rank)
    else:
        Al = A.rows(r0, r1)
    s, bounds, C = orchestrate(lambda full: oracle.rho_bounds(Al, B, full=full),
                               lambda *a: oracle.slices_for(*a)[0],
                               lambda s_: oracle.ozaki(Al, B, prec, method, s_),
                               prec, method, k)
    full = {p: {f: gather_rows(t, m, "cpu") for f, t in _to_t(getattr(C, p)).items()} for p in ("re", "im")}
    if rank == 0:
        np.savez(os.path.join(outdir, "out.npz"), s=s, b0=bounds[0], b1=bounds[1], b2=bounds[2],
                 **{f"{p}_{f}": full[p][f].numpy() for p in ("re", "im") for f in ("sign", "exp", "limbs")})
    dist.destroy_process_group()


def test_row_range_partition():
    for m in (0, 1, 7, 8, 2048, 2049):
        for w in (1, 2, 3, 8):
            rr = [row_range(m, r, w) for r in range(w)]
            assert rr[0][0] == 0 and rr[-1][1] == m
            assert all(rr[i][1] == rr[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in rr) - min(b - a for a, b in rr) <= 1


@pytest.mark.parametrize("distribute", [False, True])
@pytest.mark.parametrize("case", [(7, 9, 11, 128, 4, "3M"),      # ragged rows
                                  (9, 6, 12, 256, 16, "4M"),     # minT == 0: second round
                                  (1, 5, 8, 128, 0, "3M")])      # one rank without rows
def test_two_ranks_gloo(case, distribute):
    """distribute: A row-scattered and B broadcast from rank 0 instead of every
    rank generating its own copies."""
    m, n, k, prec, spread, method = case
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), case, d, distribute), nprocs=2, join=True)
        z = np.load(os.path.join(d, "out.npz"))
        A = mpgen.random_cmat(77, 1, m, k, prec, spread, zero_frac=0.1)
        B = mpgen.random_cmat(77, 2, k, n, prec, spread, zero_frac=0.1)
        s_ref, _ = oracle.auto_slices(A, B, prec, method)
        assert int(z["s"]) == s_ref                    # same s as one process on all rows
        R = oracle.ozaki(A, B, prec, method, s_ref)
        for p in ("re", "im"):
            Rp = getattr(R, p)
            assert np.array_equal(z[f"{p}_sign"], Rp.sign)
            assert np.array_equal(z[f"{p}_exp"], Rp.exp)
            assert np.array_equal(z[f"{p}_limbs"].view(np.uint64), Rp.limbs)


# ------------------------------------------------------------------ strong scaling (dist.StrongGemm)
def _strong_worker(rank, world, port, case, outdir, steps):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2307_06072_b200 as P
    from paper_2307_06072_b200.dist import StrongGemm, copy_cmat, packed_cmat
    m, n, k, prec, spread, method = case
    r0, r1 = row_range(m, rank, world)
    A = mpgen.random_cmat(78, 1, m, k, prec, spread, zero_frac=0.1).rows(r0, r1)    # pre-sharded rows
    Bsrc = None
    if rank == 0:                                      # B lives on rank 0 only
        Bsrc = packed_cmat(k, n, prec, "cpu")
        copy_cmat(Bsrc[0], P.to_device(mpgen.random_cmat(78, 2, k, n, prec, spread, zero_frac=0.1), "cpu"))

    def compute(Al, Bd, Cv, s_):                       # the per-rank stand-in: the oracle
        C = oracle.ozaki(P.to_host(Al), P.to_host(Bd), prec, method, s_)
        for p in ("re", "im"):
            R, D = getattr(C, p), getattr(Cv, p)
            D.sign.copy_(torch.from_numpy(R.sign)); D.exp.copy_(torch.from_numpy(R.exp))
            D.limbs.copy_(torch.from_numpy(R.limbs.view(np.int64)))
        return {"slices": s_}

    SG = StrongGemm(m, n, k, prec, method, "cpu",
                    lambda Al, Bd, full: oracle.rho_bounds(P.to_host(Al), P.to_host(Bd), full=full),
                    lambda *a: oracle.slices_for(*a)[0], compute)
    reps = SG.run(P.to_device(A, "cpu"), Bsrc, steps)
    SG.finish()
    full = SG.full_c(steps - 1)
    if rank == 0:
        np.savez(os.path.join(outdir, "out.npz"), s=reps[-1]["slices"], nsteps=len(reps),
                 **{f"{p}_{f}": full[p][f].numpy() for p in ("re", "im") for f in ("sign", "exp", "limbs")})
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [(7, 9, 11, 128, 4, "3M"),      # ragged rows
                                  (9, 6, 12, 256, 16, "4M"),     # minT == 0: second all-reduce round
                                  (1, 5, 8, 128, 0, "3M")])      # one rank without rows
def test_strong_gemm_two_ranks(case):
    """dist.StrongGemm (the bench's N > 1 path) at world size 2 on gloo: A pre-sharded, B only on
    rank 0 and broadcast inside each of 3 pipelined products (double buffers reused), the pre-pass
    all-reduce, C row blocks all-gathered; the gathered C equals one process's oracle on all rows."""
    m, n, k, prec, spread, method = case
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_strong_worker, args=(2, _free_port(), case, d, 3), nprocs=2, join=True)
        z = np.load(os.path.join(d, "out.npz"))
        A = mpgen.random_cmat(78, 1, m, k, prec, spread, zero_frac=0.1)
        B = mpgen.random_cmat(78, 2, k, n, prec, spread, zero_frac=0.1)
        s_ref, _ = oracle.auto_slices(A, B, prec, method)
        assert int(z["s"]) == s_ref and int(z["nsteps"]) == 3
        R = oracle.ozaki(A, B, prec, method, s_ref)
        for p in ("re", "im"):
            Rp = getattr(R, p)
            assert np.array_equal(z[f"{p}_sign"], Rp.sign)
            assert np.array_equal(z[f"{p}_exp"], Rp.exp)
            assert np.array_equal(z[f"{p}_limbs"].view(np.uint64), Rp.limbs)
