"""The multi-GPU driver (paper_2307_06072_b200/dist.py) through NCCL on the one GPU this
environment has: a world-size-1 NCCL process group runs the real collectives (all-reduce of the
pre-pass integers, all-gather of C row blocks) around the C ABI; the result equals the plain
single call bitwise.  (World size > 1 needs one GPU per rank; the protocol itself is covered with
gloo, world size 2, in test_dist_gloo.py.)"""
import os
import socket

import numpy as np
import pytest

import mpgen
from harness import same_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

import paper_2307_06072_b200 as P  # noqa: E402
from paper_2307_06072_b200 import dist as pdist  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_dist_gemm_nccl_world1(method):
    prec = 192
    A = mpgen.random_cmat(12, 1, 300, 80, prec, 5, zero_frac=0.1)
    B = mpgen.random_cmat(12, 2, 80, 140, prec, 5, zero_frac=0.1)
    dA, dB = P.to_device(A), P.to_device(B)
    C0, r0 = P.gemm(dA, dB, prec, method)
    torch.cuda.synchronize()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        C1, rep, full = pdist.gemm(dA, dB, A.shape[0], prec, method, gather=True)
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()
    assert rep["slices"] == r0["slices"]
    H0, H1 = P.to_host(C0), P.to_host(C1)
    assert same_bits(H0, H1)
    for p in ("re", "im"):
        R = getattr(H0, p)
        assert np.array_equal(full[p]["sign"].cpu().numpy(), R.sign)
        assert np.array_equal(full[p]["exp"].cpu().numpy(), R.exp)
        assert np.array_equal(full[p]["limbs"].cpu().numpy().view(np.uint64), R.limbs)


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_strong_gemm_nccl_world1(method):
    """dist.StrongGemm -- the bench's strong-scaling path: packed B broadcast from rank 0, the
    pre-pass all-reduce, the C ABI on this rank's rows, C all-gather, pipelined over a
    communication stream with double buffers -- through real NCCL collectives (world size 1),
    4 products: the gathered C equals the plain single call bitwise."""
    prec = 256
    m, n, k = 300, 270, 160
    A = mpgen.random_cmat(13, 1, m, k, prec, 4, zero_frac=0.05)
    B = mpgen.random_cmat(13, 2, k, n, prec, 4, zero_frac=0.05)
    dA, dB = P.to_device(A), P.to_device(B)
    C0, r0 = P.gemm(dA, dB, prec, method)
    torch.cuda.synchronize()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        Bsrc = pdist.packed_cmat(k, n, prec, "cuda")
        pdist.copy_cmat(Bsrc[0], dB)
        SG = pdist.StrongGemm(m, n, k, prec, method, "cuda",
                              lambda Al, Bd, full: P.mpcgemm_rho_bounds(Al, Bd, prec, full),
                              P.mpcgemm_slices_for,
                              lambda Al, Bd, Cv, s_: P.mpcgemm_ex(Al, Bd, Cv, prec, method, slices=s_))
        reps = SG.run(dA, Bsrc, 4)
        parts = SG.finish()
        full = SG.full_c(3)
    finally:
        dist.destroy_process_group()
    assert all(r["slices"] == r0["slices"] for r in reps)
    assert parts["compute_ms"] > 0
    H0 = P.to_host(C0)
    for p in ("re", "im"):
        R = getattr(H0, p)
        assert np.array_equal(full[p]["sign"].cpu().numpy(), R.sign)
        assert np.array_equal(full[p]["exp"].cpu().numpy(), R.exp)
        assert np.array_equal(full[p]["limbs"].cpu().numpy().view(np.uint64), R.limbs)
