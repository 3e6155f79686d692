"""GPU parity for NEXT-4 (opts.adaptive: a certified slice count per block of 256 rows,
PAPER.md:360): the CUDA path through the C ABI against oracle.ozaki_rows with the per-block
counts of oracle.block_slices, bit-exact on sampled outputs (all block edges and the ragged
tail included), and against the exact oracle within BASELINE's acceptance bound."""
import numpy as np
import pytest

import mpgen
import oracle
from harness import max_err_log2, same_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2307_06072_b200 as P  # noqa: E402

from test_gpu_parity import BOUND, sampled_equal  # noqa: E402


def mixed_rows(seed, k, prec, spreads, rows_per_block, zero_frac=0.0):
    """A stacked from blocks of rows with different exponent spreads (different rho-hat)."""
    blocks = [mpgen.random_cmat(seed, 60 + b, r, k, prec, sp, zero_frac if sp else 0.0)
              for b, (sp, r) in enumerate(zip(spreads, rows_per_block))]
    return mpgen._vstack(blocks)


def samples_for(m, n, count, seed):
    rng = np.random.default_rng(seed)
    si = list(rng.integers(0, m, count))
    sj = list(rng.integers(0, n, count))
    for i in sorted({0, 255, 256, 511, 512, m - 1} & set(range(m))):
        for j in (0, min(255, n - 1), min(256, n - 1), n - 1):
            si.append(i); sj.append(j)
    return np.array(si), np.array(sj)


@pytest.mark.parametrize("method", ["3M", "4M"])
@pytest.mark.parametrize("k,prec,spreads", [(100, 192, (0, 24, 6)), (3, 128, (16, 0, 16)), (257, 256, (2, 40, 0))])
def test_adaptive_blocks_bitexact(method, k, prec, spreads):
    rows = (256, 256, 88)                              # 3 blocks, ragged last
    A = mixed_rows(k + prec, k, prec, spreads, rows, zero_frac=0.2)
    B = mpgen.random_cmat(k + prec, 7, k, 300, prec, 2, zero_frac=0.05)
    m, n = A.shape[0], B.shape[1]
    sb, ok = oracle.block_slices(A, B, prec, method, block=256)
    assert ok
    dA, dB = P.to_device(A), P.to_device(B)
    dC, rep = P.gemm(dA, dB, prec, method, adaptive=1)
    torch.cuda.synchronize()
    C = P.to_host(dC)
    assert rep["block_slices"] == sb, (rep["block_slices"], sb)
    assert rep["slices"] == max(sb) and rep["slices_min"] == min(sb)
    s_glob, _ = oracle.auto_slices(A, B, prec, method)
    assert s_glob == max(sb)
    srow = [sb[i // 256] for i in range(m)]
    si, sj = samples_for(m, n, 250, seed=k)
    Rs = oracle.ozaki_rows(A, B, prec, method, max(sb), srow, samples=(si, sj))
    bad = sampled_equal(C, Rs, si, sj)
    assert bad is None, bad
    Xs = oracle.exact(A, B, prec + 64, method, samples=(si, sj))
    assert max_err_log2(A, B, C, Xs, samples=(si, sj), ref_is_sampled=True) <= -(prec - BOUND[method])


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_adaptive_uniform_equals_plain(method):
    """Rows of one distribution: every block gets the global s, and the result is bitwise the
    non-adaptive call's."""
    A = mpgen.random_cmat(5, 1, 520, 64, 128)
    B = mpgen.random_cmat(5, 2, 64, 130, 128)
    dA, dB = P.to_device(A), P.to_device(B)
    C0, r0 = P.gemm(dA, dB, 128, method)
    C1, r1 = P.gemm(dA, dB, 128, method, adaptive=1)
    torch.cuda.synchronize()
    assert r1["block_slices"] == [r0["slices"]] * 3
    assert same_bits(P.to_host(C0), P.to_host(C1))


def test_adaptive_accumulate_bitexact():
    """NEXT-2 + NEXT-4: C := C0 - A B with per-block slice counts, one rounding."""
    method, prec, k = "3M", 128, 40
    A = mixed_rows(11, k, prec, (0, 30), (256, 20), zero_frac=0.2)
    B = mpgen.random_cmat(11, 8, k, 70, prec, 1)
    C0 = mpgen.random_cmat(11, 9, 276, 70, prec, 3)
    m, n = 276, 70
    sb, ok = oracle.block_slices(A, B, prec, method, block=256)
    assert ok and sb[0] != sb[1]
    dA, dB, dC = P.to_device(A), P.to_device(B), P.to_device(C0)
    rep = P.mpcgemm_ex(dA, dB, dC, prec, method, beta=1, alpha_neg=1, adaptive=1)
    torch.cuda.synchronize()
    assert rep["block_slices"] == sb
    C = P.to_host(dC)
    si, sj = samples_for(m, n, 200, seed=3)
    srow = np.array([sb[i // 256] for i in range(m)], np.int32)
    # the oracle's accumulate mode with a per-row triangle: one row block at a time
    for b, s_b in enumerate(sb):
        r0, r1 = 256 * b, min(m, 256 * (b + 1))
        sel = (si >= r0) & (si < r1)
        Rs = oracle.ozaki_acc(A.rows(r0, r1), B, C0.rows(r0, r1), prec, method, s=max(sb), beta=1, alpha_neg=1,
                              samples=(si[sel] - r0, sj[sel]), srow=srow[r0:r1])
        bad = sampled_equal(C.rows(r0, r1), Rs, si[sel] - r0, sj[sel])
        assert bad is None, (b, bad)


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_adaptive_simt_crosscheck_and_cut_pairs(method, monkeypatch):
    """Blocks whose last diagonal s_b + 1 opens a diagonal pair run G = 3 units (D_r alone):
    the tensor-core kernels equal the dp4a cross-check kernel and the oracle, and the MMA count
    drops by exactly the skipped diagonals."""
    prec, k = 128, 200
    found = None
    for seed in range(40):                              # blocks with an odd s_b < s_max
        A = mixed_rows(seed, k, prec, (0, 40), (256, 40), zero_frac=0.3)
        B = mpgen.random_cmat(seed, 7, k, 260, prec, 1)
        sb, ok = oracle.block_slices(A, B, prec, method, block=256)
        if ok and min(sb) < max(sb) and min(sb) % 2 == 1:
            found = (A, B, sb)
            break
    assert found, "no seed with an odd smaller block slice count"
    A, B, sb = found
    dA, dB = P.to_device(A), P.to_device(B)
    C1, r1 = P.gemm(dA, dB, prec, method, adaptive=1)
    C0, r0 = P.gemm(dA, dB, prec, method, adaptive=0)
    monkeypatch.setenv("MPCGEMM_SLICEGEMM_SIMT", "1")
    C2, r2 = P.gemm(dA, dB, prec, method, adaptive=1)
    torch.cuda.synchronize()
    assert r1["block_slices"] == sb and same_bits(P.to_host(C1), P.to_host(C2))
    assert r1["mma_instructions"] < r0["mma_instructions"]
    m, n = A.shape[0], B.shape[1]
    si, sj = samples_for(m, n, 150, seed=9)
    srow = [sb[i // 256] for i in range(m)]
    Rs = oracle.ozaki_rows(A, B, prec, method, max(sb), srow, samples=(si, sj))
    assert sampled_equal(P.to_host(C1), Rs, si, sj) is None
