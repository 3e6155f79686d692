"""Randomised GPU parity: 160 seeded combinations of shape (incl. 1 and ragged tile tails), precision
(every limb count 1..16 and a few wide ones), exponent spread, zero fraction, method, slice count
(auto / forced), adaptive blocks, accumulate mode and padded leading dimensions -- every sampled output
bit-exact against the oracle (Algorithm 2 under the DESIGN.md readings).  MPCGEMM_FUZZ_SEEDS=N
runs N seeds (a longer sweep)."""
import os

import numpy as np
import pytest

import mpgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2307_06072_b200 as P  # noqa: E402

from test_gpu_parity import sampled_equal  # noqa: E402


def case(seed):
    rng = np.random.default_rng(1000 + seed)
    m = int(rng.choice([1, 3, 17, 129, 200, 257, 300]))
    n = int(rng.choice([1, 5, 64, 130, 255, 257, 320]))
    k = int(rng.choice([1, 2, 31, 64, 100, 129, 300]))
    prec = int(rng.choice([2, 53, 64, 65, 127, 128, 192, 256, 320, 384, 448, 512, 576, 640, 704, 768, 832, 896,
                           960, 1024, 1500]))
    spread = int(rng.choice([0, 1, 4, 16, 60]))
    zf = float(rng.choice([0.0, 0.0, 0.1, 0.5]))
    method = str(rng.choice(["3M", "4M"]))
    forced = int(rng.choice([0, 0, 0, 5, 23]))
    adaptive = int(rng.integers(0, 2))
    beta = int(rng.integers(0, 2))
    pad = int(rng.choice([0, 0, 3]))
    return m, n, k, prec, spread, zf, method, forced, adaptive, beta, pad


@pytest.mark.parametrize("seed", list(range(int(os.environ.get("MPCGEMM_FUZZ_SEEDS", "160")))))
def test_fuzz_bitexact(seed):
    m, n, k, prec, spread, zf, method, forced, adaptive, beta, pad = case(seed)
    A = mpgen.random_cmat(seed, 1, m, k, prec, spread, zero_frac=zf)
    B = mpgen.random_cmat(seed, 2, k, n, prec, spread, zero_frac=zf)
    C0 = mpgen.random_cmat(seed, 3, m, n, prec, spread, zero_frac=zf)
    dA = P.to_device(A, ld=k + pad if pad else None)
    dB = P.to_device(B, ld=n + pad if pad else None)
    dC = P.to_device(C0, ld=n + pad if pad else None) if beta else P.empty_device(m, n, prec, ld=n + pad if pad else None)
    rep = P.mpcgemm_ex(dA, dB, dC, prec, method, slices=forced, adaptive=adaptive if not forced else 0, beta=beta)
    torch.cuda.synchronize()
    C = P.to_host(dC)
    s = rep["slices"]
    if not forced:
        sb, ok = oracle.block_slices(A, B, prec, method, block=256)
        assert ok
        if adaptive:
            assert rep["block_slices"] == sb
        else:
            assert s == max(sb)
    rng = np.random.default_rng(seed)
    cnt = min(m * n, 60)
    si = np.concatenate([rng.integers(0, m, cnt), [0, m - 1]])
    sj = np.concatenate([rng.integers(0, n, cnt), [n - 1, 0]])
    srow = [rep["block_slices"][i // 256] for i in range(m)] if (adaptive and not forced) else None
    if beta:
        Rs = oracle.ozaki_acc(A, B, C0, prec, method, s=s, beta=1, samples=(si, sj), srow=srow)
    elif srow is not None:
        Rs = oracle.ozaki_rows(A, B, prec, method, s, srow, samples=(si, sj))
    else:
        Rs = oracle.ozaki(A, B, prec, method, s, samples=(si, sj))
    bad = sampled_equal(C, Rs, si, sj)
    assert bad is None, (case(seed), bad)


def case_large(seed):
    rng = np.random.default_rng(5000 + seed)
    m = int(rng.choice([257, 513, 700, 1100]))
    n = int(rng.choice([129, 300, 640, 1024]))
    k = int(rng.choice([128, 255, 600, 1300]))
    prec = int(rng.choice([256, 320, 512, 768, 1024]))
    spread = int(rng.choice([0, 2, 16]))
    method = str(rng.choice(["3M", "4M"]))
    beta = int(rng.integers(0, 2))
    return m, n, k, prec, spread, method, beta


@pytest.mark.parametrize("seed", list(range(int(os.environ.get("MPCGEMM_FUZZ_LARGE", "4")))))
def test_fuzz_large_bitexact(seed):
    """Larger shapes (many tiles, exactness chunks, p-blocks, k-phase hints, ragged k-blocks):
    sampled outputs bit-exact against the oracle.  MPCGEMM_FUZZ_LARGE=N runs N seeds."""
    m, n, k, prec, spread, method, beta = case_large(seed)
    A = mpgen.random_cmat(seed, 11, m, k, prec, spread)
    B = mpgen.random_cmat(seed, 12, k, n, prec, spread)
    C0 = mpgen.random_cmat(seed, 13, m, n, prec, spread)
    dA, dB = P.to_device(A), P.to_device(B)
    dC = P.to_device(C0) if beta else P.empty_device(m, n, prec)
    rep = P.mpcgemm_ex(dA, dB, dC, prec, method, beta=beta)
    torch.cuda.synchronize()
    C = P.to_host(dC)
    rng = np.random.default_rng(seed)
    si = np.concatenate([rng.integers(0, m, 24), [0, m - 1, 255, 256]])
    sj = np.concatenate([rng.integers(0, n, 24), [n - 1, 0, 127, 128]])
    if beta:
        Rs = oracle.ozaki_acc(A, B, C0, prec, method, s=rep["slices"], beta=1, samples=(si, sj))
    else:
        Rs = oracle.ozaki(A, B, prec, method, rep["slices"], samples=(si, sj))
    bad = sampled_equal(C, Rs, si, sj)
    assert bad is None, (case_large(seed), bad)
