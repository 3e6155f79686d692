"""Operation counts of the slice GEMM against Table 1's closed form (the
work of one real product is the triangle of d(d+1)/2 slice products, Algorithm 2's loop
beta <= d - alpha + 1).

The tcgen05 kernels count the MMA instructions their issuing thread actually issues
(rep["mma_issued"], summed over CTAs on the device); the host plan predicts the same number
(rep["mma_instructions"]).  Both must equal
    R * P * ceil(m / tile_m) * ceil(n / tile_n) * ceil(k / 32),   P = s (s + 1) / 2,
R = 3 (3M: T1, T2, T3) or 4 (4M: two products per part), K = 32 per kind::i8 MMA and the zero
padding of the last k-block skipped.  A triangle one diagonal too long or too short changes P
and fails this test even where the results could not tell (e.g. zero digits)."""
import math

import pytest

import mpgen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2307_06072_b200 as P  # noqa: E402

R_OF = {"3M": 3, "4M": 4}


def closed_form(rep, m, n, k, method):
    s = rep["slices"]
    return R_OF[method] * (s * (s + 1) // 2) * math.ceil(m / rep["tile_m"]) * math.ceil(n / rep["tile_n"]) * math.ceil(k / 32)


def timed(A, B, prec, method, slices=0):
    dA, dB = P.to_device(A), P.to_device(B)
    dC = P.empty_device(A.shape[0], B.shape[1], prec)
    rep = P.mpcgemm_ex(dA, dB, dC, prec, method, slices=slices, timing=1)
    torch.cuda.synchronize()
    return rep


@pytest.mark.parametrize("method", ["3M", "4M"])
@pytest.mark.parametrize("m,n,k,prec,slices", [(300, 520, 200, 256, 0), (256, 256, 128, 128, 0), (130, 100, 97, 192, 0),
                                               (70, 600, 1000, 128, 0), (513, 257, 33, 64, 9), (200, 300, 4200, 64, 5),
                                               (96, 400, 130, 512, 70)])
def test_mma_count_closed_form(method, m, n, k, prec, slices):
    A = mpgen.random_cmat(m + k, 1, m, k, prec, 2)
    B = mpgen.random_cmat(m + k, 2, k, n, prec, 2)
    rep = timed(A, B, prec, method, slices)
    want = closed_form(rep, m, n, k, method)
    assert rep["mma_instructions"] == want, (rep["mma_instructions"], want)
    assert rep["mma_issued"] == want, (rep["mma_issued"], want)


@pytest.mark.parametrize("cta2", ["0", "1"])
def test_mma_count_both_kernels(cta2, monkeypatch):
    """Both tcgen05 kernels (CTA pair 256 x 256 tiles; one CTA 128 x 256) and both unit kinds
    (two diagonals per unit; MPCGEMM_G2=0: one)."""
    monkeypatch.setenv("MPCGEMM_CTA2", cta2)
    m, n, k, prec = 270, 390, 300, 160
    A = mpgen.random_cmat(3, 1, m, k, prec, 3)
    B = mpgen.random_cmat(3, 2, k, n, prec, 3)
    for g2 in ("1", "0"):
        monkeypatch.setenv("MPCGEMM_G2", g2)
        for method in ("3M", "4M"):
            rep = timed(A, B, prec, method)
            assert rep["tile_m"] == (256 if cta2 == "1" else 128) and rep["tile_n"] == 256
            want = closed_form(rep, m, n, k, method)
            assert rep["mma_instructions"] == want and rep["mma_issued"] == want, (g2, method, rep["mma_issued"], want)


def test_mma_count_config4():
    """BASELINE config 4 (the bench workload): 3 * 8385 * 8 * 8 * 64 = 103,034,880 pair MMAs."""
    A, B = mpgen.config_inputs(4, seed=0)
    rep = timed(A, B, 1024, "3M")
    want = closed_form(rep, 2048, 2048, 2048, "3M")
    assert rep["slices"] == 129 and want == 3 * 8385 * 8 * 8 * 64
    assert rep["mma_instructions"] == want and rep["mma_issued"] == want
