"""Dense full-size parity at the BASELINE configurations in the bench's launch configuration
("make full-size parity dense").

* configs 3 and 4, 3M and 4M: the GPU's s equals oracle.auto_slices at full size (the certified
  rule); at least one random output in every
  128 x 256 half tile a CTA of the pair kernel writes, plus the four corners of every half tile,
  bit-exact against oracle.ozaki (Algorithm 2) and within BASELINE's bound
  2^-(prec-8) (4M) / 2^-(prec-9) (3M) against oracle.exact (the plain definition);
* config 4: ALL 4.19 M outputs of the tcgen05 path bitwise equal to the dp4a CUDA-core kernel
  (MPCGEMM_SLICEGEMM_SIMT=1) over the same work list;
* config 5: all 15 LU-update GEMMs, both methods, sampled bit-exact."""
import math

import numpy as np
import pytest

import mpgen
import oracle
from harness import first_mismatch, max_err_log2, same_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2307_06072_b200 as P  # noqa: E402

BOUND = {"4M": 8, "3M": 9}


def run(A, B, prec, method, slices=0):
    dA, dB = P.to_device(A), P.to_device(B)
    dC = P.empty_device(A.shape[0], B.shape[1], prec)
    rep = P.mpcgemm_ex(dA, dB, dC, prec, method, slices=slices)
    torch.cuda.synchronize()
    return dC, rep


def half_tile_samples(m, n, seed):
    """One random output per 128 x 256 half tile (rows r0..r0+127 of a 256-row pair tile) and
    the four corners of every half tile."""
    rng = np.random.default_rng(seed)
    si, sj = [], []
    for r0 in range(0, m, 128):
        for c0 in range(0, n, 256):
            r1, c1 = min(m, r0 + 128) - 1, min(n, c0 + 256) - 1
            si.append(int(rng.integers(r0, r1 + 1))); sj.append(int(rng.integers(c0, c1 + 1)))
            for i, j in ((r0, c0), (r0, c1), (r1, c0), (r1, c1)):
                si.append(i); sj.append(j)
    return np.array(si), np.array(sj)


def sampled_mismatch(C, Rs, si, sj):
    for part in ("re", "im"):
        a, b = getattr(C, part), getattr(Rs, part)
        ok = (a.sign[si, sj] == b.sign[0]) & (a.exp[si, sj] == b.exp[0]) & np.all(a.limbs[si, sj] == b.limbs[0], axis=-1)
        if not ok.all():
            t = int(np.argmin(ok))
            return part, int(si[t]), int(sj[t])
    return None


@pytest.mark.parametrize("cfg", [2, 3, 4])
@pytest.mark.parametrize("method", ["3M", "4M"])
def test_dense_half_tile_parity(cfg, method):
    c = mpgen.CONFIGS[cfg]
    A, B = mpgen.config_inputs(cfg, seed=0)
    dC, rep = run(A, B, c["prec"], method)
    s_ref, ok = oracle.auto_slices(A, B, c["prec"], method)
    assert ok and rep["slices"] == s_ref, (rep["slices"], s_ref)
    C = P.to_host(dC)
    si, sj = half_tile_samples(c["m"], c["n"], seed=10 * cfg + (method == "4M"))
    assert len(si) >= 5 * (c["m"] // 128) * (c["n"] // 256)
    Rs = oracle.ozaki(A, B, c["prec"], method, s_ref, samples=(si, sj))
    assert sampled_mismatch(C, Rs, si, sj) is None
    Xs = oracle.exact(A, B, c["prec"] + 64, method, samples=(si, sj))
    assert max_err_log2(A, B, C, Xs, samples=(si, sj), ref_is_sampled=True) <= -(c["prec"] - BOUND[method])


@pytest.mark.parametrize("method", ["3M"])
def test_config4_full_tcgen05_vs_simt(method, monkeypatch):
    """Every one of the 2 x 2048^2 outputs: tcgen05 kernel == dp4a kernel, bitwise."""
    A, B = mpgen.config_inputs(4, seed=0)
    dA, dB = P.to_device(A), P.to_device(B)
    C1 = P.empty_device(2048, 2048, 1024)
    r1 = P.mpcgemm_ex(dA, dB, C1, 1024, method)
    monkeypatch.setenv("MPCGEMM_SLICEGEMM_SIMT", "1")
    C2 = P.empty_device(2048, 2048, 1024)
    r2 = P.mpcgemm_ex(dA, dB, C2, 1024, method)
    monkeypatch.delenv("MPCGEMM_SLICEGEMM_SIMT")
    torch.cuda.synchronize()
    assert r1["slices"] == r2["slices"] == 129
    for p in ("re", "im"):
        for f in ("sign", "exp", "limbs"):
            assert torch.equal(getattr(getattr(C1, p), f), getattr(getattr(C2, p), f)), (p, f)


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_config5_all_updates_sampled(method):
    """BASELINE config 5: all 15 Schur-update GEMMs (n - j nb) x nb . nb x (n - j nb), prec 768."""
    count = 0
    for j, L21, U12 in mpgen.lu_update_gemms(seed=0):
        dC, rep = run(L21, U12, 768, method)
        s_ref, ok = oracle.auto_slices(L21, U12, 768, method)
        assert ok and rep["slices"] == s_ref, (j, rep["slices"], s_ref)
        C = P.to_host(dC)
        mm, nn = L21.shape[0], U12.shape[1]
        rng = np.random.default_rng(j)
        si = np.concatenate([rng.integers(0, mm, 10), [0, mm - 1, 0, mm - 1]])
        sj = np.concatenate([rng.integers(0, nn, 10), [0, nn - 1, nn - 1, 0]])
        Rs = oracle.ozaki(L21, U12, 768, method, s_ref, samples=(si, sj))
        assert sampled_mismatch(C, Rs, si, sj) is None, j
        count += 1
    assert count == 15


def test_config2_fold_occupancy_variants_bitexact(monkeypatch):
    """Config 2's fold grid (1024 CTAs) is just over one wave of 6 CTAs per SM, so it runs the
    7-CTA register budget; the 6-CTA variant (MPCGEMM_FOLD_NO7) gives the same bits."""
    c = mpgen.CONFIGS[2]
    A, B = mpgen.config_inputs(2, seed=1)
    C0, r0 = run(A, B, c["prec"], "3M")
    monkeypatch.setenv("MPCGEMM_FOLD_NO7", "1")
    C1, r1 = run(A, B, c["prec"], "3M")
    assert r0["slices"] == r1["slices"]
    H0, H1 = P.to_host(C0), P.to_host(C1)
    for part in ("re", "im"):
        a, b = getattr(H0, part), getattr(H1, part)
        assert np.array_equal(a.sign, b.sign) and np.array_equal(a.exp, b.exp) and np.array_equal(a.limbs, b.limbs)
