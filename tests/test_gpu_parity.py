"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same seeded inputs.

Bit-exact: every output entry of the GPU equals oracle.ozaki (Algorithm 2 under the DESIGN.md
readings, same s) -- the whole path is integer arithmetic plus one RNE, so no tolerance.
Within bound: against oracle.exact (the plain definition, prec+64 bits), the BASELINE.json
acceptance e <= 2^-(prec-8) (4M) / 2^-(prec-9) (3M).
Sizes span several 128-row / 256-col tiles with ragged tails; the BASELINE configs run at full
size in the bench's launch configuration and are checked on sampled outputs."""
import math
import os

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


def run_gpu(A, B, prec, method, slices=0):
    dA, dB = P.to_device(A), P.to_device(B)
    dC, rep = P.gemm(dA, dB, prec, method, slices)
    torch.cuda.synchronize()
    return P.to_host(dC), rep


def sample_idx(m, n, count, seed=0):
    rng = np.random.default_rng(seed)
    si = list(rng.integers(0, m, count))
    sj = list(rng.integers(0, n, count))
    for i in (0, m - 1, min(127, m - 1), min(128, m - 1)):         # tile edges and the ragged tail
        for j in (0, n - 1, min(255, n - 1), min(256, n - 1)):
            si.append(i); sj.append(j)
    return np.array(si), np.array(sj)


def sampled_equal(C, Rs, si, sj):
    for part in ("re", "im"):
        a, b = getattr(C, part), getattr(Rs, part)
        for t in range(len(si)):
            i, j = si[t], sj[t]
            if a.sign[i, j] != b.sign[0, t] or a.exp[i, j] != b.exp[0, t] or not np.array_equal(a.limbs[i, j], b.limbs[0, t]):
                return (part, int(i), int(j))
    return None


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_config1_full_bitexact(method):
    """BASELINE config 1 (64^3, prec 128, seed 0): every entry bit-exact vs the oracle."""
    A, B = mpgen.config_inputs(1, seed=0)
    C, rep = run_gpu(A, B, 128, method)
    s_ref, ok = oracle.auto_slices(A, B, 128, method)
    assert ok and rep["slices"] == s_ref
    R = oracle.ozaki(A, B, 128, method, s_ref)
    assert same_bits(C, R), first_mismatch(C, R)
    Cx = oracle.exact(A, B, 128 + 64, method)
    assert max_err_log2(A, B, C, Cx) <= -(128 - BOUND[method])


@pytest.mark.parametrize("method", ["3M", "4M"])
@pytest.mark.parametrize("m,n,k,prec,spread", [(200, 300, 150, 192, 8), (130, 257, 129, 64, 0), (1, 1, 1, 100, 0),
                                               (3, 517, 33, 256, 2)])
def test_ragged_sampled_bitexact(method, m, n, k, prec, spread):
    A = mpgen.random_cmat(m + n + k, 5, m, k, prec, spread, zero_frac=0.05)
    B = mpgen.random_cmat(m + n + k, 6, k, n, prec, spread, zero_frac=0.05)
    C, rep = run_gpu(A, B, prec, method)
    s_ref, ok = oracle.auto_slices(A, B, prec, method)
    assert rep["slices"] == s_ref
    si, sj = sample_idx(m, n, 300, seed=m)
    Rs = oracle.ozaki(A, B, prec, method, s_ref, samples=(si, sj))
    assert sampled_equal(C, Rs, si, sj) is None
    Xs = oracle.exact(A, B, prec + 64, method, samples=(si, sj))
    assert max_err_log2(A, B, C, Xs, samples=(si, sj), ref_is_sampled=True) <= -(prec - BOUND[method])


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_simt_crosscheck_and_forced_slices(method, monkeypatch):
    """tcgen05 kernel == dp4a SIMT kernel bitwise over the same work list; forced s values."""
    m, n, k, prec = 150, 280, 300, 160
    A = mpgen.random_cmat(3, 7, m, k, prec, 5)
    B = mpgen.random_cmat(3, 8, k, n, prec, 5)
    for s in (0, 2, 7, 40):
        C1, r1 = run_gpu(A, B, prec, method, s)
        monkeypatch.setenv("MPCGEMM_SLICEGEMM_SIMT", "1")
        C2, r2 = run_gpu(A, B, prec, method, s)
        monkeypatch.delenv("MPCGEMM_SLICEGEMM_SIMT")
        monkeypatch.setenv("MPCGEMM_G2", "0")                  # single-diagonal units only
        C3, r3 = run_gpu(A, B, prec, method, s)
        monkeypatch.delenv("MPCGEMM_G2")
        monkeypatch.setenv("MPCGEMM_CTA2", "0")                # one CTA per 128-row tile
        C4, r4 = run_gpu(A, B, prec, method, s)
        monkeypatch.delenv("MPCGEMM_CTA2")
        assert r1["slices"] == r2["slices"] == r3["slices"] == r4["slices"]
        assert same_bits(C1, C2), (s, first_mismatch(C1, C2))
        assert same_bits(C1, C3), (s, first_mismatch(C1, C3))
        assert same_bits(C1, C4), (s, first_mismatch(C1, C4))
        if s:
            si, sj = sample_idx(m, n, 60, seed=s)
            Rs = oracle.ozaki(A, B, prec, method, s, samples=(si, sj))
            assert sampled_equal(C1, Rs, si, sj) is None


def test_small_chunks_equal_default(monkeypatch):
    """Any chunking of the INT32 accumulation gives the same result (exact integer sums)."""
    m, n, k, prec = 140, 140, 700, 128
    A = mpgen.random_cmat(4, 7, m, k, prec, 2)
    B = mpgen.random_cmat(4, 8, k, n, prec, 2)
    C1, _ = run_gpu(A, B, prec, "4M")
    monkeypatch.setenv("MPCGEMM_MAXKB", "3")
    C2, _ = run_gpu(A, B, prec, "4M")
    monkeypatch.setenv("MPCGEMM_BN", "128")
    C3, _ = run_gpu(A, B, prec, "4M")
    monkeypatch.setenv("MPCGEMM_G2", "0")
    C4, _ = run_gpu(A, B, prec, "4M")
    monkeypatch.setenv("MPCGEMM_BN", "256")
    monkeypatch.setenv("MPCGEMM_CTA2", "0")
    C5, _ = run_gpu(A, B, prec, "4M")
    assert same_bits(C1, C2) and same_bits(C1, C3) and same_bits(C1, C4) and same_bits(C1, C5)


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_schedule_variants_bitexact(method, monkeypatch):
    """The CTA-pair kernel's walk order is free (exact integer sums): p-blocks of 1..7 planes (lead
    stages for D_r; even and absolute-aligned splits), k-phase hints off / per group / class-wide
    (units starting mid-walk, also from a previous call's stale hints), serpentine off, the three
    unit orders, many exactness chunks -- all bitwise equal, and equal to the oracle."""
    m, n, k, prec = 300, 260, 900, 256
    A = mpgen.random_cmat(21, 1, m, k, prec, 3)
    B = mpgen.random_cmat(21, 2, k, n, prec, 3)
    C0, rep = run_gpu(A, B, prec, method)
    variants = [{"MPCGEMM_PBLK": "1"}, {"MPCGEMM_PBLK": "3"}, {"MPCGEMM_PBLK": "7", "MPCGEMM_MAXKB": "2"},
                {"MPCGEMM_PBLK": "0", "MPCGEMM_KPHASE": "0"}, {"MPCGEMM_KPHASE": "0", "MPCGEMM_SERPENTINE": "0"},
                {"MPCGEMM_PBLK": "5", "MPCGEMM_SERPENTINE": "0", "MPCGEMM_MAXKB": "3"},
                {"MPCGEMM_KPHASE": "1", "MPCGEMM_PBLK": "32"}, {"MPCGEMM_KPHASE": "1", "MPCGEMM_ORDER": "1"},
                {"MPCGEMM_KPHASE": "2", "MPCGEMM_PBLK": "3", "MPCGEMM_MAXKB": "2"},
                {"MPCGEMM_KPHASE": "2", "MPCGEMM_PBLK": "2", "MPCGEMM_ORDER": "0"},
                {"MPCGEMM_KPHASE": "3", "MPCGEMM_PBLK": "3", "MPCGEMM_ORDER": "3"}]
    for v in variants:
        for key in ("MPCGEMM_PBLK", "MPCGEMM_KPHASE", "MPCGEMM_SERPENTINE", "MPCGEMM_MAXKB", "MPCGEMM_ORDER"):
            monkeypatch.delenv(key, raising=False)
        for key, val in v.items():
            monkeypatch.setenv(key, val)
        for _ in range(2):
            C1, _ = run_gpu(A, B, prec, method)
            assert same_bits(C0, C1), (v, first_mismatch(C0, C1))
    si, sj = sample_idx(m, n, 60, seed=5)
    Rs = oracle.ozaki(A, B, prec, method, rep["slices"], samples=(si, sj))
    assert sampled_equal(C0, Rs, si, sj) is None


@pytest.mark.parametrize("spread,k", [(16, 12), (16, 3), (0, 64), (4, 40)])
def test_prepass_matches_oracle(spread, k):
    """rho-hat pre-pass integers and the resulting s equal the oracle's (incl. the minT == 0
    max-plus stage)."""
    m, n, prec = 70, 90, 256
    A = mpgen.random_cmat(spread + k, 9, m, k, prec, spread, zero_frac=0.1)
    B = mpgen.random_cmat(spread + k, 10, k, n, prec, spread, zero_frac=0.1)
    dA, dB = P.to_device(A), P.to_device(B)
    got = P.mpcgemm_rho_bounds(dA, dB, prec)
    assert got == oracle.rho_bounds(A, B)
    for method in ("3M", "4M"):
        C, rep = run_gpu(A, B, prec, method)
        assert rep["slices"] == oracle.auto_slices(A, B, prec, method)[0]
        si, sj = sample_idx(m, n, 80)
        Rs = oracle.ozaki(A, B, prec, method, rep["slices"], samples=(si, sj))
        assert sampled_equal(C, Rs, si, sj) is None


@pytest.mark.parametrize("spread,k", [(16, 12), (0, 64), (30, 200)])
def test_planes_top_bytes_on_off(spread, k, monkeypatch):
    """The a-2 planes from the a-1 scan's top bytes (default) and from the limbs (MPCGEMM_PLANES_TB=0)
    give the same pre-pass integers, s and bits, for both methods."""
    m, n, prec = 150, 70, 320
    A = mpgen.random_cmat(spread + k, 21, m, k, prec, spread, zero_frac=0.1)
    B = mpgen.random_cmat(spread + k, 22, k, n, prec, spread, zero_frac=0.1)
    for method in ("3M", "4M"):
        out = []
        for tb in ("1", "0"):
            monkeypatch.setenv("MPCGEMM_PLANES_TB", tb)
            C, rep = run_gpu(A, B, prec, method)
            out.append((rep["slices"], rep["minT"], rep["minT1"], rep["maxD2"], C))
        assert out[0][:4] == out[1][:4]
        assert same_bits(out[0][4], out[1][4])
        assert out[0][0] == oracle.auto_slices(A, B, prec, method)[0]


def test_edge_cases():
    prec = 128
    A = mpgen.random_cmat(1, 1, 5, 0, prec)
    B = mpgen.random_cmat(1, 2, 0, 7, prec)
    C, _ = run_gpu(A, B, prec, "3M")                      # k = 0: C = 0
    assert not C.re.limbs.any() and not C.im.limbs.any() and not C.re.exp.any()
    A = mpgen.random_cmat(1, 1, 0, 9, prec)
    B = mpgen.random_cmat(1, 2, 9, 4, prec)
    C, _ = run_gpu(A, B, prec, "4M")                      # m = 0
    assert C.shape == (0, 4)
    # zero rows / columns and an all-zero operand
    A = mpgen.random_cmat(2, 1, 6, 9, prec)
    B = mpgen.random_cmat(2, 2, 9, 5, prec)
    for R in (A.re, A.im):
        R.sign[3] = 0; R.exp[3] = 0; R.limbs[3] = 0
    for R in (B.re, B.im):
        R.limbs[:, 2] = 0; R.exp[:, 2] = 0; R.sign[:, 2] = 0
    for method in ("3M", "4M"):
        C, rep = run_gpu(A, B, prec, method)
        assert same_bits(C, oracle.ozaki(A, B, prec, method, rep["slices"]))
        assert not C.re.limbs[3].any() and not C.im.limbs[:, 2].any()
    Z = mpgen.CMat(mpgen.empty_rmat(4, 6, prec), mpgen.empty_rmat(4, 6, prec))
    C, _ = run_gpu(Z, B.rows(0, 6), prec, "3M")
    assert not C.re.limbs.any()


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_integer_closure_and_identity(method):
    import random
    rnd = random.Random(1)
    m, k, n = 37, 45, 29
    mk = lambda r, c: [[rnd.randint(-8, 8) for _ in range(c)] for _ in range(r)]
    A = mpgen.CMat(mpgen.from_ints(mk(m, k), 128), mpgen.from_ints(mk(m, k), 128))
    B = mpgen.CMat(mpgen.from_ints(mk(k, n), 128), mpgen.from_ints(mk(k, n), 128))
    C, _ = run_gpu(A, B, 128, method)
    assert same_bits(C, oracle.exact(A, B, 128, method))
    # B = I with rows of equal exponent: every bit captured -> C == A
    A2 = mpgen.random_cmat(11, 1, 20, 20, 128)
    for R in (A2.re, A2.im):
        R.exp[:] = 0
    I = mpgen.CMat(mpgen.from_ints([[int(i == j) for j in range(20)] for i in range(20)], 128),
                   mpgen.from_ints([[0] * 20 for _ in range(20)], 128))
    C, _ = run_gpu(A2, I, 128, method)
    assert same_bits(C, A2)


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_transposition_bitwise(method):
    prec = 192
    A = mpgen.random_cmat(21, 1, 90, 70, prec, 6)
    B = mpgen.random_cmat(21, 2, 70, 110, prec, 6)
    s = oracle.auto_slices(A, B, prec, method)[0]
    C, _ = run_gpu(A, B, prec, method, s)
    Ct, _ = run_gpu(B.T(), A.T(), prec, method, s)
    assert same_bits(Ct, C.T())


def test_host_entry_matches_device():
    prec = 256
    A = mpgen.random_cmat(31, 1, 100, 90, prec, 3)
    B = mpgen.random_cmat(31, 2, 90, 120, prec, 3)
    for method in ("3M", "4M"):
        C1, r1 = run_gpu(A, B, prec, method)
        C2, r2 = P.mpcgemm_host(A, B, prec, method)
        assert r1["slices"] == r2["slices"] and same_bits(C1, C2)


@pytest.mark.parametrize("group", [0, 256])
def test_host_async_pipeline(monkeypatch, group):
    """mpcgemm_host_async: five products queued back to back (two staging sets in turn, row
    groups or not, different shapes / precisions / methods, one with beta = 1) -- after
    mpcgemm_host_wait every C equals the blocking mpcgemm_host result bitwise; an argument error
    while calls are queued is reported and leaves the pipeline usable."""
    monkeypatch.setenv("MPCGEMM_HOST_GROUP", str(group))
    cases = [(300, 90, 200, 192, "3M", 0), (530, 70, 260, 256, "4M", 0), (257, 40, 300, 128, "3M", 1),
             (600, 64, 129, 320, "4M", 0), (100, 33, 80, 64, "3M", 0)]
    probs = []
    for i, (m, k, n, prec, method, beta) in enumerate(cases):
        A = mpgen.random_cmat(50 + i, 1, m, k, prec, 4)
        B = mpgen.random_cmat(50 + i, 2, k, n, prec, 4)
        C0 = mpgen.random_cmat(50 + i, 3, m, n, prec, 2)
        ref, _ = P.mpcgemm_host(A, B, prec, method, C=C0.copy() if beta else None, beta=beta)
        probs.append((A, B, C0, prec, method, beta, ref))
    outs = []
    for A, B, C0, prec, method, beta, _ in probs:
        C, rep = P.mpcgemm_host_async(A, B, prec, method, C=C0.copy() if beta else None, beta=beta)
        outs.append(C)
    with pytest.raises(P.MpcgemmError):
        P.mpcgemm_host_async(probs[0][0], probs[0][1], 5000, "3M")
    P.mpcgemm_host_wait()
    for (A, B, C0, prec, method, beta, ref), C in zip(probs, outs):
        assert same_bits(ref, C), (prec, method, beta, first_mismatch(ref, C))
    C, _ = P.mpcgemm_host_async(probs[1][0], probs[1][1], probs[1][3], probs[1][4])
    P.mpcgemm_host_wait()
    assert same_bits(probs[1][6], C)


@pytest.mark.parametrize("group", [256, 512])
def test_host_entry_row_groups(monkeypatch, group):
    """mpcgemm_host in row groups (D2H of finished groups overlapping the next group's compute):
    bitwise the one-call device result, incl. a ragged last group, adaptive blocks and beta = 1."""
    monkeypatch.setenv("MPCGEMM_HOST_GROUP", str(group))
    prec = 192
    A = mpgen.random_cmat(32, 1, 700, 70, prec, 3)
    A2 = mpgen.random_cmat(32, 4, 700, 70, prec, 30, zero_frac=0.2)
    A.re.exp[300:] = A2.re.exp[300:]; A.re.limbs[300:] = A2.re.limbs[300:]; A.re.sign[300:] = A2.re.sign[300:]
    B = mpgen.random_cmat(32, 2, 70, 300, prec, 3)
    C0 = mpgen.random_cmat(32, 3, 700, 300, prec, 1)
    for method in ("3M", "4M"):
        C1, r1 = run_gpu(A, B, prec, method)
        C2, r2 = P.mpcgemm_host(A, B, prec, method)
        assert r1["slices"] == r2["slices"] and same_bits(C1, C2), first_mismatch(C1, C2)
        dA, dB = P.to_device(A), P.to_device(B)
        dC, ra = P.gemm(dA, dB, prec, method, adaptive=1)
        Ca, rb = P.mpcgemm_host(A, B, prec, method, adaptive=1)
        assert same_bits(P.to_host(dC), Ca)
        dC0 = P.to_device(C0)
        P.mpcgemm_ex(dA, dB, dC0, prec, method, beta=1, alpha_neg=1)
        Cb, _ = P.mpcgemm_host(A, B, prec, method, C=C0.copy(), beta=1, alpha_neg=1)
        assert same_bits(P.to_host(dC0), Cb)


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_workspace_limit_row_groups(monkeypatch, method):
    """A workspace budget below one call's need runs row groups (256 * 2^j rows): bitwise equal."""
    prec = 128
    A = mpgen.random_cmat(33, 1, 900, 130, prec, 2)
    B = mpgen.random_cmat(33, 2, 130, 300, prec, 2)
    C1, r1 = run_gpu(A, B, prec, method)
    need = P.mpcgemm_workspace_size(900, 300, 130, prec, method, r1["slices"])
    monkeypatch.setenv("MPCGEMM_WS_LIMIT", str(need // 3))
    C2, r2 = run_gpu(A, B, prec, method)
    assert r2["kernel_launches"] > r1["kernel_launches"]          # more than one group ran
    assert same_bits(C1, C2), first_mismatch(C1, C2)
    monkeypatch.setenv("MPCGEMM_WS_LIMIT", "1000")
    with pytest.raises(P.MpcgemmError):
        run_gpu(A, B, prec, method)


def test_concurrent_streams_share_workspace_safely():
    """Calls on different streams without host synchronisation: each call's device work is
    ordered after the previous call's (the device workspace is shared), so both results are
    the single-call results bitwise."""
    prec = 256
    A1, B1 = mpgen.random_cmat(41, 1, 300, 200, prec, 4), mpgen.random_cmat(41, 2, 200, 260, prec, 4)
    A2, B2 = mpgen.random_cmat(42, 1, 420, 150, prec, 9), mpgen.random_cmat(42, 2, 150, 310, prec, 9)
    R1, _ = run_gpu(A1, B1, prec, "3M")
    R2, _ = run_gpu(A2, B2, prec, "4M")
    dA1, dB1, dA2, dB2 = P.to_device(A1), P.to_device(B1), P.to_device(A2), P.to_device(B2)
    dC1, dC2 = P.empty_device(300, 260, prec), P.empty_device(420, 310, prec)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for _ in range(3):
        P.mpcgemm_ex(dA1, dB1, dC1, prec, "3M", stream=s1)
        P.mpcgemm_ex(dA2, dB2, dC2, prec, "4M", stream=s2)
        ipiv, _ = P.mpclu_factor(P.to_device(mpgen.random_cmat(43, 1, 40, 40, 128)), 8, "3M", stream=s1)
    torch.cuda.synchronize()
    assert same_bits(P.to_host(dC1), R1) and same_bits(P.to_host(dC2), R2)


def test_validate_and_errors():
    prec = 128
    A = mpgen.random_cmat(41, 1, 8, 8, prec)
    B = mpgen.random_cmat(41, 2, 8, 8, prec)
    bad = A.copy()
    bad.re.limbs[2, 3, -1] &= np.uint64((1 << 63) - 1)    # clear the leading bit
    dA, dB = P.to_device(bad), P.to_device(B)
    dC = P.empty_device(8, 8, prec)
    with pytest.raises(P.MpcgemmError) as e:
        P.mpcgemm_ex(dA, dB, dC, prec, "3M", validate=1)
    assert e.value.code == -4
    with pytest.raises(P.MpcgemmError) as e:
        P.mpcgemm_ex(P.to_device(A), dB, dC, 5000, "3M")
    assert e.value.code == -2
    with pytest.raises(P.MpcgemmError) as e:
        P.mpcgemm_ex(P.to_device(A), dB, dC, prec, "3M", slices=2000)
    assert e.value.code == -8


@pytest.mark.parametrize("cfg", [2, 3])
@pytest.mark.parametrize("method", ["3M", "4M"])
def test_configs_2_3_sampled(cfg, method):
    """BASELINE configs 2 and 3 at full size: sampled outputs bit-exact, within the bound."""
    c = mpgen.CONFIGS[cfg]
    A, B = mpgen.config_inputs(cfg, seed=0)
    C, rep = run_gpu(A, B, c["prec"], method)
    assert rep["slices"] == oracle.auto_slices(A, B, c["prec"], method)[0]
    si, sj = sample_idx(c["m"], c["n"], 40, seed=cfg)
    Rs = oracle.ozaki(A, B, c["prec"], method, rep["slices"], samples=(si, sj))
    assert sampled_equal(C, Rs, si, sj) is None
    Xs = oracle.exact(A, B, c["prec"] + 64, method, samples=(si, sj))
    assert max_err_log2(A, B, C, Xs, samples=(si, sj), ref_is_sampled=True) <= -(c["prec"] - BOUND[method])


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_config4_sampled(method):
    """BASELINE config 4 (2048^3, prec 1024): the bench workload, sampled bit-exact."""
    c = mpgen.CONFIGS[4]
    A, B = mpgen.config_inputs(4, seed=0)
    C, rep = run_gpu(A, B, c["prec"], method)
    assert rep["slices"] == 129 or rep["slices"] == oracle.auto_slices(A, B, c["prec"], method)[0]
    rng = np.random.default_rng(4)
    si = np.concatenate([rng.integers(0, 2048, 12), [0, 2047, 1023, 128]])
    sj = np.concatenate([rng.integers(0, 2048, 12), [2047, 0, 256, 255]])
    Rs = oracle.ozaki(A, B, c["prec"], method, rep["slices"], samples=(si, sj))
    assert sampled_equal(C, Rs, si, sj) is None
    Xs = oracle.exact(A, B, c["prec"] + 64, method, samples=(si, sj))
    assert max_err_log2(A, B, C, Xs, samples=(si, sj), ref_is_sampled=True) <= -(c["prec"] - BOUND[method])


def test_config5_lu_updates_sampled():
    """BASELINE config 5 (LU Schur updates, prec 768): first and last GEMM, sampled."""
    for j, L21, U12 in mpgen.lu_update_gemms(seed=0, js=[1, 15]):
        C, rep = run_gpu(L21, U12, 768, "3M")
        mm, nn = L21.shape[0], U12.shape[1]
        si, sj = sample_idx(mm, nn, 12, seed=j)
        Rs = oracle.ozaki(L21, U12, 768, "3M", rep["slices"], samples=(si, sj))
        assert sampled_equal(C, Rs, si, sj) is None


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_large_forced_slices(method):
    """s = 420 (fold with a 64-thread block; W = 3357 bits): sampled bit-exact."""
    m, n, k, prec = 40, 70, 20, 128
    A = mpgen.random_cmat(8, 1, m, k, prec, 30)
    B = mpgen.random_cmat(8, 2, k, n, prec, 30)
    C, rep = run_gpu(A, B, prec, method, 420)
    si, sj = sample_idx(m, n, 30, seed=5)
    Rs = oracle.ozaki(A, B, prec, method, 420, samples=(si, sj))
    assert sampled_equal(C, Rs, si, sj) is None


@pytest.mark.parametrize("method", ["3M", "4M"])
@pytest.mark.parametrize("prec,k,spread", [(2048, 12, 3), (4096, 5, 1), (1000, 9, 40)])
def test_high_precision_bitexact(method, prec, k, spread):
    """prec up to the ABI's 4096 bits (L = 64 limbs, s ~ 515): auto s, sampled bit-exact, within bound."""
    m, n = 23, 37
    A = mpgen.random_cmat(prec + k, 1, m, k, prec, spread)
    B = mpgen.random_cmat(prec + k, 2, k, n, prec, spread)
    C, rep = run_gpu(A, B, prec, method)
    assert rep["slices"] == oracle.auto_slices(A, B, prec, method)[0]
    si, sj = sample_idx(m, n, 25, seed=prec)
    Rs = oracle.ozaki(A, B, prec, method, rep["slices"], samples=(si, sj))
    assert sampled_equal(C, Rs, si, sj) is None
    Xs = oracle.exact(A, B, prec + 64, method, samples=(si, sj))
    assert max_err_log2(A, B, C, Xs, samples=(si, sj), ref_is_sampled=True) <= -(prec - BOUND[method])


@pytest.mark.parametrize("method", ["3M", "4M"])
def test_long_k_exactness_chunks(method):
    """k = 20000 (157 k-blocks): every diagonal past r ~ 7 is cut into INT32-exact chunks (<= 1023
    k-blocks per accumulator); sampled bit-exact and within bound."""
    m, n, k, prec = 33, 45, 20000, 128
    A = mpgen.random_cmat(20, 1, m, k, prec, 2)
    B = mpgen.random_cmat(20, 2, k, n, prec, 2)
    C, rep = run_gpu(A, B, prec, method)
    si, sj = sample_idx(m, n, 12, seed=20)
    Rs = oracle.ozaki(A, B, prec, method, rep["slices"], samples=(si, sj))
    assert sampled_equal(C, Rs, si, sj) is None


def test_very_long_k_many_chunks():
    """k = 800000 (6250 k-blocks): the longest diagonals are cut into > 255 exactness chunks each."""
    m, n, k, prec = 2, 3, 800000, 320
    A = mpgen.random_cmat(21, 1, m, k, prec, 1)
    B = mpgen.random_cmat(21, 2, k, n, prec, 1)
    C, rep = run_gpu(A, B, prec, "3M")
    si, sj = np.array([0, 1]), np.array([2, 0])
    Rs = oracle.ozaki(A, B, prec, "3M", rep["slices"], samples=(si, sj))
    assert sampled_equal(C, Rs, si, sj) is None


# ------------------------------------------------------------------ NEXT-2: C := C0 +- A B
def _c0_variants(m, n, prec, A, B, method):
    out = {"near": oracle.exact(A, B, prec, method)}                 # heavy cancellation
    for kind, shift, zf in (("random", 0, 0.1), ("tiny", -400, 0.0), ("huge", 300, 0.0)):
        C0 = mpgen.random_cmat(55, 9, m, n, prec, 4, zero_frac=zf)
        for R in (C0.re, C0.im):
            nz = R.limbs[..., -1] != 0
            R.exp[nz] += shift
        out[kind] = C0
    return out


@pytest.mark.parametrize("method", ["3M", "4M"])
@pytest.mark.parametrize("alpha_neg", [0, 1])
def test_accumulate_in_place_bitexact(method, alpha_neg):
    """mpcgemm_ex(beta=1): C := C + (-1)^alpha_neg A B in place, one rounding, bit-exact vs the
    oracle for every entry (incl. near-total cancellation and far-apart exponents)."""
    m, n, k, prec = 70, 300, 90, 192
    A = mpgen.random_cmat(61, 1, m, k, prec, 5, zero_frac=0.05)
    B = mpgen.random_cmat(61, 2, k, n, prec, 5, zero_frac=0.05)
    s = oracle.auto_slices(A, B, prec, method)[0]
    for kind, C0 in _c0_variants(m, n, prec, A, B, method).items():
        dA, dB, dC = P.to_device(A), P.to_device(B), P.to_device(C0)
        rep = P.mpcgemm_ex(dA, dB, dC, prec, method, beta=1, alpha_neg=alpha_neg)
        torch.cuda.synchronize()
        C = P.to_host(dC)
        assert rep["slices"] == s
        R = oracle.ozaki_acc(A, B, C0, prec, method, s, beta=1, alpha_neg=alpha_neg)
        assert same_bits(C, R), (kind, first_mismatch(C, R))


def test_accumulate_host_entry_and_beta0():
    m, n, k, prec = 33, 40, 25, 128
    A = mpgen.random_cmat(62, 1, m, k, prec, 2)
    B = mpgen.random_cmat(62, 2, k, n, prec, 2)
    C0 = mpgen.random_cmat(62, 3, m, n, prec, 2)
    s = oracle.auto_slices(A, B, prec, "3M")[0]
    C, _ = P.mpcgemm_host(A, B, prec, "3M", C=C0.copy(), beta=1, alpha_neg=1)
    assert same_bits(C, oracle.ozaki_acc(A, B, C0, prec, "3M", s, beta=1, alpha_neg=1))
    C, _ = P.mpcgemm_host(A, B, prec, "3M", alpha_neg=1)                       # beta = 0: -A B
    assert same_bits(C, oracle.ozaki_acc(A, B, C0, prec, "3M", s, beta=0, alpha_neg=1))


# ------------------------------------------------------------------ NEXT-1: binary64 carrier on DMMA
@pytest.mark.parametrize("method", ["3M", "4M"])
@pytest.mark.parametrize("m,n,k,prec,spread,d", [(70, 90, 100, 256, 4, 0), (130, 65, 257, 512, 0, 0),
                                                 (40, 50, 1024, 256, 0, 13), (33, 17, 64, 128, 8, 9)])
def test_fp64_carrier_bitexact(method, m, n, k, prec, spread, d):
    """carrier = 1: b-bit binary64 slices multiplied on FP64 DMMA, bit-exact vs the oracle's
    Algorithm 2 with the paper's slice width for the same d (auto rule when d = 0)."""
    A = mpgen.random_cmat(k + d, 1, m, k, prec, spread, zero_frac=0.05)
    B = mpgen.random_cmat(k + d, 2, k, n, prec, spread, zero_frac=0.05)
    b = oracle.fp64_slice_bits(k)
    dA, dB = P.to_device(A), P.to_device(B)
    dC, rep = P.gemm(dA, dB, prec, method, slices=d, carrier=1)
    torch.cuda.synchronize()
    C = P.to_host(dC)
    assert rep["slice_bits"] == b
    if d == 0:
        assert rep["slices"] == oracle.slices_for_bits(prec, method, k, *oracle.rho_bounds(A, B), b)
    si, sj = sample_idx(m, n, 60, seed=k)
    Rs = oracle.ozaki_bits(A, B, prec, method, rep["slices"], b, samples=(si, sj))
    assert sampled_equal(C, Rs, si, sj) is None
    if d == 0:
        Xs = oracle.exact(A, B, prec + 64, method, samples=(si, sj))
        assert max_err_log2(A, B, C, Xs, samples=(si, sj), ref_is_sampled=True) <= -(prec - BOUND[method])


@pytest.mark.parametrize("env", ["MPCGEMM_FOLD_BULK", "MPCGEMM_FOLD_SFIX", "MPCGEMM_SPLIT_V1", "MPCGEMM_FOLD_NOUNI1",
                                 "MPCGEMM_SPLIT_BYTESTG", "MPCGEMM_RESERVE_SMS", "MPCGEMM_HALFN=0",
                                 "MPCGEMM_FOLD_UNIC=0", "MPCGEMM_FOLD_UNIC=9", "MPCGEMM_FOLD_UNIC=12"])
@pytest.mark.parametrize("method", ["3M", "4M"])
def test_stage_variants_bitexact(env, method, monkeypatch):
    """The fold's bulk-copy producer, shared-memory-limbs and generic (non pair-entry) variants and the
    non-TMA / byte-staged splits give the default path's bits (the same exact integers, one rounding),
    at a ragged shape with exactness chunks and at one where every diagonal has one chunk."""
    for (m, n, k, prec) in ((200, 300, 700, 256), (130, 270, 200, 384)):
        _stage_variant_case(env, method, monkeypatch, m, n, k, prec)


def _stage_variant_case(env, method, monkeypatch, m, n, k, prec):
    A = mpgen.random_cmat(17, 1, m, k, prec, 6, zero_frac=0.05)
    B = mpgen.random_cmat(17, 2, k, n, prec, 6, zero_frac=0.05)
    C0, r0 = run_gpu(A, B, prec, method)
    name, _, val = env.partition("=")
    monkeypatch.setenv(name, val or "1")
    C1, r1 = run_gpu(A, B, prec, method)
    monkeypatch.delenv(name)
    assert r0["slices"] == r1["slices"]
    assert same_bits(C0, C1), first_mismatch(C0, C1)


@pytest.mark.parametrize("carrier", [0, 1])
def test_tall_shapes_beyond_grid_y(carrier):
    """m = 70000 > 65535 rows: every launch that once put m in gridDim.y (the fold, the zero-fill for
    k = 0, the binary64 fold) now loops or flattens -- sampled bit-exact vs the oracle."""
    m, n, k, prec = 70000, 3, 2, 64
    A = mpgen.random_cmat(23, 1, m, k, prec, 3)
    B = mpgen.random_cmat(23, 2, k, n, prec, 3)
    dA, dB = P.to_device(A), P.to_device(B)
    dC, rep = P.gemm(dA, dB, prec, "3M", carrier=carrier)
    torch.cuda.synchronize()
    C = P.to_host(dC)
    rng = np.random.default_rng(3)
    si = np.concatenate([rng.integers(0, m, 40), [0, 65535, 65536, m - 1]])
    sj = np.concatenate([rng.integers(0, n, 40), [0, 1, 2, n - 1]])
    if carrier:
        Rs = oracle.ozaki_bits(A, B, prec, "3M", rep["slices"], bits=rep["slice_bits"], samples=(si, sj))
    else:
        Rs = oracle.ozaki(A, B, prec, "3M", rep["slices"], samples=(si, sj))
    assert sampled_equal(C, Rs, si, sj) is None
    A0 = mpgen.random_cmat(23, 3, m, 0, prec)
    B0 = mpgen.random_cmat(23, 4, 0, n, prec)
    dC0, _ = P.gemm(P.to_device(A0), P.to_device(B0), prec, "4M")     # k = 0: C = 0 on every row
    torch.cuda.synchronize()
    C0 = P.to_host(dC0)
    assert not C0.re.limbs.any() and not C0.im.limbs.any() and not C0.re.exp.any()
