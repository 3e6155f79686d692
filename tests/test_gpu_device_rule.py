"""Device-side slice rule (opts.device_rule): the pre-pass integers are reduced and
the certified s is chosen by a kernel, which
selects one of the host-prepared candidate plans -- no host readback, so the call can be captured
in a CUDA graph.  Checked: the device-chosen s equals oracle.auto_slices on the pre-pass cases
(including the max-plus second stage), C is bitwise the host-rule call's, a CUDA graph of the call
replays to the same bits, and an s outside the planned range leaves C untouched with
MPCGEMM_ERR_SLICES."""
import numpy as np
import pytest

import mpgen
import oracle
from harness import first_mismatch, same_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2307_06072_b200 as P  # noqa: E402


def host_and_device(A, B, prec, method):
    dA, dB = P.to_device(A), P.to_device(B)
    m, n = A.shape[0], B.shape[1]
    C0 = P.empty_device(m, n, prec)
    r0 = P.mpcgemm_ex(dA, dB, C0, prec, method)
    C1 = P.empty_device(m, n, prec)
    r1 = P.mpcgemm_ex(dA, dB, C1, prec, method, device_rule=1)
    st, s, bounds = P.mpcgemm_device_rule_result(m, n)
    return dA, dB, C0, r0, C1, r1, st, s, bounds


@pytest.mark.parametrize("small", ["1", "0"])
@pytest.mark.parametrize("method", ["3M", "4M"])
@pytest.mark.parametrize("spread,k", [(16, 12), (16, 3), (0, 64), (4, 40), (0, 1), (30, 2), (8, 129)])
def test_device_rule_matches_oracle(method, spread, k, small, monkeypatch):
    """small = "1" (default up to m n k = 2^27): T by dp4a + stage 1 in one launch, then stage 2 +
    rule; "0": the T GEMM on tcgen05 + the reduction kernels."""
    monkeypatch.setenv("MPCGEMM_PREPASS_SMALL", small)
    m, n, prec = 70, 90, 256
    A = mpgen.random_cmat(spread + k, 9, m, k, prec, spread, zero_frac=0.1)
    B = mpgen.random_cmat(spread + k, 10, k, n, prec, spread, zero_frac=0.1)
    s_ref, ok = oracle.auto_slices(A, B, prec, method)
    dA, dB, C0, r0, C1, r1, st, s, bounds = host_and_device(A, B, prec, method)
    assert ok and s == s_ref == r0["slices"], (s, s_ref, r0["slices"])
    if st == 0:
        assert bounds == oracle.rho_bounds(A, B)
        H0, H1 = P.to_host(C0), P.to_host(C1)
        assert same_bits(H0, H1), first_mismatch(H0, H1)
    else:                                              # max-plus stage pushed s above the plans
        assert st == -8 and bounds[0] == 0
        assert not C1.re.limbs.any() and not C1.im.limbs.any()     # untouched (zero-initialised)


@pytest.mark.parametrize("spread,k", [(16, 12), (0, 64)])
def test_device_rule_fused_and_separate_launches(spread, k, monkeypatch):
    """Stage 2 + rule in one launch (the last block runs the rule; default) and as two launches
    (MPCGEMM_RULE_SEPARATE): same s, same bounds, same bits -- including the minT == 0 case where
    stage 2 runs, and repeated calls (the fused launch's done counter is re-initialised per call)."""
    m, n, prec, method = 70, 90, 256, "3M"
    A = mpgen.random_cmat(spread + k, 9, m, k, prec, spread, zero_frac=0.1)
    B = mpgen.random_cmat(spread + k, 10, k, n, prec, spread, zero_frac=0.1)
    out = []
    for sep in (False, True, False):
        if sep:
            monkeypatch.setenv("MPCGEMM_RULE_SEPARATE", "1")
        else:
            monkeypatch.delenv("MPCGEMM_RULE_SEPARATE", raising=False)
        dA, dB, C0, r0, C1, r1, st, s, bounds = host_and_device(A, B, prec, method)
        out.append((st, s, bounds, P.to_host(C1) if st == 0 else None))
    for st, s, bounds, H in out[1:]:
        assert (st, s, bounds) == out[0][:3]
        if st == 0:
            assert same_bits(out[0][3], H)


@pytest.mark.parametrize("cfg", [1, 2])
@pytest.mark.parametrize("method", ["3M", "4M"])
def test_device_rule_configs(cfg, method):
    c = mpgen.CONFIGS[cfg]
    A, B = mpgen.config_inputs(cfg, seed=0)
    s_ref, _ = oracle.auto_slices(A, B, c["prec"], method)
    dA, dB, C0, r0, C1, r1, st, s, bounds = host_and_device(A, B, c["prec"], method)
    assert st == 0 and s == s_ref == r0["slices"]
    assert same_bits(P.to_host(C0), P.to_host(C1))


@pytest.mark.parametrize("m,n,k", [(150, 260, 96), (60, 70, 40)])
def test_device_rule_cuda_graph(m, n, k):
    """The device-rule call captured once in a CUDA graph and replayed on new inputs: each replay
    gives the host-rule result bit for bit (s re-derived on the device every replay)."""
    prec, method = 192, "3M"
    A1 = mpgen.random_cmat(3, 1, m, k, prec, 3)
    B1 = mpgen.random_cmat(3, 2, k, n, prec, 3)
    A2 = mpgen.random_cmat(4, 1, m, k, prec, 8)                # other data, other s
    B2 = mpgen.random_cmat(4, 2, k, n, prec, 8)
    dA, dB = P.to_device(A1), P.to_device(B1)
    C = P.empty_device(m, n, prec)
    s1 = oracle.auto_slices(A1, B1, prec, method)[0]
    s2 = oracle.auto_slices(A2, B2, prec, method)[0]
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        for _ in range(2):                                      # warm-up: plans, workspace
            P.mpcgemm_ex(dA, dB, C, prec, method, device_rule=1)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        P.mpcgemm_ex(dA, dB, C, prec, method, device_rule=1)
    for Ah, Bh, s_ref in ((A1, B1, s1), (A2, B2, s2), (A1, B1, s1)):
        src_a, src_b = P.to_device(Ah), P.to_device(Bh)
        for dst, src in ((dA, src_a), (dB, src_b)):
            for p in ("re", "im"):
                for f in ("sign", "exp", "limbs"):
                    getattr(getattr(dst, p), f).copy_(getattr(getattr(src, p), f))
        g.replay()
        torch.cuda.synchronize()
        st, s, _ = P.mpcgemm_device_rule_result(m, n)
        assert st == 0 and s == s_ref
        R = oracle.ozaki(Ah, Bh, prec, method, s_ref)
        assert same_bits(P.to_host(C), R), first_mismatch(P.to_host(C), R)


@pytest.mark.parametrize("method", ["3M", "4M"])
@pytest.mark.parametrize("prec", [368, 384, 400])
def test_device_rule_unit_shape_boundary(method, prec):
    """m = 1024, n = 128 (1-CTA tiles, 8 row tiles): the plan switches from single-diagonal units
    to diagonal pairs at s = 49 (8 tiles x ceil(s/2) x 3 jobs >= 4 x 148 CTAs), inside these
    precisions' candidate ranges.  The device rule builds every candidate with one unit shape (the
    largest candidate's), the host rule with the chosen s's own -- same bits either way."""
    m, n, k = 1024, 128, 64
    A = mpgen.random_cmat(prec, 11, m, k, prec, 2)
    B = mpgen.random_cmat(prec, 12, k, n, prec, 2)
    dA, dB, C0, r0, C1, r1, st, s, bounds = host_and_device(A, B, prec, method)
    assert st == 0 and s == r0["slices"]
    H0, H1 = P.to_host(C0), P.to_host(C1)
    assert same_bits(H0, H1), first_mismatch(H0, H1)


@pytest.mark.parametrize("m,n,k", [(64, 64, 64), (300, 260, 150)])
def test_device_rule_pdl_on_off(m, n, k, monkeypatch):
    """Device-rule calls launch their kernels with programmatic stream serialization (each kernel
    waits in griddepcontrol.wait for its predecessor); MPCGEMM_PDL=0 launches them plainly.  Same
    s, same bits, and both equal the host-rule call."""
    prec, method = 256, "3M"
    A = mpgen.random_cmat(k + 1, 5, m, k, prec, 4)
    B = mpgen.random_cmat(k + 1, 6, k, n, prec, 4)
    out = []
    for pdl in ("1", "0"):
        monkeypatch.setenv("MPCGEMM_PDL", pdl)
        dA, dB, C0, r0, C1, r1, st, s, bounds = host_and_device(A, B, prec, method)
        assert st == 0 and s == r0["slices"]
        H0, H1 = P.to_host(C0), P.to_host(C1)
        assert same_bits(H0, H1), first_mismatch(H0, H1)
        out.append((s, H1))
    assert out[0][0] == out[1][0] and same_bits(out[0][1], out[1][1])
