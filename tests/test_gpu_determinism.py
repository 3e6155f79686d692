"""Race detector: the whole path is integer arithmetic with one rounding, so repeated calls must give
identical bits.  MPCGEMM_DBG=16 re-folds the previous call's partial planes (the slice GEMM is
skipped), so a fold that reads a ring entry the producer's next TMA / bulk copy is overwriting shows
up as a mismatch.  Round 2 found exactly that (consumers released a ring entry before their last
shared loads had completed; the producer's async-proxy write could overtake them): ~5-10 % of
config-4 folds corrupted a few outputs until the release gained a proxy fence."""
import os

import pytest

import mpgen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2307_06072_b200 as P  # noqa: E402


def _equal(C0, C1):
    return all(torch.equal(getattr(getattr(C0, p), f), getattr(getattr(C1, p), f))
               for p in ("re", "im") for f in ("sign", "exp", "limbs"))


@pytest.mark.parametrize("cfg,reps,env", [(4, 24, {}), (3, 24, {}), (4, 12, {"MPCGEMM_FOLD_BULK": "1"}),
                                          (2, 24, {"MPCGEMM_FOLD_NOUNI1": "1"})])
def test_refold_is_deterministic(cfg, reps, env, monkeypatch):
    c = mpgen.CONFIGS[cfg]
    A, B = mpgen.config_inputs(cfg, seed=0)
    dA, dB = P.to_device(A), P.to_device(B)
    C0 = P.empty_device(c["m"], c["n"], c["prec"])
    P.mpcgemm_ex(dA, dB, C0, c["prec"], "3M")
    monkeypatch.setenv("MPCGEMM_DBG", "16")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    C1 = P.empty_device(c["m"], c["n"], c["prec"])
    bad = 0
    for _ in range(reps):
        P.mpcgemm_ex(dA, dB, C1, c["prec"], "3M")
        torch.cuda.synchronize()
        bad += not _equal(C0, C1)
    assert bad == 0, f"{bad} of {reps} re-folds differ"


def test_repeated_calls_bitwise():
    """Full calls (pre-pass, split, slice GEMM, fold) at config 3, repeated."""
    c = mpgen.CONFIGS[3]
    A, B = mpgen.config_inputs(3, seed=0)
    dA, dB = P.to_device(A), P.to_device(B)
    C0 = P.empty_device(c["m"], c["n"], c["prec"])
    P.mpcgemm_ex(dA, dB, C0, c["prec"], "4M")
    C1 = P.empty_device(c["m"], c["n"], c["prec"])
    for _ in range(6):
        P.mpcgemm_ex(dA, dB, C1, c["prec"], "4M")
        torch.cuda.synchronize()
        assert _equal(C0, C1)
