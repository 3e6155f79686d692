"""GPU parity for NEXT-3: the device MP scalar operations, the blocked
complex LU (mpclu_factor) and the Eq. 7 solve (mpclu_solve), through the C ABI, bit-exact
against the oracle (oracle.cscalar / lu_factor / lu_solve) on the same seeded inputs."""
import math
from fractions import Fraction

import numpy as np
import pytest

import mpgen
import oracle
from harness import first_mismatch, same_bits, to_fraction

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2307_06072_b200 as P  # noqa: E402

from test_oracle_lu import exact_lu_instance, mat_of, rand_fr, row_of  # noqa: E402


def scalar_inputs(prec, spread, cnt, seed):
    import random
    rng = random.Random(seed)
    X = [(rand_fr(rng, prec, spread), rand_fr(rng, prec, spread)) for _ in range(cnt)]
    Y = [(rand_fr(rng, prec, spread), rand_fr(rng, prec, spread)) for _ in range(cnt)]
    A = []
    for t in range(cnt):
        if t % 3 == 0:                                    # a ~ x y: deep cancellation
            (xr, xi), (yr, yi) = X[t], Y[t]
            A.append((xr * yr - xi * yi, xr * yi + xi * yr))
        else:
            A.append((rand_fr(rng, prec, spread), rand_fr(rng, prec, spread)))
    return row_of(X, prec), row_of(Y, prec), row_of(A, prec)


@pytest.mark.parametrize("prec,spread", [(64, 0), (100, 5), (128, 300), (256, 8), (512, 2), (768, 40), (1000, 3),
                                         (1024, 70)])
def test_scalar_ops_bitexact(prec, spread):
    X, Y, A = scalar_inputs(prec, spread, 300, prec + spread)
    dX, dY, dA = P.to_device(X), P.to_device(Y), P.to_device(A)
    for op in ("mul", "fms"):
        G = P.to_host(P.mpc_scalar(op, dX, dY, dA))
        R = oracle.cscalar(op, X, Y, A)
        assert same_bits(G, R), (op, first_mismatch(G, R))
    nz = [t for t in range(X.shape[1]) if X.re.limbs[0, t, -1] or X.im.limbs[0, t, -1]]
    Xn = mpgen.CMat(mpgen.RMat(X.re.sign[:, nz], X.re.exp[:, nz], X.re.limbs[:, nz], prec),
                    mpgen.RMat(X.im.sign[:, nz], X.im.exp[:, nz], X.im.limbs[:, nz], prec))
    Xn = mpgen.CMat(Xn.re.copy(), Xn.im.copy())
    G = P.to_host(P.mpc_scalar("recip", P.to_device(Xn)))
    assert same_bits(G, oracle.cscalar("recip", Xn)), first_mismatch(G, oracle.cscalar("recip", Xn))
    keys = P.mpc_scalar("key", dX).cpu().numpy()
    ok = oracle.cscalar("key", X)
    for t in range(X.shape[1]):
        assert int(keys[t, 0]) == ok[t][0] or ok[t][1] == 0.0
        assert keys[t, 1:2].view(np.float64)[0] == ok[t][1]


def test_recip_gaps_bitexact():
    """re/im exponent gaps on both sides of the device's exact-D / dropped-tail switch
    (prec + 128 L + 4 bits between the squares), powers of two, one-part-zero pivots."""
    for prec in (64, 128, 320):
        L = (prec + 63) // 64
        sw = (prec + 128 * L + 4) // 2
        vals = []
        for g in (0, 1, 63, sw - 2, sw - 1, sw, sw + 1, sw + 3, 3 * sw):
            vals.append((Fraction(1), Fraction(3, 2 ** (g + 2))))
            vals.append((Fraction(-5, 2 ** (g + 3)), Fraction(7, 8)))
            vals.append((Fraction((1 << (prec - 1)) + 1, 1 << (prec - 1)), Fraction(-1, 2 ** g)))
        vals += [(Fraction(1), Fraction(0)), (Fraction(0), Fraction(-2)), (Fraction(2 ** 10), Fraction(2 ** 10))]
        X = row_of(vals, prec)
        G = P.to_host(P.mpc_scalar("recip", P.to_device(X)))
        R = oracle.cscalar("recip", X)
        assert same_bits(G, R), (prec, first_mismatch(G, R))


@pytest.mark.parametrize("prec", [256, 320, 512, 700])
def test_fast_path_window_edges_bitexact(prec):
    """The register fast paths' switches (DESIGN.md NEXT-3): fms/mul with term exponent gaps
    around the 2C + 3-limb window edge (~128 bits), random full mantissas, deep cancellation
    between the products; reciprocals with square-exponent gaps around 120 bits.  Bit-exact
    against the oracle on both sides of every switch."""
    import random
    rng = random.Random(prec)
    m = lambda: rng.getrandbits(prec) | (1 << (prec - 1))
    fr = lambda e, sgn=1: Fraction(sgn * m()) * Fraction(2) ** (e - prec)
    X, Y, A = [], [], []
    for g in list(range(100, 150, 3)) + [60, 64, 126, 127, 128, 129, 130, 192, 200]:
        for case in range(3):
            xr, xi, yr, yi = fr(0), fr(-g // 2), fr(1, -1), fr(-(g - g // 2))
            if case == 0:
                a = (fr(g), fr(-g, -1))                       # a far above the products
            elif case == 1:
                a = (fr(-g), fr(-g - 5))                      # a far below the products
            else:                                             # products cancel each other
                xi, yi = xr, yr
                a = (fr(-g), fr(3))
            X.append((xr, xi)); Y.append((yr, yi)); A.append(a)
    dX, dY, dA = (P.to_device(row_of(v, prec)) for v in (X, Y, A))
    Xh, Yh, Ah = (row_of(v, prec) for v in (X, Y, A))
    for op in ("mul", "fms"):
        G = P.to_host(P.mpc_scalar(op, dX, dY, dA))
        R = oracle.cscalar(op, Xh, Yh, Ah)
        assert same_bits(G, R), (op, first_mismatch(G, R))
    Z = []
    for g in list(range(50, 70)) + [0, 1, 2, 30, 100]:          # square gaps 2 g around 120
        Z.append((fr(0), fr(-g, -1)))
        Z.append((fr(-g), fr(0)))
    Zh = row_of(Z, prec)
    G = P.to_host(P.mpc_scalar("recip", P.to_device(Zh)))
    R = oracle.cscalar("recip", Zh)
    assert same_bits(G, R), first_mismatch(G, R)


@pytest.mark.parametrize("wmax", ["0", "100000"])
def test_thread_and_warp_kernels_agree(monkeypatch, wmax):
    """The LU's scalar kernels for L <= 12 exist twice -- a thread per element part and a warp per
    element part (mpwarp.cuh), chosen by launch size (MPCGEMM_MPWARP_MAX): forcing either gives
    the oracle's bits for the scalar ops and a small factorization."""
    monkeypatch.setenv("MPCGEMM_MPWARP_MAX", wmax)
    for prec, spread in ((256, 8), (512, 40), (200, 300), (768, 20), (700, 250)):
        X, Y, A = scalar_inputs(prec, spread, 120, prec + 3 * spread)
        dX, dY, dA = P.to_device(X), P.to_device(Y), P.to_device(A)
        for op in ("mul", "fms"):
            G = P.to_host(P.mpc_scalar(op, dX, dY, dA))
            R = oracle.cscalar(op, X, Y, A)
            assert same_bits(G, R), (wmax, op, first_mismatch(G, R))
    A = mpgen.random_cmat(77, 51, 40, 40, 256, 2)
    F, ipiv, rep, _ = lu_gpu(A, 8, "3M")
    R, ipiv_r, info_r, _ = oracle.lu_factor(A, 8, "3M")
    assert list(ipiv) == list(ipiv_r) and rep["info"] == info_r
    assert same_bits(F, R), first_mismatch(F, R)


def lu_gpu(A, K, method, adaptive=0):
    dA = P.to_device(A)
    ipiv, rep = P.mpclu_factor(dA, K, method, adaptive=adaptive)
    torch.cuda.synchronize()
    return P.to_host(dA), ipiv.cpu().numpy(), rep, dA


@pytest.mark.parametrize("method", ["3M", "4M"])
@pytest.mark.parametrize("n,K,prec,spread", [(1, 1, 128, 0), (5, 2, 128, 3), (40, 8, 256, 2), (70, 16, 128, 0),
                                             (33, 1, 192, 1), (48, 64, 128, 4), (64, 20, 512, 0)])
def test_lu_factor_bitexact(method, n, K, prec, spread):
    A = mpgen.random_cmat(n + K + prec, 51, n, n, prec, spread)
    F, ipiv, rep, _ = lu_gpu(A, K, method)
    R, ipiv_r, info_r, smax_r = oracle.lu_factor(A, K, method)
    assert list(ipiv) == list(ipiv_r)
    assert rep["info"] == info_r == 0
    assert rep["slices_max"] == smax_r
    assert same_bits(F, R), first_mismatch(F, R)


def test_lu_diagonally_loaded():
    """BASELINE config 5's matrix class (uniform + n on the diagonal): no row swaps."""
    n, K, prec = 96, 32, 256
    A = mpgen.random_cmat(9, 52, n, n, prec, 0)
    for i in range(n):                                      # + n on the diagonal (exact)
        v = to_fraction(A.re, i, i) + n
        from harness import entry_of_rne
        s, e, limbs = entry_of_rne(v, prec, A.re.L)
        A.re.sign[i, i], A.re.exp[i, i] = s, e
        A.re.limbs[i, i, :] = limbs
    F, ipiv, rep, _ = lu_gpu(A, K, "3M")
    R, ipiv_r, _, _ = oracle.lu_factor(A, K, "3M")
    assert list(ipiv) == list(ipiv_r) == list(range(n))
    assert same_bits(F, R), first_mismatch(F, R)


def test_lu_zero_pivot_info_and_exact_closure():
    n, prec = 12, 128
    Lv, Uv, Av = exact_lu_instance(n, 5, prec)
    A = mat_of(Av, prec)
    for K in (1, 4, 12):
        F, ipiv, rep, _ = lu_gpu(A, K, "3M")
        assert rep["info"] == 0 and list(ipiv) == list(range(n))
        want = [[Lv[r][c] if r > c else Uv[r][c] for c in range(n)] for r in range(n)]
        assert same_bits(F, mat_of(want, prec))
    vals = [[(Fraction(r + 2 * c + 1), Fraction(r - c)) if c != 1 else (Fraction(0), Fraction(0)) for c in range(4)]
            for r in range(4)]
    Z = mat_of(vals, 64)
    F, ipiv, rep, _ = lu_gpu(Z, 2, "3M")
    R, ipiv_r, info_r, _ = oracle.lu_factor(Z, 2, "3M")
    assert rep["info"] == info_r == 2
    assert same_bits(F, R) and list(ipiv) == list(ipiv_r)


@pytest.mark.parametrize("n,K,prec,nrhs", [(30, 8, 128, 1), (50, 16, 256, 3)])
def test_lu_solve_bitexact_and_eq7(n, K, prec, nrhs):
    """Eq. 7: x_k = k + k i, b = A x exact, rounded; the GPU solve equals
    the oracle's bitwise and the solution error stays within 2^-(prec-24)."""
    A = mpgen.random_cmat(n + prec, 53, n, n, prec, 0)
    xv = [[(Fraction(k + 1 + q), Fraction(k + 1)) for q in range(nrhs)] for k in range(n)]
    X = mat_of(xv, prec)
    Bm = oracle.exact(A, X, prec, "4M")
    F, ipiv, rep, dF = lu_gpu(A, K, "3M")
    dB = P.to_device(Bm)
    P.mpclu_solve(dF, torch.from_numpy(ipiv).cuda(), dB)
    torch.cuda.synchronize()
    Xg = P.to_host(dB)
    R, ipiv_r, _, _ = oracle.lu_factor(A, K, "3M")
    Xr = oracle.lu_solve(R, ipiv_r, Bm)
    assert same_bits(Xg, Xr), first_mismatch(Xg, Xr)
    err = 0.0
    for k in range(n):
        for q in range(nrhs):
            dr = float(to_fraction(Xg.re, k, q) - xv[k][q][0])
            di = float(to_fraction(Xg.im, k, q) - xv[k][q][1])
            err = max(err, math.hypot(dr, di) / abs(complex(float(xv[k][q][0]), float(xv[k][q][1]))))
    assert err <= 2.0 ** -(prec - 24)


@pytest.mark.parametrize("seed", list(range(int(__import__("os").environ.get("MPCGEMM_FUZZ_LU", "6")))))
def test_fuzz_lu_bitexact(seed):
    """Random (n, K, prec, spread, method): factorization bit-exact against the oracle, both the
    warp (small launches) and the thread (large launches) kernels in play.  MPCGEMM_FUZZ_LU=N."""
    rng = np.random.default_rng(7000 + seed)
    n = int(rng.choice([1, 3, 17, 40, 64, 90]))
    K = int(rng.choice([1, 2, 8, 16, 33, 128]))
    prec = int(rng.choice([64, 128, 200, 256, 512, 700] if n > 40 else [64, 128, 256, 512, 768, 1000]))
    spread = int(rng.choice([0, 3, 30]))
    method = str(rng.choice(["3M", "4M"]))
    A = mpgen.random_cmat(seed, 60, n, n, prec, spread)
    F, ipiv, rep, _ = lu_gpu(A, K, method)
    R, ipiv_r, info_r, smax_r = oracle.lu_factor(A, K, method)
    assert list(ipiv) == list(ipiv_r) and rep["info"] == info_r, (n, K, prec, spread, method)
    assert same_bits(F, R), ((n, K, prec, spread, method), first_mismatch(F, R))
