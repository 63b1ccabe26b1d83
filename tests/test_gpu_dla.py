"""The engine's hand-written FP64 dense algebra (csrc/dla.cuh: DMMA GEMM,
split-K, triangular inverse) against numpy in float64.

These kernels replace cuBLAS on the RRS path (Alg. 1 lines 8-21,
PAPER.md:321-347; PivotedCholesky::compress, proj/src/linalg.cpp:131-138)
and in the FETI-DP coarse factorization.  Tolerance: FP64 products of
length K differ from numpy's (differently ordered) sums by a few ulps times
sqrt(K) relative to |A||B|; 1e-13 relative to the product of the norms is
the bound written here."""
import numpy as np
import pytest

from paper_2111_11728_b200 import engine

pytestmark = pytest.mark.gpu

TOL = 1e-13


def op(X, t):
    return X.T if t else X


def check(got, want, A, B):
    scale = np.linalg.norm(A) * np.linalg.norm(B) + 1e-300
    err = np.abs(got - want).max() / scale
    assert err < TOL, err


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("shape", [(1, 1, 1), (7, 5, 3), (64, 64, 16), (130, 70, 33), (257, 129, 100),
                                   (512, 300, 1000), (40, 1200, 77)])
def test_gemm_all_transposes(ta, tb, shape):
    M, N, K = shape
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.standard_normal((K, M) if ta else (M, K))
    B = rng.standard_normal((N, K) if tb else (K, N))
    C0 = rng.standard_normal((M, N))
    got = engine.dla_gemm(A, B, ta, tb, alpha=-0.75, beta=0.5, C0=C0)
    check(got, -0.75 * op(A, ta) @ op(B, tb) + 0.5 * C0, A, B)
    got0 = engine.dla_gemm(A, B, ta, tb)
    check(got0, op(A, ta) @ op(B, tb), A, B)


@pytest.mark.parametrize("ta,tb", [(False, True), (True, True), (False, False)])
@pytest.mark.parametrize("shape", [(96, 96, 5000), (512, 512, 40000), (300, 17, 9000)])
def test_gemm_splitk_deterministic(ta, tb, shape):
    """split-K: fixed segments summed in order -> same result on every call"""
    M, N, K = shape
    rng = np.random.default_rng(K)
    A = rng.standard_normal((K, M) if ta else (M, K))
    B = rng.standard_normal((N, K) if tb else (K, N))
    g1 = engine.dla_gemm(A, B, ta, tb, flags=256)
    g2 = engine.dla_gemm(A, B, ta, tb, flags=256)
    assert np.array_equal(g1, g2)
    check(g1, op(A, ta) @ op(B, tb), A, B)


def test_gemm_lower_tiles():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((300, 500))
    C0 = np.full((300, 300), 7.0)
    got = engine.dla_gemm(A, A, False, True, beta=0.0, C0=C0, flags=1)
    want = A @ A.T
    low = np.tril(np.ones((300, 300), dtype=bool))
    check(got[low], want[low], A, A)
    assert np.all(got[~low] == 7.0)          # upper triangle untouched


def test_gemm_triangular_operands():
    rng = np.random.default_rng(4)
    n = 333
    L = np.tril(rng.standard_normal((n, n)))
    X = rng.standard_normal((200, n))
    # X L^T (L lower: column c of L^T ends at c) -- the RRS compression
    check(engine.dla_gemm(X, L, False, True, flags=2), X @ L.T, X, L)
    # Y L (L lower: column c of L starts at c)
    Y = rng.standard_normal((150, n))
    check(engine.dla_gemm(Y, L, False, False, flags=4), Y @ L, Y, L)
    # L Z (L lower as the A operand: row r ends at r)
    Z = rng.standard_normal((n, 90))
    check(engine.dla_gemm(L, Z, False, False, flags=8), L @ Z, L, Z)


@pytest.mark.parametrize("n", [1, 5, 64, 65, 200, 640, 2048])
def test_tri_inv(n):
    rng = np.random.default_rng(n)
    # a Cholesky factor of a well-conditioned SPD matrix (what Alg. 1 line 9 produces)
    G = rng.standard_normal((n, n)) / np.sqrt(n)
    L = np.linalg.cholesky(G @ G.T + np.eye(n))
    X = engine.dla_tri_inv(L + np.triu(rng.standard_normal((n, n)), 1))   # upper part must be ignored
    assert np.all(np.triu(X, 1) == 0.0)
    assert np.abs(X @ L - np.eye(n)).max() < 1e-12


def test_gemm_throughput_report():
    """DMMA GEMM rate at the RRS coefficient shapes (reported, not asserted
    beyond sanity): 2048^3 and a 2048 x 2048 x 45056 Gram."""
    peak, _ = engine.fp64_peak()
    for (M, N, K, ta, tb) in ((2048, 2048, 2048, False, False), (2048, 2048, 45056, False, False),
                              (2048, 2048, 2048, True, True), (4096, 4096, 4096, False, True)):
        ms = engine.dla_time_gemm(M, N, K, ta, tb, reps=5)
        tf = 2.0 * M * N * K / (ms * 1e-3) / 1e12
        print(f"gemm {M}x{N}x{K} ta={ta} tb={tb}: {ms:.3f} ms {tf:.1f} TFLOP/s ({tf / peak:.0%} of DMMA peak)")
        assert tf > 0.3 * peak


@pytest.mark.parametrize("name", ["C4s", "C5s", "C2s"])
def test_zblock_apply_matches_dense_block(name):
    """K5z (fresh preconditioner block, 5 local columns per subdomain, coarse
    term dense, rows written once) against the dense K5 block apply and the
    single-vector K4 apply, on the block Alg. 1 lines 2/16 produce."""
    from paper_2111_11728_b200 import problems as pb
    prob = {"C4s": lambda: pb.config4(sx=6, sy=4, n=8),
            "C5s": lambda: pb.config5(sx=5, sy=3, n=12, n_designs=3),
            "C2s": lambda: pb.config2(sx=4, sy=3, n=8)}[name]()
    g = engine.FetiSystem(prob)
    r = np.random.default_rng(2).standard_normal(g.m)
    _, Z = g.apply_precond(r, columns=True)
    Qz = g.apply_F_zblock(Z)
    Qd = g.apply_F_block(Z)
    err = np.abs(Qz - Qd).max() / np.abs(Qd).max()
    print(name, "K5z vs K5", err)
    assert err < 1e-12
    for c in (0, g.n_sub // 2, g.n_sub - 1):
        assert np.abs(Qz[:, c] - g.apply_F(Z[:, c])).max() <= 1e-12 * np.abs(Qd).max()
    g.close()


@pytest.mark.parametrize("name", ["C4s", "C5s", "C2s", "C2_roller_vertex"])
def test_edge_block_apply_bitwise(name, monkeypatch):
    """K5e (block apply by interface edge, FETIGPU_K5_EDGE=1: both owners'
    ranges per tile, the first stored and the second added, no memset or
    atomics) equals K5 bit for bit."""
    from paper_2111_11728_b200 import problems as pb
    prob = {"C4s": lambda: pb.config4(sx=6, sy=4, n=8),
            "C5s": lambda: pb.config5(sx=5, sy=3, n=12, n_designs=3),
            "C2s": lambda: pb.config2(sx=4, sy=3, n=8),
            "C2_roller_vertex": lambda: pb.config2(sx=3, sy=2, n=8).replace(
                dirichlet=[(0, 0, 0.0), (0, 1, 0.0), (3 * 8, 1, 0.0)],
                point_loads=[((2 * 8) * 25 + 12, 1, -1.0)])}[name]()
    g = engine.FetiSystem(prob)
    W = np.random.default_rng(5).standard_normal((g.m, 64))
    monkeypatch.setenv("FETIGPU_K5_EDGE", "0")
    Q0 = g.apply_F_block(W)
    monkeypatch.setenv("FETIGPU_K5_EDGE", "1")
    Q1 = g.apply_F_block(W)
    g.close()
    assert np.array_equal(Q0.view(np.uint64), Q1.view(np.uint64))
