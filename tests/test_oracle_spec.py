"""Pins the CPU oracle against every SPEC.md example / invariant on the hot
path and the derived known answers of SURVEY.md Appendix B
(tests/golden/spec_examples.json).  The reference ships no executable tests
(SURVEY.md 4), so these are the golden vectors for this path."""
import json
import os

import numpy as np
import pytest

from paper_2111_11728_b200 import problems as pb

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


# ---------------------------------------------------------------- fem-model
def test_simp_modulus(oracle_mod):
    for rho, e in GOLD["simp_modulus"]["cases"]:
        assert abs(oracle_mod.simp_modulus(rho) - e) <= 1e-15 * max(1.0, e)
    with pytest.raises(oracle_mod.OracleError) as ei:
        oracle_mod.simp_modulus(1.5)
    assert ei.value.code == 21  # std::domain_error (fem.cpp:20-22)


def test_q4_element_stiffness(oracle_mod):
    k = oracle_mod.q4_element_stiffness()
    np.testing.assert_allclose(k[0], GOLD["q4_row0_nu03"]["values"], atol=1e-15)
    assert np.array_equal(k, k.T)                       # bit-exact symmetry (fem.cpp:79-81)
    ev = np.sort(np.linalg.eigvalsh(k))
    assert np.all(np.abs(ev[:3]) <= 1e-12)              # 3 rigid modes
    np.testing.assert_allclose(ev[3:], GOLD["q4_eigs_nu03"]["nonzero"], atol=1e-9)
    t = np.array([1, 0] * 4, float)
    assert np.abs(k @ t).max() <= 1e-12 * np.abs(k).max()
    assert np.array_equal(oracle_mod.q4_element_stiffness(modulus=10.0), 10.0 * k)


def test_traction_lumping(oracle_mod):
    # unit normal traction on an edge of length 2 with 2 elements -> (0.5, 1.0, 0.5)
    p = pb.Problem(1, 1, 2, np.ones((1, 2, 2)), np.zeros(1, np.int32),
                   tractions=[(0, pb.RIGHT, 0, 2, 1.0, 0.0)])
    f = oracle_mod.Oracle(p).loads()[0]
    right = [2 * (iy * 3 + 2) for iy in range(3)]
    np.testing.assert_allclose(f[right], [0.5, 1.0, 0.5])
    assert abs(f.sum() - 2.0) < 1e-12


def test_assembly_nullspace(oracle_mod):
    # K^s R = 0 for a random-density subdomain; 1x1 = element
    p = pb.config4(sx=1, sy=1, n=6)
    o = oracle_mod.Oracle(p)
    R = oracle_mod.rigid_body_modes(6)
    Kn = max(np.abs(o.local_apply(0, np.eye(o.local_dofs)[:, i])).max() for i in range(5))
    for c in range(3):
        assert np.abs(o.local_apply(0, R[:, c])).max() <= 1e-10 * Kn
    p1 = pb.Problem(1, 1, 1, np.ones((1, 1, 1)), np.zeros(1, np.int32))
    o1 = oracle_mod.Oracle(p1)
    K1 = np.stack([o1.local_apply(0, np.eye(8)[:, i]) for i in range(8)], axis=1)
    # element nodes are ccw {(0,0),(1,0),(1,1),(0,1)} (fem.hpp:42-45); mesh ids are row-major
    perm = [0, 1, 2, 3, 6, 7, 4, 5]
    assert np.array_equal(K1, oracle_mod.q4_element_stiffness()[np.ix_(perm, perm)])


def test_rigid_body_modes(oracle_mod):
    R = oracle_mod.rigid_body_modes(4)
    np.testing.assert_array_equal(R[0::2, 0], 1.0)
    np.testing.assert_array_equal(R[1::2, 0], 0.0)
    x = np.tile(np.arange(5.0), 5)
    y = np.repeat(np.arange(5.0), 5)
    np.testing.assert_allclose(R[0::2, 2], -(y - 2.0))
    np.testing.assert_allclose(R[1::2, 2], x - 2.0)


def test_fixing_dofs(oracle_mod):
    for n in GOLD["fixing_dofs"]["n"]:
        assert oracle_mod.select_fixing_dofs(oracle_mod.rigid_body_modes(n)) == [0, 1, 2 * n * (n + 1)]


# -------------------------------------------------------------- core-linalg
def test_cholesky_examples(oracle_mod):
    np.testing.assert_allclose(oracle_mod.cholesky_solve(np.eye(4), [1, 2, 3, 4]), [1, 2, 3, 4])
    np.testing.assert_allclose(oracle_mod.cholesky_solve(np.diag([4.0, 9.0]), [8, 27]), [2, 3])
    M = np.random.default_rng(1).standard_normal((20, 20))
    A = M.T @ M + np.eye(20)
    b = np.random.default_rng(2).standard_normal(20)
    assert rel(oracle_mod.cholesky_solve(A, b), np.linalg.solve(A, b)) < 1e-10
    with pytest.raises(oracle_mod.OracleError) as ei:
        oracle_mod.cholesky_solve(-np.eye(3), [1, 1, 1])
    assert ei.value.code == 1                           # NotPositiveDefinite


def test_pivoted_cholesky_examples(oracle_mod):
    perm, L, r = oracle_mod.pivoted_cholesky(np.eye(3))
    assert r == 3 and list(perm) == [0, 1, 2]
    np.testing.assert_allclose(L, np.eye(3))
    v = np.array([1.0, 2.0, 2.0])
    perm, L, r = oracle_mod.pivoted_cholesky(np.outer(v, v))
    assert r == 1 and perm[0] == 1                      # SPEC.md:50 (ties -> lowest index)
    # duplicated columns: rank 1, reconstruction within 1e-10
    w = np.random.default_rng(3).standard_normal(12)
    F = np.random.default_rng(4).standard_normal((12, 12))
    F = F @ F.T + 12 * np.eye(12)
    W = np.stack([w, w], axis=1)
    D = W.T @ F @ W
    perm, L, r = oracle_mod.pivoted_cholesky(D)
    assert r == 1
    P = np.eye(2)[perm]
    assert rel(L @ L.T, P @ D @ P.T) < 1e-10


@pytest.mark.parametrize("n", [1, 2, 5, 13, 30])
def test_pivoted_cholesky_exact_rank(n, oracle_mod):
    """Q^T D Q with r nonzeros >= 1 -> exact rank, all 1 <= r <= n
    (the shipped linalg.cpp:108-119 fails this)."""
    rng = np.random.default_rng(n)
    Qm, _ = np.linalg.qr(rng.standard_normal((n, n)))
    for r in range(1, n + 1):
        d = np.zeros(n)
        d[:r] = 1.0 + rng.random(r) * 9.0
        A = Qm.T @ np.diag(d) @ Qm
        A = 0.5 * (A + A.T)
        perm, L, rk = oracle_mod.pivoted_cholesky(A)
        assert rk == r, (n, r, rk)
        P = np.eye(n)[perm]
        assert rel(L @ L.T, P @ A @ P.T) < 1e-12


def test_pivoted_cholesky_indefinite(oracle_mod):
    with pytest.raises(oracle_mod.OracleError) as ei:
        oracle_mod.pivoted_cholesky(np.diag([1.0, -1.0]))
    assert ei.value.code == 2                           # IndefiniteInput


def test_compress_orthonormalizes(oracle_mod):
    """Alg. 1 lines 9-12: after compression W^T F W = I."""
    rng = np.random.default_rng(7)
    F = rng.standard_normal((30, 30))
    F = F @ F.T + np.eye(30)
    W = rng.standard_normal((30, 6))
    W[:, 5] = W[:, 0] + W[:, 1]                          # rank deficient block
    D = (F @ W).T @ W
    perm, L, r = oracle_mod.pivoted_cholesky(D, 1e-12)
    assert r == 5
    Wc = oracle_mod.compress(perm, L, r, W)
    assert np.abs(Wc.T @ F @ Wc - np.eye(r)).max() < 1e-8


def test_pseudo_solve(oracle_mod):
    p = pb.config1(sx=2, sy=1, n=4)
    o = oracle_mod.Oracle(p)
    assert o.fixed_dofs() == [0, 1, 2 * 4 * 5]
    y = np.random.default_rng(0).standard_normal(o.local_dofs)
    Ky = o.local_apply(0, y)
    x = o.pseudo_solve(0, Ky)
    assert rel(o.local_apply(0, x), Ky) < 1e-9
    assert np.all(x[o.fixed_dofs()] == 0.0)             # zeros at the fixed DOFs (linalg.cpp:206)
    np.testing.assert_array_equal(o.pseudo_solve(0, np.zeros(o.local_dofs)), 0.0)
    R = oracle_mod.rigid_body_modes(4)
    with pytest.raises(oracle_mod.OracleError) as ei:
        o.pseudo_solve(0, R[:, 2])
    assert ei.value.code == 3


# ------------------------------------------------------------ decomposition
def test_mbb_geometry(oracle_mod):
    """Acceptance 1: 12x8 modules of 30x30 ->
    184,512 subdomain DOFs and > 10,000 interface unknowns for both methods."""
    g = GOLD["mbb_geometry"]
    dens = np.ones((1, 30, 30))
    mt = np.zeros(96, np.int32)
    for method, key in ((0, "tfeti_m"), (1, "fetidp_m")):
        p = pb.Problem(12, 8, 30, dens, mt, method=method, dirichlet=pb.bottom_corner_pins(12, 8, 30),
                       point_loads=[(8 * 30 * 361 + 180, 1, -1.0)])
        o = oracle_mod.Oracle(p)
        assert o.n_sub * o.local_dofs == g["total_dofs"]
        assert o.m == g[key] and o.m + o.n_c > 10000   # FETI-DP: 9,976 dual + 234 primal
        if method == 0:
            assert o.n_iface == g["tfeti_iface"]
        if method == 1:   # 234 corner DOFs minus the 4 pinned (eliminated)
            assert o.n_c == g["fetidp_nc"] - 4


def test_constraint_counts(oracle_mod):
    # 2 subdomains sharing an edge of k nodes -> 2k rows, c = 0
    p = pb.Problem(2, 1, 3, np.ones((1, 3, 3)), np.zeros(2, np.int32))
    o = oracle_mod.Oracle(p)
    r = o.rows()
    assert o.m == 2 * 4 and np.all(r["kind"] == 0) and np.all(r["gap"] == 0)
    # one clamped node -> 2 Dirichlet rows with +1
    p = pb.Problem(1, 1, 2, np.ones((1, 2, 2)), np.zeros(1, np.int32), dirichlet=[(0, 0, 0.0), (0, 1, 0.0)])
    r = oracle_mod.Oracle(p).rows()
    assert list(r["kind"]) == [1, 1]
    # cross point shared by 4 -> 6 pairwise rows per DOF
    p = pb.Problem(2, 2, 2, np.ones((1, 2, 2)), np.zeros(4, np.int32))
    r = oracle_mod.Oracle(p).rows()
    center = 2 * 5 + 2
    assert np.sum(r["mult"] == 4) == 12 and np.sum((r["mult"] == 4) & (r["kind"] == 0)) == 12


def test_corner_counts(oracle_mod):
    for sx, sy, nc in GOLD["corners"]["cases"]:
        p = pb.Problem(sx, sy, 2, np.ones((1, 2, 2)), np.zeros(sx * sy, np.int32), method=1)
        assert oracle_mod.Oracle(p).n_c == nc


def test_config_sizes(oracle_mod):
    s = GOLD["config_sizes"]
    o = oracle_mod.Oracle(pb.config1())
    assert (o.m, o.n_iface) == (s["C1"]["m"], s["C1"]["iface"])
    o = oracle_mod.Oracle(pb.config2())
    assert (o.m, o.n_c) == (s["C2"]["m"], s["C2"]["nc"])


@pytest.mark.parametrize("scaling", [0, 1])
@pytest.mark.parametrize("grid", [(2, 2), (3, 3)])
def test_admissibility(scaling, grid, oracle_mod):
    """Eq. (13) for both scalings on 2x2 and 3x3 partitions to 1e-12 (acceptance 8)."""
    p = pb.config4(sx=grid[0], sy=grid[1], n=4).replace(method=0, scaling=scaling)
    assert oracle_mod.Oracle(p).admissibility_error() <= 1e-12


def test_multiplicity_and_k_scaling_values(oracle_mod):
    p = pb.Problem(2, 2, 2, np.ones((1, 2, 2)), np.zeros(4, np.int32), scaling=0)
    r = oracle_mod.Oracle(p).rows()
    assert set(np.round(r["w_plus"], 15)) == {0.5, 0.25}
    # homogeneous: k-scaling == multiplicity
    rk = oracle_mod.Oracle(p.replace(scaling=1)).rows()
    np.testing.assert_allclose(rk["w_plus"], r["w_plus"], atol=1e-15)
    np.testing.assert_allclose(rk["w_minus"], r["w_minus"], atol=1e-15)


def test_k_scaling_contrast(oracle_mod):
    """K^s = 1, K^r = 1e6 -> W^s = 1e6/(1+1e6): two modules with
    moduli 1 and 1e6 (diagonals scale linearly with the modulus)."""
    dens = np.stack([np.zeros((2, 2)), np.ones((2, 2))])
    p = pb.Problem(2, 1, 2, dens, np.array([0, 1], np.int32), E0=1e6, Emin=1.0, p=1.0, scaling=1)
    r = oracle_mod.Oracle(p).rows()
    mid = r["mult"] == 2
    # plus side is subdomain 0 (soft, K=1x), weight = opposite (stiff) / sum
    np.testing.assert_allclose(r["w_plus"][mid], 1e6 / (1.0 + 1e6), rtol=1e-12)
    np.testing.assert_allclose(r["w_minus"][mid], 1.0 / (1.0 + 1e6), rtol=1e-12)


# ------------------------------------------------- preconditioner / operators
@pytest.mark.parametrize("case", ["tfeti", "fetidp"])
def test_operator_properties(case, oracle_mod):
    p = pb.config3(method=0 if case == "tfeti" else 1, sx=3, sy=2, n=6)
    o = oracle_mod.Oracle(p)
    assert np.all(o.apply_F(np.zeros(o.m)) == 0.0)
    a, b = np.random.default_rng(0).standard_normal((2, o.m))
    Fa, Fb = o.apply_F(a), o.apply_F(b)
    assert abs(b @ Fa - a @ Fb) <= 1e-12 * np.linalg.norm(a) * np.linalg.norm(Fb) * 10
    assert a @ Fa > 0
    z0, Z0 = o.apply_precond(np.zeros(o.m), columns=True)
    assert np.all(z0 == 0) and np.all(Z0 == 0)
    za, Za = o.apply_precond(a, columns=True)
    assert rel(Za.sum(axis=1), za) < 1e-15
    zb = o.apply_precond(b)
    assert abs(b @ za - a @ zb) <= 1e-12 * np.linalg.norm(a) * np.linalg.norm(zb)
    assert a @ za >= 0
    if case == "tfeti":
        d, l0 = o.rhs()
        assert o.coarse_residual(l0) < 1e-10                 # G lambda0 = e
        Pa = o.project(a)
        assert rel(o.project(Pa), Pa) < 1e-12                # P^2 = P


def test_dense_operator_2x2_fetidp(oracle_mod):
    """condensed FETI-DP operator == dense Schur complement of the
    full Eq. (12) block system, built column-wise."""
    p = pb.config2(sx=2, sy=2, n=3).replace(precond=0)
    o = oracle_mod.Oracle(p)
    Fcols = np.stack([o.apply_F(np.eye(o.m)[:, i]) for i in range(o.m)], axis=1)
    assert rel(Fcols, Fcols.T) < 1e-12
    assert np.linalg.eigvalsh(0.5 * (Fcols + Fcols.T)).min() > 0


# ------------------------------------------------------------------ engine
def test_engine_trivial(oracle_mod):
    # zero load -> converged at iteration 0, eps_r(0) = 0
    p = pb.config1(sx=2, sy=1, n=4).replace(tractions=[])
    o = oracle_mod.Oracle(p)
    lam, tr = o.solve()
    assert tr["status"] == 0 and tr["iterations"] == 0 and tr["eps0"] == 0.0
    assert np.abs(o.recover(lam)).max() == 0.0


def test_rrs_single_subdomain_equals_fo(oracle_mod):
    """SPEC.md:441 / acceptance 7: N_s = 1 -> RRS trace == FO-PCG trace within 1e-10."""
    p = pb.config1(sx=1, sy=1, n=6)
    o = oracle_mod.Oracle(p)
    _, t1 = o.solve(directions=1, tol=1e-10)
    _, t2 = o.solve(directions=2, tol=1e-10)
    assert t1["iterations"] == t2["iterations"]
    assert np.abs(t1["eps"] - t2["eps"]).max() <= 1e-10 * t1["eps"][0]


@pytest.mark.parametrize("method", [0, 1])
def test_solutions_match_direct_oracle(method, oracle_mod):
    """Converged solves of every direction strategy match the global direct
    oracle (acceptance 2)."""
    p = pb.config3(method=method, sx=3, sy=2, n=6).replace(Emin=1e-4)
    o = oracle_mod.Oracle(p)
    ud = o.direct()
    for dirs in (0, 1, 2):
        lam, tr = o.solve(tol=1e-10, max_it=2000, directions=dirs)
        assert tr["status"] == 0
        assert rel(o.recover(lam), ud) < 1e-6, dirs
        if method == 0:
            assert o.coarse_residual(lam) < 1e-10


def test_fo_conjugacy_and_deterministic_traces(oracle_mod):
    """repeated runs give identical traces; k-scaling and
    multiplicity traces coincide on homogeneous problems (to rounding: the
    summed cross-point denominator x+x+x+x is not always exactly 4x)."""
    p = pb.config1(sx=3, sy=2, n=6).replace(densities=np.ones((6, 6, 6)), scaling=0)
    o = oracle_mod.Oracle(p)
    _, a = o.solve(directions=1)
    _, b = o.solve(directions=1)
    assert np.array_equal(a["eps"], b["eps"])
    ok = oracle_mod.Oracle(p.replace(scaling=1))
    _, c = ok.solve(directions=1)
    assert len(a["eps"]) == len(c["eps"])
    np.testing.assert_allclose(a["eps"], c["eps"], rtol=1e-10)


def test_golden_fixture_reproduces(oracle_mod):
    """The committed oracle fixture (tests/golden/oracle_small.npz) is
    reproduced bit-for-bit by the current oracle build."""
    g = np.load(os.path.join(HERE, "golden", "oracle_small.npz"))
    o = oracle_mod.Oracle(pb.config1(sx=4, sy=2, n=8))
    X = g["c1s_x"]
    for c in range(2):
        np.testing.assert_array_equal(o.apply_F(X[:, c]), g["c1s_Fx"][:, c])
