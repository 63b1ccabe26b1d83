"""GPU parity against the CPU oracle (the reference's implicit algorithm
restated in oracle/): operator applications, preconditioners, projector,
right-hand sides, full solves and primal recovery on identical seeded inputs.

Tolerances (north star, BASELINE.json): iteration count +-1, final relative
dual residual within 1e-6, subdomain displacements within 1e-8 relative L2.

At SIMP contrasts of 1e6-1e9 the local solves are ill-conditioned (cond(K_rr)
~ contrast * h^-2), so two correct FP64 implementations differ by rounding
amplified by the condition number.  Operator-level parity is therefore
measured against an *accuracy reference*: the same oracle with two steps of
iterative refinement on long-double residuals (``fo_set_refine``).  The GPU
must be within ACC_FACTOR x the double-precision oracle's own distance to that
reference (floor 1e-11); at low contrast (C1) both are ~1e-11.  Iteration
counts are required to match +-1 for FO/RRS; single-direction PCG is
roundoff-chaotic (the double oracle and the refined oracle differ by up to
36% on these cases), so there the GPU must stay within the reference's own
roundoff spread (+1)."""
ACC_FACTOR = 10.0

import os

import numpy as np
import pytest

from paper_2111_11728_b200 import problems as pb

pytestmark = pytest.mark.gpu

CASES = {
    "C1": lambda: pb.config1(),
    "C1b": lambda: pb.config1(random_blocks=True, seed=3),
    "C2s": lambda: pb.config2(sx=4, sy=2, n=8),
    "C3tf_s": lambda: pb.config3(method=0, sx=4, sy=2, n=8),
    "C3dp_s": lambda: pb.config3(method=1, sx=4, sy=2, n=8),
    "C5s": lambda: pb.config5(sx=4, sy=2, n=12, n_designs=3),
    "C4s": lambda: pb.config4(sx=4, sy=2, n=8),
    "C1_dir_k": lambda: pb.config1(sx=3, sy=3, n=8).replace(scaling=1, precond=1),
    "C2_lumped": lambda: pb.config2(sx=3, sy=2, n=10).replace(precond=0),
    "C3tf_super": lambda: pb.config3(method=0, sx=3, sy=2, n=8).replace(precond=2),
    # one-direction supports: a roller at a partition vertex gives
    # that subdomain an odd n_c, a roller on an interface edge node an odd n_s
    "C2_roller_vertex": lambda: pb.config2(sx=3, sy=2, n=8).replace(
        dirichlet=[(0, 0, 0.0), (0, 1, 0.0), (3 * 8, 1, 0.0)], point_loads=[((2 * 8) * 25 + 12, 1, -1.0)]),
    "C2_roller_edge": lambda: pb.config2(sx=3, sy=2, n=8).replace(
        dirichlet=pb.left_clamp(3, 2, 8) + [(3 * 25 + 8, 0, 0.0)]),
}



def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


_cache = {}


def systems(name, oracle_mod):
    """(gpu, oracle double, oracle refined) for a case."""
    if name not in _cache:
        from paper_2111_11728_b200 import engine
        prob = CASES[name]()
        L = oracle_mod.lib()
        L.fo_set_refine(0)
        o = oracle_mod.Oracle(prob)
        L.fo_set_refine(1)
        r = oracle_mod.Oracle(prob)
        L.fo_set_refine(0)
        _cache[name] = (engine.FetiSystem(prob), o, r)
    return _cache[name]


def accurate(got, dbl, ref, what):
    eg, ed = rel(got, ref), rel(dbl, ref)
    print(f"{what}: gpu-vs-ref {eg:.2e}  oracle-vs-ref {ed:.2e}")
    assert eg <= max(ACC_FACTOR * ed, 1e-11), (what, eg, ed)


@pytest.mark.parametrize("name", list(CASES))
def test_apply_F(name, oracle_mod):
    g, o, r = systems(name, oracle_mod)
    rng = np.random.default_rng(11)
    X = rng.standard_normal((g.m, 3))
    Yg = g.apply_F(X)
    for c in range(3):
        accurate(Yg[:, c], o.apply_F(X[:, c]), r.apply_F(X[:, c]), f"{name} F col{c}")


@pytest.mark.parametrize("name", list(CASES))
def test_apply_precond(name, oracle_mod):
    g, o, r = systems(name, oracle_mod)
    x = np.random.default_rng(5).standard_normal(g.m)
    zg, Zg = g.apply_precond(x, columns=True)
    zo, Zo = o.apply_precond(x, columns=True)
    zr, Zr = r.apply_precond(x, columns=True)
    accurate(zg, zo, zr, f"{name} precond")
    accurate(Zg, Zo, Zr, f"{name} precond columns")
    assert rel(Zg.sum(axis=1), zg) < 1e-14   # z = Z 1
    # symmetry / PSD of the preconditioner
    y = np.random.default_rng(6).standard_normal(g.m)
    zy = g.apply_precond(y)
    assert abs(y @ zg - x @ zy) <= 1e-12 * np.linalg.norm(x) * np.linalg.norm(zy)
    assert x @ zg >= 0


@pytest.mark.parametrize("name", [n for n in CASES if CASES[n]().method == 0])
def test_project(name, oracle_mod):
    g, o, r = systems(name, oracle_mod)
    v = np.random.default_rng(7).standard_normal(g.m)
    pg = g.project(v)
    assert rel(pg, o.project(v)) < 1e-11
    assert rel(g.project(pg), pg) < 1e-12      # P^2 = P


@pytest.mark.parametrize("name", list(CASES))
def test_rhs(name, oracle_mod):
    g, o, r = systems(name, oracle_mod)
    dg, lg = g.rhs()
    do, lo = o.rhs()
    dr, lr = r.rhs()
    accurate(dg, do, dr, f"{name} d")
    if np.linalg.norm(lo) > 0:
        assert rel(lg, lo) < 1e-11


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("directions", [0, 1, 2])
def test_solve(name, directions, oracle_mod):
    g, o, r = systems(name, oracle_mod)
    kw = dict(tol=1e-6, max_it=400, directions=directions)
    lg, tg = g.solve(**kw)
    lo, to = o.solve(**kw)
    try:
        lr, tr = r.solve(**kw)
    except oracle_mod.OracleError as e:
        # the refined diagnostic run may hit the contract's IndefiniteInput
        # on a roundoff-level Delta pivot; compare to the
        # double-precision oracle only
        assert e.code == 2 and directions == 2
        tr = to
    print(name, directions, "iters gpu", tg["iterations"], "oracle", to["iterations"],
          "refined", tr["iterations"])
    assert tg["status"] == to["status"] == tr["status"]
    if directions == 0:
        spread = abs(to["iterations"] - tr["iterations"])
        dev = min(abs(tg["iterations"] - to["iterations"]), abs(tg["iterations"] - tr["iterations"]))
        assert dev <= spread + 1
    else:
        assert abs(tg["iterations"] - to["iterations"]) <= 1
        assert abs(tg["iterations"] - tr["iterations"]) <= 1
    if to["status"] == 0:
        assert tg["eps_final"] / tg["eps0"] <= 1e-6
        # ||d - F lambda|| projected residual, measured by the oracle itself
        d, _ = o.rhs()
        res = o.project(d - o.apply_F(lg))
        res_o = o.project(d - o.apply_F(lo))
        assert np.linalg.norm(res) <= 10 * np.linalg.norm(res_o) + 1e-14
    if directions == 2:
        np.testing.assert_array_equal(tg["kept"], to["kept"])


@pytest.mark.parametrize("name", ["C2s", "C3dp_s", "C5s", "C4s", "C2_lumped"])
def test_solve_rrs_implicit_store(name, oracle_mod):
    """FETI-DP RRS with the implicit direction store (W_j as coefficients over
    the packed preconditioner blocks, Q_j never stored; solve_rrs.cuh) against
    the oracle's dense-store Alg. 1: same status, iterations +-1, identical
    kept-direction counts, residual and displacements as close as the
    explicit store's."""
    g, o, r = systems(name, oracle_mod)
    kw = dict(tol=1e-6, max_it=60, directions=2)
    g.set_rrs_store("explicit")
    le, te = g.solve(**kw)
    g.set_rrs_store("implicit")
    try:
        li, ti = g.solve(**kw)
    finally:
        g.set_rrs_store("auto")
    lo, to = o.solve(**kw)
    print(name, "iters implicit", ti["iterations"], "explicit", te["iterations"], "oracle", to["iterations"])
    assert ti["status"] == to["status"] == 0
    assert abs(ti["iterations"] - to["iterations"]) <= 1
    np.testing.assert_array_equal(ti["kept"], to["kept"])
    assert ti["f_applies"] > te["f_applies"]           # three block applies per iteration
    d, _ = o.rhs()
    res_i = np.linalg.norm(d - o.apply_F(li))
    res_o = np.linalg.norm(d - o.apply_F(lo))
    assert res_i <= 10 * res_o + 1e-14
    ui, ue, uo = g.recover(li), g.recover(le), o.recover(lo)
    assert rel(ui, uo) <= 10 * rel(ue, uo) + 1e-12


def test_rrs_store_modes(oracle_mod):
    """The implicit store is FETI-DP only; unknown modes are rejected."""
    from paper_2111_11728_b200 import engine
    g, _, _ = systems("C3tf_s", oracle_mod)
    with pytest.raises(engine.ConfigError):
        g.set_rrs_store("implicit")
    with pytest.raises(KeyError):
        g.set_rrs_store("bogus")
    g.set_rrs_store("explicit")
    g.set_rrs_store("auto")


@pytest.mark.parametrize("name", list(CASES))
def test_recover(name, oracle_mod):
    g, o, r = systems(name, oracle_mod)
    lo, to = o.solve(tol=1e-6, max_it=400, directions=1)
    accurate(g.recover(lo), o.recover(lo), r.recover(lo), f"{name} u(lambda)")


@pytest.mark.parametrize("name", ["C1", "C1b", "C2s", "C3tf_s", "C3dp_s", "C5s", "C4s"])
def test_displacements_tight(name, oracle_mod):
    """Converged displacements: GPU vs oracle within 1e-8 relative L2 when the
    oracle's own accuracy allows it, and both against the global direct
    oracle."""
    g, o, r = systems(name, oracle_mod)
    lg, tg = g.solve(tol=1e-10, max_it=2000, directions=1)
    lo, to = o.solve(tol=1e-10, max_it=2000, directions=1)
    lr, tr = r.solve(tol=1e-10, max_it=2000, directions=1)
    assert tg["status"] == 0 and to["status"] == 0
    ug, uo, ur = g.recover(lg), o.recover(lo), r.recover(lr)
    print(name, "u gpu-vs-oracle %.2e oracle-vs-ref %.2e gpu-vs-ref %.2e" % (
        rel(ug, uo), rel(uo, ur), rel(ug, ur)))
    assert rel(ug, ur) <= max(1e-8, ACC_FACTOR * rel(uo, ur))
    if rel(uo, ur) < 1e-9:
        assert rel(ug, uo) < 1e-8
    ud = o.direct()
    assert rel(ug, ud) <= max(1e-6, 2 * rel(uo, ud))


def test_dense_operator_C1(oracle_mod):
    g, o, r = systems("C1", oracle_mod)
    E = np.eye(g.m)
    Fg = g.apply_F(E)
    Fo = np.stack([o.apply_F(E[:, i]) for i in range(g.m)], axis=1)
    assert rel(Fg, Fo) < 1e-10
    assert rel(Fg, Fg.T) < 1e-13          # symmetry
    assert np.linalg.eigvalsh(0.5 * (Fg + Fg.T)).min() > -1e-10 * np.abs(Fg).max()


def test_dmma_fragment_layout():
    from paper_2111_11728_b200 import engine
    rng = np.random.default_rng(0)
    A, B = rng.standard_normal((8, 4)), rng.standard_normal((4, 8))
    Cm = engine.dmma_selftest(A, B)
    assert np.abs(Cm - A @ B).max() < 1e-14


def test_fp64_peak_reported():
    from paper_2111_11728_b200 import engine
    dmma, dfma = engine.fp64_peak()
    print("FP64 peak TFLOP/s: DMMA %.1f DFMA %.1f" % (dmma, dfma))
    assert dmma > 1.0 and dfma > 1.0


@pytest.mark.parametrize("name", ["C1", "C1b", "C2s", "C3tf_s", "C3dp_s", "C5s", "C4s", "C1_dir_k",
                                  "C2_roller_vertex", "C2_roller_edge"])
@pytest.mark.parametrize("k", [1, 7, 64, 130])
def test_block_apply(name, k, oracle_mod):
    """K5 (DMMA block apply, fused gather/scatter) against the per-column GEMV
    apply and the oracle."""
    g, o, r = systems(name, oracle_mod)
    W = np.random.default_rng(k).standard_normal((g.m, k))
    Qb = g.apply_F_block(W)
    Qc = g.apply_F(W)
    for c in sorted({0, k // 2, k - 1}):
        accurate(Qb[:, c], o.apply_F(W[:, c]), r.apply_F(W[:, c]), f"{name} block col{c}")
    assert rel(Qb, Qc) <= max(1e-12, 10 * rel(o.apply_F(W[:, 0]), r.apply_F(W[:, 0])))


@pytest.mark.parametrize("name", ["C1", "C1b", "C2s", "C3tf_s", "C3dp_s", "C4s"])
def test_symmetric_packed_apply(name, oracle_mod, monkeypatch):
    """The symmetric-packed F_s GEMV (lower block-triangle tiles, used by
    default when subdomains are plentiful) against the full-matrix kernel and
    the oracle; forced on here for small cases."""
    from paper_2111_11728_b200 import engine
    g, o, r = systems(name, oracle_mod)
    monkeypatch.setenv("FETIGPU_FORCE_SYM", "1")
    gs = engine.FetiSystem(CASES[name]())
    monkeypatch.delenv("FETIGPU_FORCE_SYM")
    st = gs.stats()
    assert st["main_kernel_bytes"] > 0
    X = np.random.default_rng(21).standard_normal((g.m, 2))
    Ys, Yf = gs.apply_F(X), g.apply_F(X)
    for c in range(2):
        accurate(Ys[:, c], o.apply_F(X[:, c]), r.apply_F(X[:, c]), f"{name} sym col{c}")
    assert rel(Ys, Yf) <= max(1e-12, 10 * rel(o.apply_F(X[:, 0]), r.apply_F(X[:, 0])))
    # deterministic: repeated applies are bit-identical
    assert np.array_equal(gs.apply_F(X[:, 0]), Ys[:, 0])
    lg, tg = gs.solve(tol=1e-6, max_it=400, directions=1)
    lo, to = o.solve(tol=1e-6, max_it=400, directions=1)
    assert abs(tg["iterations"] - to["iterations"]) <= 1
    gs.close()


SYM_TMA_CASES = dict(CASES)
SYM_TMA_CASES.update({
    # many small subdomains: one or three tiles each, so the ring runs several
    # subdomains ahead of the CTA's consumer warps
    "C4_tiny": lambda: pb.config4(sx=24, sy=20, n=2),
    "C1_tiny": lambda: pb.config1(sx=20, sy=16, n=3),
    # more subdomains than the persistent grid holds (2 CTAs per SM): every
    # CTA walks several subdomains
    "C4_many": lambda: pb.config4(sx=28, sy=24, n=6),
})


@pytest.mark.parametrize("flags", [None, "1"])
@pytest.mark.parametrize("ring", [None, "2", "1"])
@pytest.mark.parametrize("name", ["C1", "C2s", "C3tf_s", "C3dp_s", "C5s", "C4s", "C4_tiny", "C1_tiny", "C4_many"])
def test_symmetric_packed_tma_vs_ldg(name, ring, flags, monkeypatch):
    """k_sym_gemv_tma (operator tiles moved by cp.async.bulk into per-warp
    mbarrier rings, persistent grid, prefetch across subdomain boundaries,
    next x_s gathered inside the tile loop) against the LDG kernel it
    replaces -- with two CTAs per SM and one slot per warp (default), and with
    one CTA per SM and two or one slots.  FETIGPU_SYM_FLAGS=1: the same
    arithmetic everywhere, so F, the preconditioner and the host-buffer apply
    must be bit-identical.  Default: FETI-DP's coarse pre-pass t_s = A''^T x_s
    is streamed through the rings too and summed chunk-wise, so F agrees to
    rounding (1e-13 of |y|); the preconditioner and T-FETI stay bit-identical."""
    from paper_2111_11728_b200 import engine
    prob = SYM_TMA_CASES[name]()
    monkeypatch.setenv("FETIGPU_FORCE_SYM", "1")
    if ring:
        monkeypatch.setenv("FETIGPU_SYM_CTAS", "1")
        monkeypatch.setenv("FETIGPU_SYM_RING", ring)
    if flags:
        monkeypatch.setenv("FETIGPU_SYM_FLAGS", flags)
    gt = engine.FetiSystem(prob)
    monkeypatch.setenv("FETIGPU_SYM_TMA", "0")
    gl = engine.FetiSystem(prob)
    for k in ("FETIGPU_FORCE_SYM", "FETIGPU_SYM_TMA", "FETIGPU_SYM_CTAS", "FETIGPU_SYM_RING", "FETIGPU_SYM_FLAGS"):
        monkeypatch.delenv(k, raising=False)
    assert gt.stats()["apply_kernel"] == 2 and gl.stats()["apply_kernel"] == 1
    exact = flags == "1" or prob.method == 0

    def same(a, b, what):
        if exact:
            assert np.array_equal(a, b), what
        else:
            assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(b), what

    X = np.random.default_rng(33).standard_normal((gt.m, 3))
    for c in range(3):
        same(gt.apply_F(X[:, c]), gl.apply_F(X[:, c]), f"{name} F col {c}")
        assert np.array_equal(gt.apply_precond(X[:, c]), gl.apply_precond(X[:, c])), f"{name} M col {c}"
    same(gt.apply_F(X), gl.apply_F(X), f"{name} F block")
    y0 = gt.apply_F(X[:, 0])
    for _ in range(3):                       # deterministic
        assert np.array_equal(gt.apply_F(X[:, 0]), y0)
    lt, tt = gt.solve(tol=1e-6, max_it=300, directions=1)
    ll, tl = gl.solve(tol=1e-6, max_it=300, directions=1)
    if exact:
        assert tt["iterations"] == tl["iterations"] and np.array_equal(lt, ll)
    else:
        assert abs(tt["iterations"] - tl["iterations"]) <= 1
    gt.close()
    gl.close()


@pytest.mark.parametrize("name", ["C1", "C2s", "C3tf_s", "C3dp_s", "C5s", "C4s"])
def test_recovered_interface_jump(name, oracle_mod):
    """after convergence at eps 1e-8 the recovered
    displacements satisfy B u = c to 1e-6 relative (T-FETI rows incl.
    Dirichlet gaps; FETI-DP: every pair row, plus corners and supports by
    construction), and the copies of every shared global DOF agree.  At
    contrast 1e9 (void E = 1e-9, displacements ~1e9) the bound is 1e-5."""
    g, o, r = systems(name, oracle_mod)
    bound = 1e-5 if g.prob.E0 / g.prob.Emin >= 1e8 and g.prob.densities.min() == 0.0 else 1e-6
    lam, tr = g.solve(tol=1e-8, max_it=2000, directions=1)
    assert tr["status"] == 0
    u = g.recover(lam)
    rows = g.rows()
    jump = np.where(rows["kind"] == 0,
                    u[rows["sub_plus"], rows["dof_plus"]] - u[rows["sub_minus"], rows["dof_minus"]],
                    u[rows["sub_plus"], rows["dof_plus"]] - rows["gap"])
    assert np.linalg.norm(jump) <= bound * np.linalg.norm(u)
    # all owner copies of each global node agree (covers FETI-DP corners)
    p = g.prob
    n, gx = p.n, p.gx_nodes
    vals = {}
    for s in range(p.n_sub):
        si, sj = s % p.sx, s // p.sx
        for iy in (0, n):
            for ix in range(n + 1):
                key = ((sj * n + iy) * gx + si * n + ix)
                vals.setdefault(key, []).append(u[s, 2 * (iy * (n + 1) + ix):2 * (iy * (n + 1) + ix) + 2])
        for ix in (0, n):
            for iy in range(n + 1):
                key = ((sj * n + iy) * gx + si * n + ix)
                vals.setdefault(key, []).append(u[s, 2 * (iy * (n + 1) + ix):2 * (iy * (n + 1) + ix) + 2])
    spread = max(np.abs(np.array(v) - v[0]).max() for v in vals.values())
    assert spread <= bound * np.abs(u).max()


@pytest.mark.parametrize("preset", ["laminated_beam", "grid3x3_layered", "grid4x4_inclusion"])
def test_twelve_variant_grid(preset, oracle_mod, tmp_path):
    """The paper's 12-variant protocol on the desk-scale
    academic presets: GPU vs oracle iteration counts, FO/RRS exact to +-1,
    single direction within 10% (roundoff-chaotic, see module docstring)."""
    import subprocess, sys, csv as _csv
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / preset
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "run_grid.py"), "--problem", preset,
                        "--out", str(out), "--oracle"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    rows = list(_csv.DictReader(open(out / "summary.csv")))
    assert len(rows) == 12
    for row in rows:
        gi, oi = int(row["iterations"]), int(row["oracle_iterations"])
        assert row["status"] == row["oracle_status"], row
        tol = 1 if not row["variant"].endswith("single") else max(1, int(0.1 * oi))
        assert abs(gi - oi) <= tol, row
    header = open(out / "tfeti_k_rrs.csv").readline().strip()
    assert header == "iter,eps_r,kept_dirs,F_applies,cum_local_solves"


def test_modular_simp_loop(oracle_mod):
    """a few modular SIMP/OC iterations driven by the GPU
    solver: compliance equals f^T u of the state solve,
    decreases over the run, and the volume constraint holds."""
    from paper_2111_11728_b200 import simp
    n, sx, sy = 8, 6, 2
    types = np.array([0, 1, 2, 2, 1, 0] * 2, np.int32)          # mirror-symmetric module layout
    gxn = sx * n + 1
    prob = pb.Problem(sx, sy, n, np.full((3, n, n), 0.5), types, method=pb.FETIDP, scaling=pb.KSCALING,
                      precond=pb.DIRICHLET, Emin=1e-9, dirichlet=pb.bottom_corner_pins(sx, sy, n),
                      point_loads=[((sy * n) * gxn + (sx * n) // 2, 1, -1.0)])
    st = simp.optimize(prob, iterations=8, volfrac=0.5, directions=2)
    c = st.compliance
    assert all(s["status"] == 0 for s in st.solves)
    assert c[-1] < c[0]
    assert abs(st.volume[-1] - 0.5) < 1e-4
    # compliance of the first (uniform) design against the oracle's f^T u
    o = oracle_mod.Oracle(prob.replace(densities=np.full((3, n, n), 0.5)))
    lo, to = o.solve(tol=1e-10, max_it=1000, directions=1)
    fu = float((o.loads() * o.recover(lo)).sum())
    assert abs(c[0] - fu) <= 1e-5 * abs(fu)


def test_floating_tfeti_rank_deficient_coarse(oracle_mod):
    """No supports, self-equilibrated load: G G^T has rank 3N_s - 3 and the
    rank-revealing filter keeps 9 of 12 rows; the GPU solve
    matches the oracle and the displacements agree up to rigid motion."""
    from paper_2111_11728_b200 import engine
    p = pb.config1(sx=2, sy=2, n=4).replace(dirichlet=[], tractions=[(1, pb.RIGHT, 0, 4, 1.0, 0.0),
                                                                        (0, pb.LEFT, 0, 4, -1.0, 0.0)])
    g, o = engine.FetiSystem(p), oracle_mod.Oracle(p)
    assert g.stats()["n_kept"] == o.n_kept == 9
    lg, tg = g.solve(tol=1e-10, directions=1)
    lo, to = o.solve(tol=1e-10, directions=1)
    assert tg["status"] == to["status"] == 0 and abs(tg["iterations"] - to["iterations"]) <= 1
    # same multipliers on range(P)
    assert np.linalg.norm(g.project(lg - lo)) < 1e-8 * np.linalg.norm(lo)


@pytest.mark.gpu
@pytest.mark.parametrize("n,deficit", [(1, 0), (5, 0), (32, 3), (96, 7), (160, 0), (161, 3), (300, 20),
                                       (512, 0), (640, 11), (700, 5), (1024, 0), (2048, 40)])
def test_pivoted_cholesky_device(n, deficit, oracle_mod):
    """fetigpu_pivoted_cholesky (linalg.hpp:80) vs the oracle on
    graded PSD Gram matrices of rank n - deficit.  Covers the cluster kernel
    at every cluster size (1..16 CTAs, n <= 640) and the cooperative-grid
    kernel above.  Rank and pivot order must be identical; L agrees to
    rounding (the device contracts a*b+c into FMA, the oracle does not)."""
    from paper_2111_11728_b200 import engine
    rng = np.random.default_rng(1000 + n)
    r = n - deficit
    X = rng.standard_normal((n, r)) * np.logspace(0, -3, r)
    A = X @ X.T
    pg, Lg, rg = engine.pivoted_cholesky(A)
    po, Lo, ro = oracle_mod.pivoted_cholesky(A)
    assert rg == ro == r
    assert np.array_equal(pg, po)
    assert np.linalg.norm(Lg - Lo) <= 1e-9 * np.linalg.norm(Lo)
    Ap = A[np.ix_(pg, pg)]
    assert np.linalg.norm(Ap[:, :r] - (Lg @ Lg[:r].T)) <= 1e-13 * n * np.linalg.norm(A)
    # compression W N^T [L~^{-T}; 0] (PivotedCholesky::compress) vs the oracle's
    W = rng.standard_normal((257, n))
    cg = engine.compress(pg, Lg, rg, W)
    co = oracle_mod.compress(po, Lo, ro, W)
    assert cg.shape == co.shape == (257, r)
    # W L~^{-T} amplifies the rounding difference of L by cond(L~) ~ 1e3 here
    assert np.linalg.norm(cg - co) <= 1e-6 * np.linalg.norm(co)


@pytest.mark.gpu
@pytest.mark.parametrize("n,deficit", [(700, 5), (1500, 0), (2048, 300)])
def test_pivoted_cholesky_blocked_bitwise(n, deficit):
    """The blocked panel / trailing pivoted Cholesky (n > 640) reorganises the
    right-looking k_pivchol_coop1 without changing any per-entry operation:
    rank, permutation and L are identical bit for bit (one process per
    variant: FETIGPU_PIVCHOL_BLOCKED is read once)."""
    import subprocess
    import sys
    code = ("import sys, hashlib, numpy as np; sys.path.insert(0, %r);"
            "from paper_2111_11728_b200 import engine;"
            "rng = np.random.default_rng(%d); X = rng.standard_normal((%d, %d)) * np.logspace(0, -3, %d);"
            "A = X @ X.T; p, L, r = engine.pivoted_cholesky(A);"
            "print(r, hashlib.sha1(p.tobytes() + L.tobytes()).hexdigest())"
            % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), n, n, n - deficit, n - deficit))
    out = {}
    for v in ("0", "1"):
        env = dict(os.environ, FETIGPU_PIVCHOL_BLOCKED=v)
        out[v] = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                                check=True).stdout.split()
    assert int(out["1"][0]) == n - deficit
    assert out["0"] == out["1"]


@pytest.mark.parametrize("n,deficit", [(48, 0), (300, 17), (512, 0), (640, 40)])
def test_pivoted_cholesky_cluster_one_barrier_bitwise(n, deficit):
    """k_pivchol_cl1 (one cluster barrier per pivot, rows in original order,
    replicated diagonal and position map) against k_pivchol_cl (physical
    swaps, three barriers): rank, permutation and L bit for bit (one process
    per variant: FETIGPU_PIVCHOL_CL1 is read once)."""
    import subprocess
    import sys
    code = ("import sys, hashlib, numpy as np; sys.path.insert(0, %r);"
            "from paper_2111_11728_b200 import engine;"
            "rng = np.random.default_rng(%d); X = rng.standard_normal((%d, %d)) * np.logspace(0, -3, %d);"
            "A = X @ X.T; p, L, r = engine.pivoted_cholesky(A);"
            "print(r, hashlib.sha1(p.tobytes() + L.tobytes()).hexdigest())"
            % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), n, n, n - deficit, n - deficit))
    out = {}
    for v in ("0", "1"):
        env = dict(os.environ, FETIGPU_PIVCHOL_CL1=v)
        out[v] = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                                check=True).stdout.split()
    assert int(out["1"][0]) == n - deficit
    assert out["0"] == out["1"]


@pytest.mark.gpu
def test_pivoted_cholesky_device_edge_cases(oracle_mod):
    from paper_2111_11728_b200 import engine
    # negative remaining diagonal -> IndefiniteInput, like the oracle (code 2)
    with pytest.raises(engine.IndefiniteInput):
        engine.pivoted_cholesky(np.diag([1.0, -1.0]))
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.pivoted_cholesky(np.diag([1.0, -1.0]))
    # all-zero matrix: rank 0, identity permutation
    p, L, r = engine.pivoted_cholesky(np.zeros((4, 4)))
    assert r == 0 and list(p) == [0, 1, 2, 3] and L.shape == (4, 0)
    # ties -> lowest index
    p, L, r = engine.pivoted_cholesky(np.eye(3) * 2.0)
    assert r == 3 and list(p) == [0, 1, 2]
    assert np.allclose(L, np.sqrt(2.0) * np.eye(3))


def test_host_pipelined_apply(oracle_mod, monkeypatch):
    """fetigpu_apply_F on host buffers overlaps the H2D copy of lambda with
    the phase-1 GEMV (row-prefix chunks on separate streams, FETI-DP on the
    symmetric path).  Same kernels per subdomain and the same phase-2 order as
    the device path, so the result must be bit-identical to it, and match the
    oracle."""
    from paper_2111_11728_b200 import engine
    import ctypes as C
    prob = pb.config4(sx=8, sy=4, n=8)
    monkeypatch.setenv("FETIGPU_FORCE_SYM", "1")
    g = engine.FetiSystem(prob)
    monkeypatch.delenv("FETIGPU_FORCE_SYM")
    assert g.stats()["host_pipeline"] == 1
    m = g.m
    x = np.random.default_rng(5).standard_normal(m)
    y_host = g.apply_F(x)                                  # pipelined host path
    L = engine.lib()
    dx, dy = C.c_void_p(), C.c_void_p()
    engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m), C.byref(dx)))
    engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m), C.byref(dy)))
    engine.check(L.fetigpu_memcpy(g.h, dx, x.ctypes.data_as(C.c_void_p), C.c_size_t(8 * m), 1))
    engine.check(L.fetigpu_apply_F_device(g.h, C.cast(dx, C.POINTER(C.c_double)),
                                          C.cast(dy, C.POINTER(C.c_double)), 1, m))
    y_dev = np.zeros(m)
    engine.check(L.fetigpu_memcpy(g.h, y_dev.ctypes.data_as(C.c_void_p), dy, C.c_size_t(8 * m), 2))
    engine.check(L.fetigpu_synchronize(g.h))
    L.fetigpu_device_free(g.h, dx)
    L.fetigpu_device_free(g.h, dy)
    assert np.array_equal(y_host, y_dev)
    for _ in range(3):                                     # repeated, back to back
        assert np.array_equal(g.apply_F(x), y_host)
    # FETIGPU_PIPE_FLAG=1: ONE persistent phase-1 kernel gated on the landed row
    # prefix of lambda instead of a kernel per chunk and stream
    monkeypatch.setenv("FETIGPU_PIPE_FLAG", "1")
    for _ in range(2):
        assert np.array_equal(g.apply_F(x), y_host)
    monkeypatch.delenv("FETIGPU_PIPE_FLAG")
    x2 = np.random.default_rng(6).standard_normal(m)
    y2 = g.apply_F(x2)
    assert np.array_equal(g.apply_F(x), y_host) and np.array_equal(g.apply_F(x2), y2)
    o = oracle_mod.Oracle(prob)
    assert rel(y_host, o.apply_F(x)) <= 1e-8
    g.close()


def test_concurrent_contexts_from_two_threads():
    """SURVEY 8b threading contract: a context owns its stream, distinct
    contexts may be driven from different host threads, and results do not
    depend on concurrency (fixed reduction orders).  Two FO solves and two
    applies run at the same time from two threads must be bit-identical to
    the same calls made one after the other."""
    import threading
    from paper_2111_11728_b200 import engine
    probs = [CASES["C2s"](), CASES["C3tf_s"]()]
    sys_ = [engine.FetiSystem(p) for p in probs]
    xs = [np.random.default_rng(40 + i).standard_normal(g.m) for i, g in enumerate(sys_)]
    ref = [(g.solve(tol=1e-8, max_it=500, directions=1)[0], g.apply_F(x)) for g, x in zip(sys_, xs)]
    out = [None, None]

    def work(i):
        g, x = sys_[i], xs[i]
        res = []
        for _ in range(3):
            res.append((g.solve(tol=1e-8, max_it=500, directions=1)[0], g.apply_F(x)))
        out[i] = res

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in range(2):
        for lam, y in out[i]:
            assert np.array_equal(lam, ref[i][0])
            assert np.array_equal(y, ref[i][1])
    for g in sys_:
        g.close()


def test_rrs_store_cache_owned_by_context():
    """The RRS direction store is recycled through a per-context block cache:
    a second solve on the same context reuses the chunks (same results), and
    destroying the context returns them to the driver."""
    from paper_2111_11728_b200 import engine
    before = engine.device_memory()
    g = engine.FetiSystem(pb.config5(sx=16, sy=8))     # m ~ 22k, k = 128: store chunks of ~100 MB
    g.set_rrs_store("explicit")                        # auto would pick the implicit store (m > 32 k)
    assert engine.device_memory(g)["cached"] == 0
    lam, tr = g.solve(tol=1e-6, max_it=100, directions=2)
    assert tr["status"] == 0
    held = engine.device_memory(g)["cached"]
    assert held > 0                                    # the solve's chunks went to the cache
    lam2, _ = g.solve(tol=1e-6, max_it=100, directions=2)
    assert np.array_equal(lam, lam2)
    assert engine.device_memory(g)["cached"] == held   # reused, not grown
    g.close()
    after = engine.device_memory()
    assert after["cached"] == 0
    assert after["free"] >= before["free"] - (64 << 20)


def test_rrs_implicit_store_deterministic():
    """Two implicit-store RRS solves on one context are bitwise identical (the
    packed scatter sums each row's two owner contributions in a zeroed buffer),
    use no cached direction chunks, and leave no device memory behind."""
    from paper_2111_11728_b200 import engine
    before = engine.device_memory()
    g = engine.FetiSystem(pb.config5(sx=16, sy=8))
    g.set_rrs_store("implicit")
    lam, tr = g.solve(tol=1e-6, max_it=100, directions=2)
    lam2, tr2 = g.solve(tol=1e-6, max_it=100, directions=2)
    assert tr["status"] == 0 and tr["iterations"] == tr2["iterations"]
    assert np.array_equal(lam, lam2)
    assert engine.device_memory(g)["cached"] == 0
    g.close()
    assert engine.device_memory()["free"] >= before["free"] - (64 << 20)
