"""Full-size parity where FP64 rounding, amplified by the SIMP contrast,
dominates: the GPU must stay inside the reference algorithm's OWN rounding
spread, measured here as the distance between the double-precision oracle and
the accuracy reference (the oracle with long-double refined local / coarse
solves, fo_set_refine).  Round-1 measurements (profiles/): C2 single
direction GPU 3189 vs oracle 3105 vs refined 3422 iterations; C3 FETI-DP FO
displacements GPU-vs-oracle 5.5e-4 against oracle-vs-refined 5.3e-3.

* C2 (BASELINE configs[1], single direction as configured): the GPU's
  iteration count lies within the oracle's own last-bit spread of the
  oracle's median (see the test);
* C3 FETI-DP FO and C3 T-FETI FO: ||u_gpu - u_oracle|| <=
  max(||u_oracle - u_refined||, 1e-8) (relative L2), and iteration counts
  within +-1 of the oracle;
* C5 RRS: the GPU's true preconditioned residual within 10x the oracle's,
  both measured with the accuracy reference's operator (the refined
  oracle's RRS itself breaks down on C5).
C3 T-FETI (about 4 min of CPU oracle time) and C5 (about 12 min) are marked
slow (FETIGPU_SLOW_TESTS=1).
"""
import numpy as np
import pytest

from paper_2111_11728_b200 import problems as pb

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _runs(prob, oracle_mod, **kw):
    from paper_2111_11728_b200 import engine
    L = oracle_mod.lib()
    o = oracle_mod.Oracle(prob)
    lo, to = o.solve(**kw)
    L.fo_set_refine(1)
    r = oracle_mod.Oracle(prob)
    lr, tr = r.solve(**kw)
    L.fo_set_refine(0)
    g = engine.FetiSystem(prob)
    lg, tg = g.solve(**kw)
    res = dict(g=(lg, tg, g.recover(lg)), o=(lo, to, o.recover(lo)), r=(lr, tr, r.recover(lr)))
    g.close()
    return res


def test_c2_single_direction_iterations_within_spread(oracle_mod):
    """Single-direction PCG at contrast 1e6 over ~3000 iterations is
    roundoff-chaotic: the reference's own count moves by hundreds under
    last-bit changes of the input (E0 or Emin scaled by 1 +- 2^-46, 2^-40:
    3030..3126 on the box; the long-double refined oracle: 3422).  The GPU
    (a different FP64 implementation: explicit F_s) must lie within that
    spread of the oracle's median: |gpu - median| <= max - min."""
    from paper_2111_11728_b200 import engine
    prob = pb.config2()
    kw = dict(tol=1e-6, max_it=6000, directions=0)
    L = oracle_mod.lib()
    counts = []
    for q in (prob, prob.replace(E0=prob.E0 * (1 + 2.0 ** -46)), prob.replace(E0=prob.E0 * (1 - 2.0 ** -46)),
              prob.replace(Emin=prob.Emin * (1 + 2.0 ** -40)), prob.replace(Emin=prob.Emin * (1 - 2.0 ** -40))):
        _, t = oracle_mod.Oracle(q).solve(**kw)
        assert t["status"] == 0
        counts.append(t["iterations"])
    L.fo_set_refine(1)
    _, tr = oracle_mod.Oracle(prob).solve(**kw)
    L.fo_set_refine(0)
    counts.append(tr["iterations"])
    g = engine.FetiSystem(prob)
    _, tg = g.solve(**kw)
    g.close()
    med, spread = float(np.median(counts)), max(counts) - min(counts)
    print("C2 single: gpu", tg["iterations"], "oracle runs", counts, "median", med, "spread", spread)
    assert tg["status"] == 0
    assert abs(tg["iterations"] - med) <= spread


def _displacement_spread(name, prob, oracle_mod, directions, max_it):
    R = _runs(prob, oracle_mod, tol=1e-6, max_it=max_it, directions=directions)
    ug, uo, ur = (R[x][2] for x in "gor")
    eg, eo = rel(ug, uo), rel(uo, ur)
    print(name, "its gpu/oracle/refined", [R[x][1]["iterations"] for x in "gor"],
          "u gpu-vs-oracle %.2e oracle-vs-refined %.2e gpu-vs-refined %.2e" % (eg, eo, rel(ug, ur)))
    assert all(R[x][1]["status"] == 0 for x in "gor")
    assert abs(R["g"][1]["iterations"] - R["o"][1]["iterations"]) <= 1
    assert eg <= max(eo, 1e-8)


def test_c3_fetidp_fo_displacements_within_spread(oracle_mod):
    _displacement_spread("C3 FETI-DP FO", pb.config3(method=1), oracle_mod, 1, 2000)


@pytest.mark.slow
def test_c3_tfeti_fo_displacements_within_spread(oracle_mod):
    _displacement_spread("C3 T-FETI FO", pb.config3(method=0), oracle_mod, 1, 2000)


@pytest.mark.slow
def test_c5_rrs_true_residual_vs_oracle(oracle_mod):
    """Full C5 (1e9 contrast, 0/1 designs) with RRS.  The refined oracle's RRS
    breaks down there (a roundoff-negative pivot: IndefiniteInput), and the
    recursively updated residual of Alg. 1 drifts from the true one at this
    conditioning (profiles/r01_c5_conditioning_diag.json), so both solutions
    are scored by their TRUE preconditioned residual rho(lambda) =
    sqrt(r^T M r), r = d - F lambda, relative to rho(0), with F, M and d of
    the ACCURACY REFERENCE (the oracle with long-double refined local and
    coarse solves): the GPU's must be within ACC_FACTOR (10) of the oracle's,
    with the same iteration count +-1.  Measured with the double oracle's own
    F instead, each solution would be scored against that operator's rounding
    (F_oracle is 3.5e-3 from the reference on C5, F_gpu 8.1e-4: DESIGN.md 2),
    which favours the oracle by construction (round-2 run: 3.7e-2 vs 6.9e-7).
    Both measures and the dual energies are printed."""
    from paper_2111_11728_b200 import engine
    prob = pb.config5()
    L = oracle_mod.lib()
    L.fo_set_refine(0)
    o = oracle_mod.Oracle(prob)
    lo, to = o.solve(tol=1e-6, max_it=200, directions=2)
    g = engine.FetiSystem(prob)
    lg, tg = g.solve(tol=1e-6, max_it=200, directions=2)
    g.close()
    L.fo_set_refine(1)
    ref = oracle_mod.Oracle(prob)
    L.fo_set_refine(0)

    def scores(sys_):
        d, _ = sys_.rhs()

        def rho(lam):
            r = d - sys_.apply_F(lam)
            return np.sqrt(max(r @ sys_.apply_precond(r), 0.0))
        r0 = rho(np.zeros_like(d))
        J = lambda lam: 0.5 * lam @ sys_.apply_F(lam) - d @ lam   # noqa: E731
        return rho(lg) / r0, rho(lo) / r0, J(lg), J(lo)
    rg, ro, Jg, Jo = scores(ref)
    og, oo, _, _ = scores(o)
    print("C5 RRS its gpu", tg["iterations"], "oracle", to["iterations"],
          "| true rel residual (reference operator) gpu %.3e oracle %.3e" % (rg, ro),
          "| J gpu %.10e oracle %.10e" % (Jg, Jo),
          "| with the double oracle's operator gpu %.3e oracle %.3e" % (og, oo))
    assert tg["status"] == to["status"] == 0
    assert abs(tg["iterations"] - to["iterations"]) <= 1
    assert rg <= 10.0 * ro
