"""Seeded randomized GPU-vs-oracle sweep.

Each case draws:
* a partition from 1x1 to 4x3 subdomains (including the degenerate 1x1
  FETI-DP problem with m = 0 dual rows, and 1 x k strips);
* modules of 2..8 elements;
* a method (T-FETI / FETI-DP), a scaling (multiplicity / k) and a
  preconditioner (lumped / Dirichlet / super-lumped);
* 1-3 module designs of uniform, 0/1 or constant densities at contrasts
  1e-2..1e-6;
* supports: left clamp, bottom pins, or a clamp with prescribed nonzero
  displacements (constraint gaps);
* loads: right-edge traction or a point load on a module perimeter.

GPU and oracle see identical inputs.  The operator, preconditioner,
right-hand side and recovered displacements follow the accuracy policy of
test_gpu_parity.py (within ACC_FACTOR x the double oracle's own distance to
the refined oracle).  FO and RRS iteration counts must agree within +-1."""
import numpy as np
import pytest

from paper_2111_11728_b200 import problems as pb

pytestmark = pytest.mark.gpu
ACC_FACTOR = 10.0
SEEDS = list(range(64))


def random_problem(seed):
    rng = np.random.default_rng(7000 + seed)
    sx, sy = int(rng.integers(1, 5)), int(rng.integers(1, 4))
    n = int(rng.choice([2, 3, 4, 6, 8]))
    method, scaling, precond = int(rng.integers(0, 2)), int(rng.integers(0, 2)), int(rng.integers(0, 3))
    nd = int(rng.integers(1, 4))
    emin = float(10.0 ** -rng.uniform(2, 6))
    kind = int(rng.integers(0, 3))
    if kind == 0:
        dens = rng.uniform(0.0, 1.0, (nd, n, n))
    elif kind == 1:
        dens = (rng.uniform(0.0, 1.0, (nd, n, n)) < 0.6).astype(float)
    else:
        dens = np.full((nd, n, n), float(rng.uniform(0.2, 1.0)))
    mt = rng.integers(0, nd, sx * sy).astype(np.int32)
    bc = int(rng.integers(0, 3))
    if bc == 0:
        dirichlet = pb.left_clamp(sx, sy, n)
    elif bc == 1:
        dirichlet = pb.bottom_corner_pins(sx, sy, n)
    else:  # clamp with small prescribed displacements -> nonzero gaps
        dirichlet = [(g, d, float(rng.uniform(-1e-2, 1e-2))) for g, d, _ in pb.left_clamp(sx, sy, n)]
    gx_n = sx * n + 1
    if rng.uniform() < 0.5:
        tractions, point_loads = pb.right_edge_traction(sx, sy, n), []
    else:  # top edge node on a vertical module line
        gx = int(rng.integers(0, sx + 1)) * n
        tractions, point_loads = [], [((sy * n) * gx_n + gx, int(rng.integers(0, 2)), -1.0)]
    return pb.Problem(sx, sy, n, dens, mt, method=method, scaling=scaling, precond=precond, Emin=emin,
                      dirichlet=dirichlet, tractions=tractions, point_loads=point_loads, name=f"fuzz{seed}")


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


def accurate(got, dbl, ref, what):
    eg, ed = rel(got, ref), rel(dbl, ref)
    assert eg <= max(ACC_FACTOR * ed, 1e-11), (what, eg, ed)


@pytest.mark.parametrize("seed", SEEDS)
def test_random_problem(seed, oracle_mod):
    from paper_2111_11728_b200 import engine
    prob = random_problem(seed)
    L = oracle_mod.lib()
    L.fo_set_refine(0)
    o = oracle_mod.Oracle(prob)
    L.fo_set_refine(1)
    r = oracle_mod.Oracle(prob)
    L.fo_set_refine(0)
    g = engine.FetiSystem(prob)
    try:
        assert g.m == o.m
        m = g.m
        if m > 0:
            x = np.random.default_rng(seed).standard_normal(m)
            accurate(g.apply_F(x), o.apply_F(x), r.apply_F(x), f"seed {seed} F")
            accurate(g.apply_precond(x), o.apply_precond(x), r.apply_precond(x), f"seed {seed} M")
            dg, _ = g.rhs()
            do, _ = o.rhs()
            dr, _ = r.rhs()
            accurate(dg, do, dr, f"seed {seed} d")
        for dirs in (1, 2):  # FO, then RRS
            res = {}
            for name, sysm in (("gpu", g), ("oracle", o), ("ref", r)):
                try:
                    res[name] = sysm.solve(tol=1e-8, max_it=2000 if dirs == 1 else 300, directions=dirs)
                except (engine.NegativeInnerProduct, engine.IndefiniteInput, oracle_mod.OracleError) as e:
                    res[name] = e
            if any(isinstance(v, Exception) for v in res.values()):
                # A tiny projected Krylov space can be exhausted exactly (e.g. 6 dims
                # on a 12-row T-FETI problem): the next residual / Gram block is pure
                # rounding noise and the sign tests of residual_metric /
                # pivoted_cholesky may fire on either side.
                # Accept that only if every side that did not raise had reached
                # rounding level.
                for v in res.values():
                    if not isinstance(v, Exception):
                        t = v[1]
                        assert (t["eps"] / max(t["eps0"], 1e-300)).min() <= 1e-12, (dirs, t["eps"])
                continue
            (lg, tg), (lo, to), (lr, tr) = res["gpu"], res["oracle"], res["ref"]
            assert tg["status"] == to["status"], dirs
            assert abs(tg["iterations"] - to["iterations"]) <= 1, (dirs, tg["iterations"], to["iterations"])
            if dirs == 1:
                ug, uo, ur = g.recover(lg), o.recover(lo), r.recover(lr)
                accurate(np.ravel(ug), np.ravel(uo), np.ravel(ur), f"seed {seed} u")
    finally:
        g.close()
