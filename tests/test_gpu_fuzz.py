"""Seeded randomized GPU-vs-oracle sweep.

Each case draws:
* a partition from 1x1 to 4x3 subdomains (including the degenerate 1x1
  FETI-DP problem with m = 0 dual rows, and 1 x k strips);
* modules of 2..8 elements;
* a method (T-FETI / FETI-DP), a scaling (multiplicity / k) and a
  preconditioner (lumped / Dirichlet / super-lumped);
* 1-3 module designs of uniform, 0/1 or constant densities at contrasts
  1e-2..1e-6;
* element sizes hx != hy, Poisson ratio 0..0.45, thickness, SIMP exponent
  1..4 and E0 0.1..100;
* supports: left clamp, bottom pins, or a clamp with prescribed nonzero
  displacements (constraint gaps);
* loads: right-edge traction or a point load on a module perimeter.

GPU and oracle see identical inputs.  The accuracy yardstick is the
problem's own sensitivity to last-bit rounding: a third oracle runs on
densities perturbed by 2^-47..2^-45 relative noise, and the GPU's distance to the
oracle must stay within SENS_FACTOR x that perturbed oracle's distance (plus
a small floor).  The refined-oracle policy of test_gpu_parity.py is not used
here: its reference shares the oracle's own K assembly, so on anisotropic
elements or non-unit moduli it favours the oracle by the conditioning-amplified
assembly rounding, which an ND-Schur assembly cannot reproduce bit for bit.
FO and RRS iteration counts must agree within +-1."""
import os

import numpy as np
import pytest

from paper_2111_11728_b200 import problems as pb

pytestmark = pytest.mark.gpu
SENS_FACTOR = 100.0
SEEDS = list(range(int(os.environ.get("FETIGPU_FUZZ_SEEDS", "64"))))  # longer sweeps: raise the count


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
    # material / geometry: anisotropic elements, Poisson ratio, thickness, SIMP exponent, E0
    mat = dict(hx=float(rng.uniform(0.5, 2.0)), hy=float(rng.uniform(0.5, 2.0)), nu=float(rng.uniform(0.0, 0.45)),
               thickness=float(rng.uniform(0.5, 2.0)), p=float(rng.choice([1.0, 2.0, 3.0, 4.0])),
               E0=float(10.0 ** rng.uniform(-1, 2)))
    mat["Emin"] = emin * mat["E0"]
    return pb.Problem(sx, sy, n, dens, mt, method=method, scaling=scaling, precond=precond,
                      dirichlet=dirichlet, tractions=tractions, point_loads=point_loads, name=f"fuzz{seed}", **mat)


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


def close(got, dbl, pert, what, floor=5e-11):
    """|got - dbl| within SENS_FACTOR x the rounding sensitivity |pert - dbl|."""
    eg, es = rel(got, dbl), rel(pert, dbl)
    assert eg <= max(SENS_FACTOR * es, floor), (what, eg, es)


def perturbed(prob, seed):
    rng = np.random.default_rng(10_000 + seed)
    # a few ulps (2^-47..2^-45 relative): large enough never to round away
    d = prob.densities * (1.0 - rng.uniform(2.0 ** -47, 2.0 ** -45, prob.densities.shape))
    return prob.replace(densities=d)


@pytest.mark.parametrize("seed", SEEDS)
def test_random_problem(seed, oracle_mod):
    from paper_2111_11728_b200 import engine
    prob = random_problem(seed)
    o = oracle_mod.Oracle(prob)
    r = oracle_mod.Oracle(perturbed(prob, seed))
    g = engine.FetiSystem(prob)
    try:
        assert g.m == o.m
        m = g.m
        if m > 0:
            x = np.random.default_rng(seed).standard_normal(m)
            close(g.apply_F(x), o.apply_F(x), r.apply_F(x), f"seed {seed} F")
            close(g.apply_precond(x), o.apply_precond(x), r.apply_precond(x), f"seed {seed} M")
            dg, _ = g.rhs()
            do, _ = o.rhs()
            dr, _ = r.rhs()
            close(dg, do, dr, f"seed {seed} d")
        for dirs in (1, 2):  # FO, then RRS
            res = {}
            for name, sysm in (("gpu", g), ("oracle", o), ("pert", r)):
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
            (lg, tg), (lo, to), (lr, tr) = res["gpu"], res["oracle"], res["pert"]
            assert tg["status"] == to["status"], dirs
            assert abs(tg["iterations"] - to["iterations"]) <= 1, (dirs, tg["iterations"], to["iterations"])
            if dirs == 1:
                ug, uo, ur = g.recover(lg), o.recover(lo), r.recover(lr)
                # solves stop at 1e-8 relative residual: floor at that level
                close(np.ravel(ug), np.ravel(uo), np.ravel(ur), f"seed {seed} u", floor=1e-7)
    finally:
        g.close()
