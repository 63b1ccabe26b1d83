"""K15, the persistent PCG / FO loop (kernels_persist.cuh), against the
CUDA-graph loop it replaces: the same solve on the same context must give
bit-identical lambda and eps traces and the same iteration count, for both
methods, all three preconditioners, both scalings, single direction and FO,
grid and cluster barriers, and problems with rollers, lumped / super-lumped
preconditioners and one-direction supports.  (The graph loop itself is
checked against the CPU oracle in test_gpu_parity.py.)"""
import os

import numpy as np
import pytest

from paper_2111_11728_b200 import problems as pb

pytestmark = pytest.mark.gpu

CASES = {
    "C1": lambda: pb.config1(),
    "C1b": lambda: pb.config1(random_blocks=True, seed=3),
    "C2": lambda: pb.config2(),
    "C2s": lambda: pb.config2(sx=4, sy=2, n=8),
    "C3tf_s": lambda: pb.config3(method=0, sx=4, sy=2, n=8),
    "C3dp_s": lambda: pb.config3(method=1, sx=4, sy=2, n=8),
    "C5s": lambda: pb.config5(sx=4, sy=2, n=12, n_designs=3),
    "C1_dir_k": lambda: pb.config1(sx=3, sy=3, n=8).replace(scaling=1, precond=1),
    "C2_lumped": lambda: pb.config2(sx=3, sy=2, n=10).replace(precond=0),
    "C3tf_super": lambda: pb.config3(method=0, sx=3, sy=2, n=8).replace(precond=2),
    "C2_roller_vertex": lambda: pb.config2(sx=3, sy=2, n=8).replace(
        dirichlet=[(0, 0, 0.0), (0, 1, 0.0), (3 * 8, 1, 0.0)], point_loads=[((2 * 8) * 25 + 12, 1, -1.0)]),
    "C2_roller_edge": lambda: pb.config2(sx=3, sy=2, n=8).replace(
        dirichlet=pb.left_clamp(3, 2, 8) + [(3 * 25 + 8, 0, 0.0)]),
}
KEYS = ("FETIGPU_PERSIST", "FETIGPU_PERSIST_G", "FETIGPU_PERSIST_BAR", "FETIGPU_PERSIST_RED", "FETIGPU_CLUSTER")


def solve(g, dirs, env, max_it=3000):
    old = {k: os.environ.pop(k, None) for k in KEYS}
    os.environ.update(env)
    try:
        lam, tr = g.solve(tol=1e-6, max_it=max_it, directions=dirs)
        loop = g.stats()["solve_loop"]
    finally:
        for k in KEYS:
            os.environ.pop(k, None)
            if old[k] is not None:
                os.environ[k] = old[k]
    return lam, tr, loop


def same(a, b):
    (la, ta, _), (lb, tb, _) = a, b
    assert ta["iterations"] == tb["iterations"], (ta["iterations"], tb["iterations"])
    assert ta["status"] == tb["status"]
    assert np.array_equal(la.view(np.uint64), lb.view(np.uint64)), "lambda differs"
    assert np.array_equal(ta["eps"].view(np.uint64), tb["eps"].view(np.uint64)), "eps trace differs"


@pytest.mark.parametrize("dirs", [0, 1])
@pytest.mark.parametrize("name", list(CASES))
def test_persistent_equals_graph(name, dirs):
    from paper_2111_11728_b200 import engine
    prob = CASES[name]()
    g = engine.FetiSystem(prob)
    try:
        ref = solve(g, dirs, {"FETIGPU_PERSIST": "0", "FETIGPU_CLUSTER": "0"})
        assert ref[2] == 1, "graph loop expected"
        got = solve(g, dirs, {"FETIGPU_PERSIST": "1", "FETIGPU_CLUSTER": "0"})
        assert got[2] == 2, f"persistent loop did not run (solve_loop {got[2]})"
        same(ref, got)
        print(name, dirs, ref[1]["iterations"], "iterations, bit-identical")
        if dirs == 0 and prob.method == 0 and g.stats()["n_sub"] <= 16:
            clu = solve(g, dirs, {"FETIGPU_CLUSTER": "1"})
            assert clu[2] == 4, f"cluster-resident loop did not run (solve_loop {clu[2]})"
            same(ref, clu)
    finally:
        g.close()


@pytest.mark.parametrize("name,dirs", [("C1", 0), ("C1", 1), ("C2s", 1), ("C3tf_s", 0)])
@pytest.mark.parametrize("env", [{"FETIGPU_PERSIST_G": "16", "FETIGPU_PERSIST_BAR": "cluster"},
                                 {"FETIGPU_PERSIST_G": "37", "FETIGPU_PERSIST_BAR": "grid"},
                                 {"FETIGPU_PERSIST_RED": "1"}])
def test_persistent_grid_variants(name, dirs, env):
    """Grid size, barrier kind and the redundant coarse applies do not change a bit."""
    from paper_2111_11728_b200 import engine
    g = engine.FetiSystem(CASES[name]())
    try:
        ref = solve(g, dirs, {"FETIGPU_PERSIST": "0", "FETIGPU_CLUSTER": "0"})
        got = solve(g, dirs, dict(env, FETIGPU_PERSIST="1", FETIGPU_CLUSTER="0"))
        assert got[2] == (3 if env.get("FETIGPU_PERSIST_BAR") == "cluster" else 2)
        same(ref, got)
    finally:
        g.close()


def test_persistent_default_policy():
    """The default picks the cluster-resident loop for C1 (T-FETI single
    direction, operators in shared memory), the persistent loop where it is
    faster (small operators) and the graph loop for C3-sized ones (DESIGN.md
    4, K15)."""
    from paper_2111_11728_b200 import engine
    for prob, dirs, want in ((pb.config1(), 0, 4), (pb.config1(), 1, 2), (pb.config2(), 0, 2),
                             (pb.config2(), 1, 2), (pb.config3(method=1), 1, 1)):
        g = engine.FetiSystem(prob)
        try:
            _, tr, loop = solve(g, dirs, {}, max_it=20)
            assert loop == want, (prob, dirs, loop)
        finally:
            g.close()


def test_persistent_repeat_and_breakdown_free_restart():
    """Two persistent solves on one context are identical (barrier counters,
    coarse-gather arrival counters and direction counts are reset)."""
    from paper_2111_11728_b200 import engine
    g = engine.FetiSystem(pb.config2(sx=4, sy=2, n=8))
    try:
        a = solve(g, 1, {"FETIGPU_PERSIST": "1"})
        b = solve(g, 1, {"FETIGPU_PERSIST": "1"})
        same(a, b)
        c = solve(g, 0, {"FETIGPU_PERSIST": "1"}, max_it=5)
        assert c[1]["iterations"] == 5 and c[1]["status"] == 1   # max_iter
        d = solve(g, 0, {"FETIGPU_PERSIST": "0"}, max_it=5)
        same(c, d)
    finally:
        g.close()
    g = engine.FetiSystem(pb.config1())
    try:
        a = solve(g, 0, {"FETIGPU_CLUSTER": "1"})
        b = solve(g, 0, {"FETIGPU_CLUSTER": "1"})
        assert a[2] == 4
        same(a, b)
        c = solve(g, 0, {"FETIGPU_CLUSTER": "1"}, max_it=7)
        d = solve(g, 0, {"FETIGPU_CLUSTER": "0", "FETIGPU_PERSIST": "0"}, max_it=7)
        assert c[1]["iterations"] == 7
        same(c, d)
    finally:
        g.close()
