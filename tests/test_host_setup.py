"""Host-side logic of the GPU library (no device needed): the C-ABI loads,
exports every declared symbol, and fetigpu_create's setup (constraint rows,
gaps, multiplicities, scaling weights; decomposition.hpp:58-180) matches the
independent CPU oracle row by row."""
import re
import os

import numpy as np
import pytest

from paper_2111_11728_b200 import problems as pb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    txt = open(os.path.join(ROOT, "include", "fetigpu.h")).read()
    return sorted(set(re.findall(r"\b(fetigpu_[a-z_0-9A-Z]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2111_11728_b200 import engine
    L = engine.lib()
    syms = _declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(engine.EXPORTED) <= set(syms)


def _cases():
    return [pb.config1(), pb.config1(random_blocks=True, seed=3),
            pb.config2(sx=4, sy=2, n=8), pb.config3(method=0, sx=4, sy=2, n=8),
            pb.config3(method=1, sx=4, sy=2, n=8), pb.config5(sx=4, sy=2, n=12, n_designs=3),
            pb.config4(sx=3, sy=3, n=6), pb.config1(sx=3, sy=3, n=8).replace(scaling=1)]


@pytest.mark.parametrize("case", range(8))
def test_rows_and_weights_match_oracle(case, oracle_mod):
    from paper_2111_11728_b200 import engine
    prob = _cases()[case]
    o = oracle_mod.Oracle(prob)
    g = engine.FetiSystem(prob, build=False)
    assert g.m == o.m
    ro, rg = o.rows(), g.rows()
    for k in ("kind", "sub_plus", "dof_plus", "mult"):
        np.testing.assert_array_equal(ro[k], rg[k], err_msg=k)
    iface = ro["kind"] == 0
    np.testing.assert_array_equal(ro["sub_minus"][iface], rg["sub_minus"][iface])
    np.testing.assert_array_equal(ro["dof_minus"][iface], rg["dof_minus"][iface])
    np.testing.assert_array_equal(ro["gap"], rg["gap"])
    # weights: same arithmetic (diagonals summed in element order) -> bit-exact
    np.testing.assert_array_equal(ro["w_plus"], rg["w_plus"])
    np.testing.assert_array_equal(ro["w_minus"][iface], rg["w_minus"][iface])
    st = g.stats()
    assert st["n_c"] == o.n_c
    if prob.method == 0:
        assert st["n_kept"] == o.n_kept


def test_create_errors_map_to_reference_exceptions():
    from paper_2111_11728_b200 import engine
    p = pb.config1(sx=2, sy=1, n=4)
    with pytest.raises(engine.DomainError):
        engine.FetiSystem(p.replace(densities=p.densities * 2.0), build=False)
    with pytest.raises(engine.InvalidArgument):
        engine.FetiSystem(p.replace(Emin=2.0), build=False)
    with pytest.raises(engine.NodeNotFound):
        engine.FetiSystem(p.replace(dirichlet=[(10 ** 6, 0, 0.0)]), build=False)
    with pytest.raises(engine.EdgeNotOnBoundary):
        engine.FetiSystem(p.replace(tractions=[(0, 1, 2, 5, 0.0, -1.0)]), build=False)
    with pytest.raises(engine.ConfigError):
        engine.FetiSystem(p.replace(method=7), build=False)


def test_build_without_device_fails_loudly():
    from conftest import has_gpu
    if has_gpu():
        pytest.skip("device present")
    from paper_2111_11728_b200 import engine
    g = engine.FetiSystem(pb.config1(sx=2, sy=1, n=4), build=False)
    with pytest.raises((engine.NoDevice, engine.CudaError)):
        g.build()


def test_bench_work_formula_matches_library():
    """bench.py's analytic C4 work (used by the reference arm) equals the
    library's own count, and SURVEY.md App. A's figures."""
    import bench
    from paper_2111_11728_b200 import engine
    w = bench.c4_work()
    g = engine.FetiSystem(pb.config4(), build=False)
    s = g.stats()
    assert s["m"] == w["m"] == 504000 and s["n_c"] == w["n_c"] == 4224
    assert s["op_bytes"] == w["bytes"] == 4279246848.0
    assert abs(s["op_flops_per_col"] * 2048 - 2.183e12) < 1e9
    for fn, m, nc in ((pb.config2, 3224, 80), (lambda: pb.config3(method=1), 14384, 302),
                      (pb.config5, 91744, 1118), (lambda: pb.config3(method=0), 15736, 0)):
        st = engine.FetiSystem(fn(), build=False).stats()
        assert (st["m"], st["n_c"]) == (m, nc)
