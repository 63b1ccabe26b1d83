"""Seeded synthetic inputs: deterministic, in range, and with
the shapes / statistics each BASELINE.json config names."""
import numpy as np
import pytest

from paper_2111_11728_b200 import problems as pb


def test_splitmix64_reference_values():
    # SplitMix64 from seed 0: first outputs of the published generator
    out = pb.splitmix64(0, 3)
    assert [int(v) for v in out] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    u = pb.uniform(7, 10000)
    assert u.min() >= 0.0 and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.01
    z = pb.normal(7, 20000)
    assert abs(z.mean()) < 0.03 and abs(z.std() - 1.0) < 0.03


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_configs_deterministic_and_in_range(name):
    kw = dict(C4=dict(sx=8, sy=4), C5=dict(sx=8, sy=4)).get(name, {})
    a, b = pb.CONFIGS[name](**kw), pb.CONFIGS[name](**kw)
    assert np.array_equal(a.densities, b.densities)
    assert np.array_equal(a.module_type, b.module_type)
    assert a.densities.min() >= 0.0 and a.densities.max() <= 1.0
    assert len(a.module_type) == a.sx * a.sy
    assert a.module_type.max() < a.densities.shape[0]


def test_config_shapes_and_statistics():
    c1 = pb.config1()
    assert (c1.sx, c1.sy, c1.n) == (4, 2, 16) and set(np.unique(c1.densities)) == {0.1, 1.0}
    # seeded checkerboard of 4x4 blocks, phase = seed & 1
    assert not np.array_equal(pb.config1(seed=1).densities, pb.config1(seed=2).densities)
    c2 = pb.config2()
    assert (c2.sx, c2.sy, c2.n, c2.Emin) == (8, 4, 32, 1e-6) and set(np.unique(c2.densities)) <= {0.0, 1.0}
    assert abs(c2.densities.mean() - 0.5) < 0.01                       # Bernoulli(0.5)
    c3 = pb.config3()
    vals = np.unique(c3.densities)
    assert {0.0, 0.25, 0.75, 1.0} <= set(np.round(vals, 12))           # 2-element ramp
    c4 = pb.config4(sx=8, sy=4)
    assert c4.n == 64 and abs(c4.densities.mean() - 0.5) < 0.01        # U(0,1)
    c5 = pb.config5()
    assert c5.densities.shape == (10, 48, 48) and (c5.sx, c5.sy) == (32, 16)
    for d in c5.densities:                                             # volume fraction 0.4
        assert abs(d.mean() - 0.4) < 0.01
    assert len(np.unique(c5.module_type)) == 10


def test_presets():
    lb = pb.laminated_beam()
    assert (lb.sx, lb.sy) == (9, 1) and lb.n % 7 == 0
    assert lb.densities[0][0::2].sum() > 0   # layers alternate
    g3 = pb.grid3x3_layered()
    assert (g3.sx, g3.sy) == (3, 3)
    inc = pb.grid4x4_inclusion()
    d = inc.densities[0]
    assert (inc.sx, inc.sy) == (4, 4) and d[0].sum() == 0 and d[:, 0].sum() == 0   # inclusion off the boundary
    with pytest.raises(ValueError):
        pb.laminated_beam(n=10)


def test_bench_stream_bytes_and_shared_config():
    """bench.py: the headline byte count (symmetric storage, SURVEY 8d layout)
    and the config dict both arms print (same workload, same constant)."""
    import bench
    w = bench.c4_work()
    assert w["bytes"] == 4279246848.0                 # SURVEY App. A full-storage formula
    assert w["packed_main_bytes"] == 2190999552.0     # the packed kernel's bytes per launch
    assert w["stream_bytes"] == 2407302912.0
    assert w["m"] == 504000 and w["n_c"] == 4224
    c1, c2 = bench.c4_config(), bench.c4_config()
    assert c1 == c2 and c1["value_bytes_per_apply"] == w["stream_bytes"]
