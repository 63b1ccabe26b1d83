"""The symmetric-packed GEMV kernels (TMA ring form and LDG form) on small
problems, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FETIGPU_FORCE_SYM"] = "1"
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

for prob in (pb.config4(sx=8, sy=5, n=6), pb.config1(sx=5, sy=4, n=5), pb.config4(sx=12, sy=10, n=2)):
    g = engine.FetiSystem(prob)
    x = np.random.default_rng(0).standard_normal(g.m)
    y = g.apply_F(x)
    z = g.apply_precond(x)
    assert g.stats()["apply_kernel"] == 2
    lam, tr = g.solve(tol=1e-6, max_it=20, directions=0)
    g.close()
print("sanitize sym ok")
