"""Small end-to-end exercise of every device path (for compute-sanitizer)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

for prob in (pb.config1(sx=3, sy=2, n=4), pb.config2(sx=3, sy=2, n=6),
             pb.config3(method=0, sx=3, sy=2, n=6).replace(precond=0),
             pb.config5(sx=3, sy=2, n=6, n_designs=2), pb.config1(sx=2, sy=2, n=5).replace(precond=2)):
    g = engine.FetiSystem(prob)
    x = np.random.default_rng(0).standard_normal(g.m)
    g.apply_F(x)
    g.apply_F_block(np.random.default_rng(1).standard_normal((g.m, 6)))
    g.apply_precond(x, columns=True)
    g.project(x)
    for d in (0, 1, 2):
        lam, tr = g.solve(tol=1e-8, max_it=50, directions=d)
    g.recover(lam)
    g.close()
print("sanitize run ok")
