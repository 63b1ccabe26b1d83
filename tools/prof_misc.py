"""Profiling driver for the non-GEMV kernel families: the device build of
C4 (ND tree + slot eliminations), then a few FO iterations of C4 (dots,
re-orthogonalization) and of C3 T-FETI (projector).  Used under ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

g = engine.FetiSystem(pb.config4())
print("C4 build_ms", g.stats()["build_ms"])
_, tr = g.solve(tol=1e-12, max_it=20, directions=1)
print("C4 FO 20 its", tr["solve_ms"])
g.close()
g = engine.FetiSystem(pb.config3(method=0))
_, tr = g.solve(tol=1e-12, max_it=20, directions=1)
print("C3 tfeti FO 20 its", tr["solve_ms"])
