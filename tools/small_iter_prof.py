"""One short solve of C1 (single) and C2 (FO) for a per-kernel launch list
(ncu) of the device-resident iteration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "C1"
prob = pb.config1() if which == "C1" else pb.config2()
g = engine.FetiSystem(prob)
lam, tr = g.solve(tol=1e-12, max_it=5, directions=0 if which == "C1" else 1)
print(which, tr["iterations"], tr["solve_ms"])
