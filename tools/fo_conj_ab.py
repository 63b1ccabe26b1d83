"""FO conjugacy of the device solver under the runtime switches (A/B)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

for name, p in (("C3dp_s", pb.config3(method=1, sx=4, sy=2, n=8)), ("C3tf_s", pb.config3(method=0, sx=4, sy=2, n=8))):
    g = engine.FetiSystem(p)
    g.set_check(True)
    for passes in (1, 2, 3):
        _, tr = g.solve(tol=1e-8, max_it=500, directions=1, reorth_passes=passes)
        print(os.environ.get("TAG", ""), name, "passes", passes, "its", tr["iterations"], "err %.2e" % g.check_result()[0],
              flush=True)
    g.close()
