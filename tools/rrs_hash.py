"""Bit-identity probe for RRS changes: sha1 of lambda and solve time of
implicit-store RRS solves (warm: second solve on the context)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

for name, fn in (("C2", pb.config2), ("C5", pb.config5), ("C4", pb.config4)):
    g = engine.FetiSystem(fn())
    g.set_rrs_store("implicit")
    if name != "C4":
        g.solve(tol=1e-6, max_it=100, directions=2)
    lam, tr = g.solve(tol=1e-6, max_it=100, directions=2)
    print(name, tr["iterations"], hashlib.sha1(lam.tobytes()).hexdigest()[:16], round(tr["solve_ms"], 1),
          [round(x, 1) for x in tr["phase_ms"]], flush=True)
    g.close()
