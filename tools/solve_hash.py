"""Bit-identity probe for solver-loop changes: sha1 of lambda and the device
solve time of a few PCG / FO solves (warm: second solve on the context)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

cases = [("C1", pb.config1, 0), ("C2-fo", pb.config2, 1), ("C3tf-fo", lambda: pb.config3(method=0), 1),
         ("C3dp-fo", lambda: pb.config3(method=1), 1), ("C2-rrs", pb.config2, 2)]
for name, fn, dirs in cases:
    g = engine.FetiSystem(fn())
    g.solve(tol=1e-6, max_it=2000, directions=dirs)
    lam, tr = g.solve(tol=1e-6, max_it=2000, directions=dirs)
    print(name, tr["iterations"], hashlib.sha1(lam.tobytes()).hexdigest()[:16], round(tr["solve_ms"], 2), flush=True)
    g.close()
