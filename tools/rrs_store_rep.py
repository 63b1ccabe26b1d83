import sys, os
sys.path.insert(0, os.getcwd())
from paper_2111_11728_b200 import engine, problems as pb
for name, fn in (("C5", pb.config5), ("C2", pb.config2)):
    g = engine.FetiSystem(fn())
    for mode in ("implicit", "explicit", "implicit", "explicit", "implicit"):
        g.set_rrs_store(mode)
        lam, tr = g.solve(tol=1e-6, max_it=200, directions=2)
        print(name, mode, tr["iterations"], round(tr["solve_ms"], 1), [round(x, 1) for x in tr["phase_ms"]], flush=True)
    g.close()
