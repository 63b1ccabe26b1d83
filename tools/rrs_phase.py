"""Per-phase RRS timing on the MBB snapshots (profiles/r01_mbb_study.json's
slow RRS cases).  Phases: F W (K5), Gram, pivoted Cholesky, compression,
update, preconditioner+dots, next W, CGS2.

    python tools/rrs_phase.py --iters 30 --snapshots 4,30
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb, simp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--snapshots", default="4,30")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--out", default="")
args = ap.parse_args()

sx, sy, n = 12, 8, args.n
types = np.minimum((pb.uniform(2111, sx * sy) * 16).astype(np.int32), 15)
gxn = sx * n + 1
base = pb.Problem(sx, sy, n, np.full((16, n, n), 0.5), types, method=pb.FETIDP, scaling=pb.KSCALING,
                  precond=pb.DIRICHLET, Emin=1e-9, dirichlet=pb.bottom_corner_pins(sx, sy, n),
                  point_loads=[((sy * n) * gxn + (sx * n) // 2, 1, -1.0)], name="mbb")
snaps = tuple(int(s) for s in args.snapshots.split(","))
st = simp.optimize(base, iterations=args.iters, volfrac=0.5, directions=2, snapshots=snaps)
names = ["FW", "gram", "pivchol", "compress", "update", "precond", "nextW", "cgs2"]
res = []
for it in snaps:
    for mname, method in (("tfeti", pb.TFETI), ("fetidp", pb.FETIDP)):
        for sname, scaling in (("multiplicity", pb.MULTIPLICITY), ("k", pb.KSCALING)):
            g = engine.FetiSystem(base.replace(densities=st.snapshots[it], method=method, scaling=scaling))
            for rep in range(args.reps):
                t0 = time.perf_counter()
                try:
                    lam, tr = g.solve(tol=1e-6, max_it=300, directions=2)
                except engine.FetiError as e:
                    print(it, mname, sname, "error", type(e).__name__, flush=True)
                    break
                wall = (time.perf_counter() - t0) * 1e3
                ph = {k: round(v, 2) for k, v in zip(names, tr["phase_ms"])}
                row = dict(snapshot=it, variant=f"{mname}_{sname}", rep=rep, iterations=tr["iterations"],
                           solve_ms=round(tr["solve_ms"], 1), wall_ms=round(wall, 1),
                           kept_total=int(np.sum(tr["kept"][1:tr["iterations"] + 1])), phase_ms=ph)
                res.append(row)
                print(json.dumps(row), flush=True)
            g.close()
if args.out:
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
