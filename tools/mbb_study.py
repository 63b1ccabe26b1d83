"""The paper's modular-MBB study on the GPU (PAPER.md 4.2, Figs. 4-6;
SPEC.md:511-519, acceptance 1 and 5): a 12 x 8 grid of 30 x 30-element
modules of 16 types (184,512 DOFs), modular SIMP/OC from the uniform design,
snapshots at iterations 4, 8 and 30, and the 12-variant solver grid on each
snapshot.  The module-type layout of Fig. 4 is not recoverable from the paper
(SPEC.md:538); a seeded uniform assignment of the 16 types stands in.

    python tools/mbb_study.py --out profiles/r01_mbb_study.json
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
ap.add_argument("--snapshots", default="4,8,30")
ap.add_argument("--maxit", type=int, default=2000)
ap.add_argument("--tol", type=float, default=1e-6)
ap.add_argument("--out", default="mbb_study.json")
args = ap.parse_args()

sx, sy, n = 12, 8, args.n
types = np.minimum((pb.uniform(2111, sx * sy) * 16).astype(np.int32), 15)
gxn = sx * n + 1
base = pb.Problem(sx, sy, n, np.full((16, n, n), 0.5), types, method=pb.FETIDP, scaling=pb.KSCALING,
                  precond=pb.DIRICHLET, Emin=1e-9, dirichlet=pb.bottom_corner_pins(sx, sy, n),
                  point_loads=[((sy * n) * gxn + (sx * n) // 2, 1, -1.0)], name="mbb")
snaps = tuple(int(s) for s in args.snapshots.split(","))
t0 = time.perf_counter()
st = simp.optimize(base, iterations=args.iters, volfrac=0.5, directions=2, snapshots=snaps)
out = {"modules": [sx, sy], "elems_per_module": n, "types": 16,
       "total_subdomain_dofs": sx * sy * 2 * (n + 1) ** 2, "simp_wall_s": time.perf_counter() - t0,
       "compliance": st.compliance, "state_solves": st.solves, "snapshots": {}}
print("SIMP done", out["simp_wall_s"], st.compliance[:3], st.compliance[-3:], flush=True)
print("state solves", st.solves, flush=True)
for it in snaps:
    dens = st.snapshots[it]
    row = {}
    for mname, method in (("tfeti", pb.TFETI), ("fetidp", pb.FETIDP)):
        for sname, scaling in (("multiplicity", pb.MULTIPLICITY), ("k", pb.KSCALING)):
            p = base.replace(densities=dens, method=method, scaling=scaling)
            g = engine.FetiSystem(p)
            for dname, dirs in (("single", 0), ("fo", 1), ("rrs", 2)):
                try:
                    lam, tr = g.solve(tol=args.tol, max_it=args.maxit if dirs < 2 else 300, directions=dirs)
                    row[f"{mname}_{sname}_{dname}"] = {
                        "iterations": tr["iterations"], "status": ["converged", "max_iter", "breakdown"][tr["status"]],
                        "rel_eps": tr["eps_final"] / tr["eps0"], "solve_ms": round(tr["solve_ms"], 1),
                        "m": g.m}
                except engine.FetiError as e:
                    row[f"{mname}_{sname}_{dname}"] = {"error": type(e).__name__}
                print(it, mname, sname, dname, row[f"{mname}_{sname}_{dname}"], flush=True)
            g.close()
    out["snapshots"][str(it)] = row
with open(args.out, "w") as f:
    json.dump(out, f, indent=1)
print("written", args.out)
