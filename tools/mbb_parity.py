"""GPU vs CPU-oracle parity on the paper-scale modular MBB snapshots
(profiles/r01_mbb_study.json): the SIMP loop runs on the GPU, then every
variant of the 12-variant grid is solved on each snapshot by both the GPU
engine and the oracle (test infrastructure) with the same tolerance / cap.

    python tools/mbb_parity.py --snapshots 4,30 --out gpurun_out/mbb_parity.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_11728_b200 import engine, problems as pb, simp  # noqa: E402
from oracle import pyoracle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--snapshots", default="4,30")
ap.add_argument("--maxit", type=int, default=2000)
ap.add_argument("--rrs-maxit", type=int, default=300)
ap.add_argument("--tol", type=float, default=1e-6)
ap.add_argument("--out", default="mbb_parity.json")
args = ap.parse_args()

sx, sy, n = 12, 8, args.n
types = np.minimum((pb.uniform(2111, sx * sy) * 16).astype(np.int32), 15)
gxn = sx * n + 1
base = pb.Problem(sx, sy, n, np.full((16, n, n), 0.5), types, method=pb.FETIDP, scaling=pb.KSCALING,
                  precond=pb.DIRICHLET, Emin=1e-9, dirichlet=pb.bottom_corner_pins(sx, sy, n),
                  point_loads=[((sy * n) * gxn + (sx * n) // 2, 1, -1.0)], name="mbb")
snaps = tuple(int(s) for s in args.snapshots.split(","))
st = simp.optimize(base, iterations=max(snaps), volfrac=0.5, directions=2, snapshots=snaps)
STATUS = ["converged", "max_iter", "breakdown"]
res = {"snapshots": {}, "tol": args.tol}


def run(sys_, dirs):
    cap = args.maxit if dirs < 2 else args.rrs_maxit
    t0 = time.perf_counter()
    try:
        lam, tr = sys_.solve(tol=args.tol, max_it=cap, directions=dirs)
    except (engine.FetiError, pyoracle.OracleError) as e:
        return {"error": f"{type(e).__name__}: {e}"}, None
    return {"iterations": int(tr["iterations"]), "status": STATUS[tr["status"]],
            "rel_eps": float(tr["eps_final"] / tr["eps0"]), "kept_total": int(np.sum(tr["kept"][1:])),
            "s": round(time.perf_counter() - t0, 3)}, lam


for it in snaps:
    row = {}
    for mname, method in (("tfeti", pb.TFETI), ("fetidp", pb.FETIDP)):
        for sname, scaling in (("multiplicity", pb.MULTIPLICITY), ("k", pb.KSCALING)):
            p = base.replace(densities=st.snapshots[it], method=method, scaling=scaling)
            g = engine.FetiSystem(p)
            o = pyoracle.Oracle(p)
            for dname, dirs in (("single", 0), ("fo", 1), ("rrs", 2)):
                rg, lg = run(g, dirs)
                ro, lo = run(o, dirs)
                e = {"gpu": rg, "oracle": ro}
                if lg is not None and lo is not None:
                    e["lambda_rel_diff"] = float(np.linalg.norm(lg - lo) / max(np.linalg.norm(lo), 1e-300))
                    e["iter_diff"] = rg["iterations"] - ro["iterations"]
                row[f"{mname}_{sname}_{dname}"] = e
                print(it, mname, sname, dname, json.dumps(e), flush=True)
            g.close()
    res["snapshots"][str(it)] = row
with open(args.out, "w") as f:
    json.dump(res, f, indent=1)
print("written", args.out)
