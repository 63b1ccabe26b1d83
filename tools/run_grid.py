"""12-variant comparison grid (SPEC.md:553-577 run_grid):
{T-FETI, FETI-DP} x {multiplicity, k} x {single, FO, RRS} on one problem,
solved on the GPU, one CSV trace per variant with the SPEC's schema
`iter,eps_r,kept_dirs,F_applies,cum_local_solves` plus a summary.csv.

    python tools/run_grid.py --problem grid4x4_inclusion --out grid_out [--oracle]

--oracle also runs the CPU oracle and adds its iteration counts to the summary.
"""
import argparse
import csv
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import problems as pb  # noqa: E402

METHODS = {"tfeti": pb.TFETI, "fetidp": pb.FETIDP}
SCALINGS = {"multiplicity": pb.MULTIPLICITY, "k": pb.KSCALING}
DIRECTIONS = {"single": pb.SINGLE, "fo": pb.FO, "rrs": pb.RRS}
STATUS = ["converged", "max_iter", "breakdown"]


def problem(name, method, scaling, precond, contrast, elems):
    if name in pb.PRESETS:
        kw = dict(method=method, scaling=scaling, precond=precond, contrast=contrast)
        if elems:
            kw["n"] = elems
        return pb.PRESETS[name](**kw)
    return pb.CONFIGS[name]().replace(method=method, scaling=scaling, precond=precond)


def run(args):
    from paper_2111_11728_b200 import engine
    os.makedirs(args.out, exist_ok=True)
    rows = []
    for mname, method in METHODS.items():
        for sname, scaling in SCALINGS.items():
            prob = problem(args.problem, method, scaling, args.precond, args.contrast, args.elems)
            g = engine.FetiSystem(prob)
            o = None
            if args.oracle:
                from oracle import pyoracle
                o = pyoracle.Oracle(prob)
            for dname, dirs in DIRECTIONS.items():
                lam, tr = g.solve(tol=args.tol, max_it=args.maxit, directions=dirs, rel=args.tol_mode == "rel")
                variant = f"{mname}_{sname}_{dname}"
                with open(os.path.join(args.out, variant + ".csv"), "w", newline="") as f:
                    w = csv.writer(f)
                    w.writerow(["iter", "eps_r", "kept_dirs", "F_applies", "cum_local_solves"])
                    for i, e in enumerate(tr["eps"]):
                        # every F column costs one local solve per subdomain
                        w.writerow([i, repr(float(e)), int(tr["kept"][i]), int(tr["f_app"][i]),
                                    int(tr["f_app"][i]) * g.n_sub])
                row = {"variant": variant, "iterations": tr["iterations"], "final_eps_r": tr["eps_final"],
                       "status": STATUS[tr["status"]], "dual_size": g.m, "solve_ms": round(tr["solve_ms"], 3)}
                if o is not None:
                    lo, to = o.solve(tol=args.tol, max_it=args.maxit, directions=dirs, rel=args.tol_mode == "rel")
                    row["oracle_iterations"] = to["iterations"]
                    row["oracle_status"] = STATUS[to["status"]]
                rows.append(row)
                print(row, flush=True)
            g.close()
    with open(os.path.join(args.out, "summary.csv"), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
        w.writeheader()
        w.writerows(rows)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problem", default="grid4x4_inclusion")
    ap.add_argument("--precond", type=int, default=pb.DIRICHLET)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--tol-mode", choices=["abs", "rel"], default="rel")
    ap.add_argument("--maxit", type=int, default=3000)
    ap.add_argument("--contrast", type=float, default=1e4)
    ap.add_argument("--elems", type=int, default=0)
    ap.add_argument("--out", default="grid_out")
    ap.add_argument("--oracle", action="store_true")
    run(ap.parse_args())


if __name__ == "__main__":
    main()
