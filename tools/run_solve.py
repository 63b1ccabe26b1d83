"""Full-size solve driver: GPU solve of one BASELINE config (optionally
against the CPU oracle).  python tools/run_solve.py C5 --dirs 2 [--oracle]"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--method", type=int, default=None)
ap.add_argument("--dirs", type=int, default=None)
ap.add_argument("--tol", type=float, default=1e-6)
ap.add_argument("--max-it", type=int, default=1000)
ap.add_argument("--oracle", action="store_true")
ap.add_argument("--recover", action="store_true")
ap.add_argument("--verify", action="store_true",
                help="recompute eps = sqrt(r^T M r), r = P(d - F lambda), from scratch and compare with the trace")
args = ap.parse_args()
fn = pb.CONFIGS[args.config]
prob = fn(method=args.method) if (args.method is not None and args.config == "C3") else fn()
dirs = prob.directions if args.dirs is None else args.dirs
t0 = time.perf_counter()
g = engine.FetiSystem(prob)
tb = time.perf_counter() - t0
st = g.stats()
lam, tr = g.solve(tol=args.tol, max_it=args.max_it, directions=dirs)
out = {"config": args.config, "method": prob.method, "dirs": dirs, "m": g.m, "build_ms": st["build_ms"],
       "build_wall_s": tb, "gpu": {k: tr[k] for k in ("status", "iterations", "f_applies", "solve_ms")},
       "gpu_rel_res": tr["eps_final"] / max(tr["eps0"], 1e-300), "kept_head": tr["kept"][:8].tolist(),
       "eps_rel_head": [float(e / tr["eps0"]) for e in tr["eps"][:16]],
       "phase_ms": dict(zip(["FW", "gram", "pivchol", "compress", "update", "precond", "projZ", "reorth"],
                            [round(x, 2) for x in tr["phase_ms"]]))}
if args.verify:
    d, _ = g.rhs()
    rr = g.project(d - g.apply_F(lam))
    zz = g.apply_precond(rr)
    eps_true = float(np.sqrt(max(rr @ zz, 0.0)))
    out["verify"] = {"eps_trace": tr["eps_final"], "eps_recomputed": eps_true, "eps0": tr["eps0"],
                     "rel_recomputed": eps_true / tr["eps0"], "lambda_norm": float(np.linalg.norm(lam))}
if args.recover:
    t0 = time.perf_counter()
    u = g.recover(lam)
    out["recover_s"] = time.perf_counter() - t0
if args.oracle:
    from oracle import pyoracle
    t0 = time.perf_counter()
    o = pyoracle.Oracle(prob)
    out["oracle_build_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    lo, to = o.solve(tol=args.tol, max_it=args.max_it, directions=dirs)
    out["oracle"] = {"status": to["status"], "iterations": to["iterations"], "solve_s": time.perf_counter() - t0}
    out["oracle_rel_res"] = to["eps_final"] / max(to["eps0"], 1e-300)
    out["lambda_rel_diff"] = float(np.linalg.norm(lam - lo) / max(np.linalg.norm(lo), 1e-300))
    if args.recover:
        uo = o.recover(lo)
        out["u_rel_diff"] = float(np.linalg.norm(u - uo) / np.linalg.norm(uo))
print(json.dumps(out))
