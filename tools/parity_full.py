"""Full-size GPU vs oracle solve parity for one config (one-off evidence run).
python tools/parity_full.py C5 > profiles/r01_parity_C5.json"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle  # noqa: E402
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

name = sys.argv[1]
max_it = int(sys.argv[2]) if len(sys.argv) > 2 else 200
prob = pb.CONFIGS[name]()
out = {"config": name, "method": prob.method, "directions": prob.directions, "tol": 1e-6,
       "host_cores": os.cpu_count()}
g = engine.FetiSystem(prob)
st = g.stats()
lg, tg = g.solve(tol=1e-6, max_it=max_it, directions=prob.directions)
ug = g.recover(lg)
out["gpu"] = {"build_ms": st["build_ms"], "solve_ms": tg["solve_ms"], "iterations": tg["iterations"],
              "status": tg["status"], "kept": tg["kept"].tolist(), "rel_res": tg["eps_final"] / tg["eps0"],
              "phase_ms": tg["phase_ms"]}
t0 = time.perf_counter()
o = pyoracle.Oracle(prob)
tb = time.perf_counter() - t0
t0 = time.perf_counter()
lo, to = o.solve(tol=1e-6, max_it=max_it, directions=prob.directions)
ts = time.perf_counter() - t0
uo = o.recover(lo)
out["oracle"] = {"build_s": tb, "solve_s": ts, "iterations": to["iterations"], "status": to["status"],
                 "kept": to["kept"].tolist(), "rel_res": to["eps_final"] / to["eps0"]}
out["u_rel_l2_gpu_vs_oracle"] = float(np.linalg.norm(ug - uo) / np.linalg.norm(uo))
out["iteration_diff"] = tg["iterations"] - to["iterations"]
print(json.dumps(out))
