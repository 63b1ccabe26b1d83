"""Full-size GPU vs oracle solve parity for one config (one-off evidence run).
python tools/parity_full.py C5 > profiles/r01_parity_C5.json
python tools/parity_full.py C4 400 1e-6 1   (max_it, tol, directions override: FO)"""
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
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-6
prob = pb.CONFIGS[name]()
if len(sys.argv) > 4:  # directions override (C4's RRS exceeds one GPU: run it with FO / single)
    prob = prob.replace(directions=int(sys.argv[4]))
out = {"config": name, "method": prob.method, "directions": prob.directions, "tol": tol,
       "host_cores": os.cpu_count()}
g = engine.FetiSystem(prob)
st = g.stats()
lg, tg = g.solve(tol=tol, max_it=max_it, directions=prob.directions)
ug = g.recover(lg)
out["gpu"] = {"build_ms": st["build_ms"], "solve_ms": tg["solve_ms"], "iterations": tg["iterations"],
              "status": tg["status"], "kept": tg["kept"].tolist(), "rel_res": tg["eps_final"] / tg["eps0"],
              "phase_ms": tg["phase_ms"]}
t0 = time.perf_counter()
o = pyoracle.Oracle(prob)
tb = time.perf_counter() - t0
t0 = time.perf_counter()
lo, to = o.solve(tol=tol, max_it=max_it, directions=prob.directions)
ts = time.perf_counter() - t0
uo = o.recover(lo)
out["oracle"] = {"build_s": tb, "solve_s": ts, "iterations": to["iterations"], "status": to["status"],
                 "kept": to["kept"].tolist(), "rel_res": to["eps_final"] / to["eps0"]}
out["u_rel_l2_gpu_vs_oracle"] = float(np.linalg.norm(ug - uo) / np.linalg.norm(uo))
# energy norm ||u_g - u_o||_K / ||u_o||_K with the oracle's assembled K^s
num = den = 0.0
for s_ in range(o.n_sub):
    du = ug[s_] - uo[s_]
    num += du @ o.local_apply(s_, du)
    den += uo[s_] @ o.local_apply(s_, uo[s_])
out["u_rel_energy_gpu_vs_oracle"] = float(np.sqrt(max(num, 0.0) / den))
# L2 restricted to nodes that touch a solid element (rho > 0.5)
n = prob.n
mask = np.zeros((o.n_sub, o.local_dofs), bool)
for d in range(prob.densities.shape[0]):  # per design: nodes touching a solid element
    solid = prob.densities[d] > 0.5
    node = np.zeros((n + 1, n + 1), bool)
    node[:-1, :-1] |= solid
    node[:-1, 1:] |= solid
    node[1:, :-1] |= solid
    node[1:, 1:] |= solid
    dof = np.repeat(node.reshape(-1), 2)
    mask[np.asarray(prob.module_type) == d] = dof
out["u_rel_l2_solid_nodes"] = float(np.linalg.norm((ug - uo)[mask]) / np.linalg.norm(uo[mask]))
out["iteration_diff"] = tg["iterations"] - to["iterations"]
print(json.dumps(out))
