"""Is the GPU-vs-oracle displacement gap on C5 a property of the problem?
Quarter-size C5 (same design law), RRS at tol 1e-8: GPU, double oracle and
refined oracle (long-double residual refinement of every local solve); each
multiplier is scored by the dual energy J = 1/2 l^T F l - d^T l evaluated
with the refined operator (smaller is closer to the true minimiser)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle  # noqa: E402
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

sx, sy = int(sys.argv[1]), int(sys.argv[2])
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-8
prob = pb.config5(sx=sx, sy=sy)
L = pyoracle.lib()
out = {"sx": sx, "sy": sy, "tol": tol}
g = engine.FetiSystem(prob)
lg, tg = g.solve(tol=tol, max_it=300, directions=2)
ug = g.recover(lg)
L.fo_set_refine(0)
o = pyoracle.Oracle(prob)
t0 = time.perf_counter()
lo, to = o.solve(tol=tol, max_it=300, directions=2)
out["oracle_s"] = time.perf_counter() - t0
uo = o.recover(lo)
L.fo_set_refine(1)
r = pyoracle.Oracle(prob)
t0 = time.perf_counter()
lr, tr = r.solve(tol=tol, max_it=300, directions=2)
out["refined_s"] = time.perf_counter() - t0
ur = r.recover(lr)
d, _ = r.rhs()
J = lambda lam: float(0.5 * lam @ r.apply_F(lam) - d @ lam)
res = lambda lam: float(np.linalg.norm(d - r.apply_F(lam)) / np.linalg.norm(d))
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
out.update(m=g.m, iters={"gpu": tg["iterations"], "oracle": to["iterations"], "refined": tr["iterations"]},
           J={"gpu": J(lg), "oracle": J(lo), "refined": J(lr)},
           dual_res={"gpu": res(lg), "oracle": res(lo), "refined": res(lr)},
           u_rel={"gpu_vs_oracle": rel(ug, uo), "gpu_vs_refined": rel(ug, ur), "oracle_vs_refined": rel(uo, ur)},
           lam_rel={"gpu_vs_oracle": rel(lg, lo), "gpu_vs_refined": rel(lg, lr), "oracle_vs_refined": rel(lo, lr)})
print(json.dumps(out))
