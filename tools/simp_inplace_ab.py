"""Modular MBB SIMP study (tools/mbb_study.py setup) with the system
re-created per snapshot vs rebuilt in place (fetigpu_rebuild), and with the
warm start: wall time and compliance history of each variant."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import problems as pb, simp  # noqa: E402

sx, sy, n = 12, 8, 30
types = np.minimum((pb.uniform(2111, sx * sy) * 16).astype(np.int32), 15)
gxn = sx * n + 1
base = pb.Problem(sx, sy, n, np.full((16, n, n), 0.5), types, method=pb.FETIDP, scaling=pb.KSCALING,
                  precond=pb.DIRICHLET, Emin=1e-9, dirichlet=pb.bottom_corner_pins(sx, sy, n),
                  point_loads=[((sy * n) * gxn + (sx * n) // 2, 1, -1.0)], name="mbb")
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
res = {}
for name, kw in (("recreate", dict(in_place=False)), ("in_place", dict(in_place=True)),
                 ("in_place_warm", dict(in_place=True, warm=True)), ("recreate_again", dict(in_place=False))):
    t0 = time.perf_counter()
    st = simp.optimize(base, iterations=iters, volfrac=0.5, directions=2, **kw)
    wall = time.perf_counter() - t0
    res[name] = {"wall_s": wall, "compliance": st.compliance,
                 "iterations": [s["iterations"] for s in st.solves],
                 "solve_ms": sum(s["solve_ms"] for s in st.solves)}
    print(name, "wall %.2f s" % wall, "solve %.0f ms" % res[name]["solve_ms"], "c0 %.6f c_end %.6f" %
          (st.compliance[0], st.compliance[-1]), "its", res[name]["iterations"][:10], flush=True)
c0 = np.array(res["recreate"]["compliance"])
for k in res:
    print(k, "max rel compliance diff vs recreate", float(np.max(np.abs(np.array(res[k]["compliance"]) - c0) / c0)))
print(json.dumps(res))
