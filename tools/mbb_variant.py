"""One variant of the modular-MBB study on a SIMP snapshot (bit-identity /
regression probe): SIMP to `--it` with FETI-DP + k + RRS state solves, then
one (method, scaling, directions) solve; prints the compliance history tail,
an F-apply hash and the iteration count."""
import argparse
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb, simp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--it", type=int, default=30)
ap.add_argument("--method", default="tfeti")
ap.add_argument("--scaling", default="multiplicity")
ap.add_argument("--dirs", type=int, default=2)
args = ap.parse_args()
sx, sy, n = 12, 8, 30
types = np.minimum((pb.uniform(2111, sx * sy) * 16).astype(np.int32), 15)
gxn = sx * n + 1
base = pb.Problem(sx, sy, n, np.full((16, n, n), 0.5), types, method=pb.FETIDP, scaling=pb.KSCALING,
                  precond=pb.DIRICHLET, Emin=1e-9, dirichlet=pb.bottom_corner_pins(sx, sy, n),
                  point_loads=[((sy * n) * gxn + (sx * n) // 2, 1, -1.0)], name="mbb")
st = simp.optimize(base, iterations=args.it, volfrac=0.5, directions=2, snapshots=(args.it,))
dens = st.snapshots[args.it]
print("compliance", st.compliance[-2:], "dens hash", hashlib.sha1(np.ascontiguousarray(dens).tobytes()).hexdigest()[:16])
p = base.replace(densities=dens, method=pb.TFETI if args.method == "tfeti" else pb.FETIDP,
                 scaling=pb.MULTIPLICITY if args.scaling == "multiplicity" else pb.KSCALING)
g = engine.FetiSystem(p)
x = np.random.default_rng(7).standard_normal(g.m)
print("F hash", hashlib.sha1(g.apply_F(x).tobytes()).hexdigest()[:16],
      "M hash", hashlib.sha1(g.apply_precond(x).tobytes()).hexdigest()[:16])
lam, tr = g.solve(tol=1e-6, max_it=300, directions=args.dirs)
print("iterations", tr["iterations"], "status", tr["status"], "kept", list(tr["kept"][:6]), list(tr["kept"][-4:]))
