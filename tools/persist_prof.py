"""K15 phase profile: build with -DFG_PERSIST_PROF (libfetigpu_prof.so), run one
persistent solve per case and print the mean time between consecutive grid
barriers (CTA 0's %globaltimer after each barrier), phase by phase.
usage: FETIGPU_LIB=.../libfetigpu_prof.so python tools/persist_prof.py C1 C2 ..."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine  # noqa: E402
from persist_ab import CASES  # noqa: E402

lib = engine.lib()
lib.fetigpu_pprof.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * (64 * 1024))()
for name in sys.argv[1:]:
    fn, dirs = CASES[name]
    g = engine.FetiSystem(fn())
    g.solve(tol=1e-6, max_it=5000, directions=dirs)
    lib.fetigpu_pprof(buf, 64 * 1024)
    lam, tr = g.solve(tol=1e-6, max_it=5000, directions=dirs)
    n = lib.fetigpu_pprof(buf, 64 * 1024)
    t = np.array(buf[:n], dtype=np.float64)
    it = tr["iterations"]
    per = int(round(n / max(1, it))) if it else 0
    print(f"{name}: {it} iterations, {n} stamps, {per} barriers/iteration, "
          f"{(t[-1] - t[0]) / 1e3 / max(1, it):.2f} us/iteration", flush=True)
    if per and it > 4:
        d = np.diff(t[per - 1:per - 1 + per * (it - 2) + 1]).reshape(it - 2, per)
        print("  us per phase (between barrier k-1 and k):", " ".join(f"{x / 1e3:.2f}" for x in d.mean(axis=0)))
    g.close()
