"""One seed of tests/test_gpu_fuzz.py in detail: the problem drawn, and for FO
and RRS what the GPU, the oracle and the perturbed oracle do (status,
iterations, eps trace, kept counts or the exception raised).
python tools/fuzz_seed.py 1636"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_fuzz as tf  # noqa: E402
from oracle import pyoracle as om  # noqa: E402
from paper_2111_11728_b200 import engine  # noqa: E402

seed = int(sys.argv[1])
prob = tf.random_problem(seed)
print("problem", prob.sx, "x", prob.sy, "modules of", prob.n, "| method", prob.method, "scaling", prob.scaling,
      "precond", prob.precond, "| E0", prob.E0, "Emin", prob.Emin, "p", prob.p, "nu", prob.nu)
g = engine.FetiSystem(prob)
o = om.Oracle(prob)
r = om.Oracle(tf.perturbed(prob, seed))
print("m", g.m)
for dirs in (1, 2):
    for name, s in (("gpu", g), ("oracle", o), ("pert", r)):
        try:
            lam, t = s.solve(tol=1e-8, max_it=2000 if dirs == 1 else 300, directions=dirs)
            e = np.asarray(t["eps"]) / max(t["eps0"], 1e-300)
            print(f"dirs {dirs} {name:6s} status {t['status']} its {t['iterations']} eps/eps0 "
                  f"{np.array2string(e[:14], precision=2)} kept {list(np.asarray(t.get('kept', []))[:14])}")
        except Exception as ex:  # noqa: BLE001
            print(f"dirs {dirs} {name:6s} raised {type(ex).__name__}: {str(ex)[:160]}")
g.close()
