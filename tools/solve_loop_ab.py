"""Device-resident PCG/FO loop (CUDA-graph while node) vs the host-driven
loop (FETIGPU_HOST_LOOP=1): same iterations, bit-identical lambda, solve time.
    python tools/solve_loop_ab.py"""
import os
import subprocess
import sys
import json

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ".")
    import numpy as np
    from paper_2111_11728_b200 import engine, problems as pb
    out = {}
    for name, fn, dirs in (("C1", pb.config1, 0), ("C2-fo", pb.config2, 1), ("C3-tfeti", lambda: pb.config3(method=0), 1),
                           ("C3-fetidp", lambda: pb.config3(method=1), 1), ("C4-cg", pb.config4, 0)):
        g = engine.FetiSystem(fn())
        g.solve(tol=1e-6, max_it=3000, directions=dirs)                   # warm
        lam, tr = g.solve(tol=1e-6, max_it=3000, directions=dirs)
        out[name] = {"iterations": tr["iterations"], "solve_ms": round(tr["solve_ms"], 2),
                     "lam_sum": float(np.sum(lam)), "eps_last": float(tr["eps"][-1])}
        g.close()
    print(json.dumps(out))
    sys.exit(0)
res = {}
for mode, env in (("device", {}), ("host", {"FETIGPU_HOST_LOOP": "1"})):
    r = subprocess.run([sys.executable, __file__, "--child"], capture_output=True, text=True,
                       env={**os.environ, **env})
    res[mode] = json.loads(r.stdout.strip().splitlines()[-1])
for k in res["device"]:
    d, h = res["device"][k], res["host"][k]
    print(f"{k:10s} its {d['iterations']:4d}/{h['iterations']:4d}  device {d['solve_ms']:8.2f} ms  host {h['solve_ms']:8.2f} ms"
          f"  identical {d['lam_sum'] == h['lam_sum'] and d['eps_last'] == h['eps_last']}")
