"""GPU vs oracle: max |W^T F W - I| over the stored directions of FO / RRS
solves (fetigpu_set_check / fo_set_check) on the desk problems."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402
from oracle import pyoracle as po  # noqa: E402

po.lib().fo_set_threads(os.cpu_count() or 1)
po.set_check(True)
DESK = {
    "C1s": lambda: pb.config1(sx=4, sy=2, n=8),
    "C2s": lambda: pb.config2(sx=4, sy=2, n=8),
    "C3tf_s": lambda: pb.config3(method=0, sx=4, sy=2, n=8),
    "C3dp_s": lambda: pb.config3(method=1, sx=4, sy=2, n=8),
    "C4s": lambda: pb.config4(sx=4, sy=2, n=8),
    "C5s": lambda: pb.config5(sx=4, sy=2, n=12, n_designs=3),
}
for name, fn in DESK.items():
    p = fn()
    o = po.Oracle(p)
    g = engine.FetiSystem(p)
    g.set_check(True)
    for d, store in ((1, "auto"), (2, "explicit"), (2, "implicit")):
        if store == "implicit" and p.method == 0:
            continue
        g.set_rrs_store(store)
        _, tg = g.solve(tol=1e-8, max_it=500, directions=d)
        eg = g.check_result()
        _, to = o.solve(tol=1e-8, max_it=500, directions=d)
        eo = po.check_result()
        print(f"{name:7s} dirs {d} {store:8s} its gpu {tg['iterations']:3d} oracle {to['iterations']:3d}  "
              f"gpu err {eg[0]:.2e} (n {eg[1]})  oracle err {eo[0]:.2e} (n {eo[1]})", flush=True)
    g.close()
