"""K15 A/B: the persistent PCG / FO loop (forced, FETIGPU_PERSIST=1) against the graph loop
(FETIGPU_PERSIST=0).
For each case: iterations, sha1 of lambda and of the eps trace (bit-identity),
and the best-of-N device solve time per variant (grid size / barrier kind).

usage: python tools/persist_ab.py [--reps 3] [--grids 0,16,32,64,148] [--cases C1,C2,...]"""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

CASES = {
    "C1": (pb.config1, 0),
    "C1-fo": (pb.config1, 1),
    "C2": (pb.config2, 0),
    "C2-fo": (pb.config2, 1),
    "C3tf-fo": (lambda: pb.config3(method=0), 1),
    "C3dp-fo": (lambda: pb.config3(method=1), 1),
    "C3dp": (lambda: pb.config3(method=1), 0),
    "C5-fo": (pb.config5, 1),
}


def variants(grids):
    out = [("graph", {"FETIGPU_PERSIST": "0", "FETIGPU_CLUSTER": "0"}), ("default", {})]
    for g in grids:
        if g == 0:
            out.append(("persist-auto", {"FETIGPU_PERSIST": "1", "FETIGPU_CLUSTER": "0"}))
        else:
            out.append((f"grid{g}", {"FETIGPU_PERSIST": "1", "FETIGPU_CLUSTER": "0", "FETIGPU_PERSIST_G": str(g),
                                     "FETIGPU_PERSIST_BAR": "grid"}))
            if g <= 16:
                out.append((f"cluster{g}", {"FETIGPU_PERSIST": "1", "FETIGPU_CLUSTER": "0", "FETIGPU_PERSIST_G": str(g),
                                            "FETIGPU_PERSIST_BAR": "cluster"}))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--grids", default="0,8,16,32,64,148")
    ap.add_argument("--cases", default=",".join(CASES))
    args = ap.parse_args()
    grids = [int(x) for x in args.grids.split(",") if x]
    keys = ("FETIGPU_PERSIST", "FETIGPU_PERSIST_G", "FETIGPU_PERSIST_BAR", "FETIGPU_CLUSTER")
    for name in args.cases.split(","):
        fn, dirs = CASES[name]
        g = engine.FetiSystem(fn())
        ref = None
        for vname, env in variants(grids):
            for k in keys:
                os.environ.pop(k, None)
            os.environ.update(env)
            best, hl = 1e30, None
            for _ in range(args.reps):
                lam, tr = g.solve(tol=1e-6, max_it=5000, directions=dirs)
                best = min(best, tr["solve_ms"])
                h = (tr["iterations"], hashlib.sha1(lam.tobytes()).hexdigest()[:12],
                     hashlib.sha1(tr["eps"].tobytes()).hexdigest()[:12])
                hl = h if hl is None or hl == h else ("NONDET",) + h
            if ref is None:
                ref = hl
            same = "same" if hl == ref else "DIFF"
            print(f"{name:8s} {vname:13s} it={hl[0]} lam={hl[1]} eps={hl[2]} {same} "
                  f"{best:8.2f} ms  {1000 * best / max(1, hl[0]):6.1f} us/it", flush=True)
        for k in keys:
            os.environ.pop(k, None)
        g.close()


if __name__ == "__main__":
    main()
