"""C4 create + device build (profiling driver): wall time of fetigpu_create
(host setup) and fetigpu_build, `--reps` times in one process.
FETIGPU_TIMING=1 prints the phase marks."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=1)
args = ap.parse_args()
prob = pb.config4()
for r in range(args.reps):
    t0 = time.perf_counter()
    g = engine.FetiSystem(prob, build=False)
    t1 = time.perf_counter()
    g.build()
    t2 = time.perf_counter()
    s = g.stats()
    print(f"rep {r}: create_s {t1 - t0:.3f} build_wall_s {t2 - t1:.3f} build_ms {s['build_ms']:.1f} "
          f"nd_ms {s['nd_ms']:.1f} slot_ms {s['slot_ms']:.1f}", flush=True)
    g.close()
