"""C4 block apply Q = F W (k columns) timing: mean of `--reps` back-to-back
device applies after one warm-up (fetigpu_time_apply_block)."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=2048)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--hash", action="store_true", help="also print sha1 of Q (bit-identity probe)")
args = ap.parse_args()
g = engine.FetiSystem(pb.config4())
L, m, k = engine.lib(), g.m, args.k
dW, dQ = C.c_void_p(), C.c_void_p()
engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m * k), C.byref(dW)))
engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m * k), C.byref(dQ)))
Wp, Qp = C.cast(dW, C.POINTER(C.c_double)), C.cast(dQ, C.POINTER(C.c_double))
engine.check(L.fetigpu_fill_random(g.h, Wp, C.c_size_t(m * k), C.c_ulonglong(99)))
ms = (C.c_double * 1)()
engine.check(L.fetigpu_time_apply_block(g.h, Wp, Qp, k, 1, ms))
engine.check(L.fetigpu_time_apply_block(g.h, Wp, Qp, k, args.reps, ms))
print(f"k {k}: {ms[0]:.2f} ms per block apply")
if args.hash:
    import hashlib
    import numpy as np
    q = np.empty(m * k)
    engine.check(L.fetigpu_memcpy(g.h, q.ctypes.data_as(C.c_void_p), dQ, C.c_size_t(8 * m * k), 2))
    print("Q sha1", hashlib.sha1(q.tobytes()).hexdigest()[:16])
