"""Profiling driver for the K5 block apply: C4 density law on a reduced
module grid, k columns, a few block applies (used under ncu)."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sx", type=int, default=16)
ap.add_argument("--sy", type=int, default=8)
ap.add_argument("--k", type=int, default=512)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
g = engine.FetiSystem(pb.config4(sx=args.sx, sy=args.sy))
L = engine.lib()
m, k = g.m, args.k
dW, dQ = C.c_void_p(), C.c_void_p()
engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m * k), C.byref(dW)))
engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m * k), C.byref(dQ)))
Wp, Qp = C.cast(dW, C.POINTER(C.c_double)), C.cast(dQ, C.POINTER(C.c_double))
engine.check(L.fetigpu_fill_random(g.h, Wp, C.c_size_t(m * k), C.c_ulonglong(5)))
ms = (C.c_double * 1)()
engine.check(L.fetigpu_time_apply_block(g.h, Wp, Qp, k, args.reps, ms))
st = g.stats()
tf = st["op_flops_per_col"] * k / (ms[0] * 1e-3) / 1e12
print(f"m={m} k={k} block apply {ms[0]:.3f} ms  {tf:.2f} TFLOP/s")
