"""C4 single-vector F-apply: device time per apply (fetigpu_time_apply, 200
back-to-back applies after warm-up) and sha1 of y (bit-identity probe for
switches such as FETIGPU_L2_PERSIST)."""
import ctypes as C
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

g = engine.FetiSystem(pb.config4())
L, m = engine.lib(), g.m
dx, dy = C.c_void_p(), C.c_void_p()
engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m), C.byref(dx)))
engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m), C.byref(dy)))
xp, yp = C.cast(dx, C.POINTER(C.c_double)), C.cast(dy, C.POINTER(C.c_double))
engine.check(L.fetigpu_fill_random(g.h, xp, C.c_size_t(m), C.c_ulonglong(7)))
ms, n = (C.c_double * 3)(), C.c_int()
engine.check(L.fetigpu_time_apply(g.h, xp, yp, 1, 20, 0, ms, C.byref(n)))
for _ in range(3):
    engine.check(L.fetigpu_time_apply(g.h, xp, yp, 1, 200, 0, ms, C.byref(n)))
    print(f"C4 apply {ms[0] * 1e3:.1f} us, dominant kernel {ms[1] * 1e3:.1f} us ({ms[2]:.3f})", flush=True)
y = np.empty(m)
engine.check(L.fetigpu_memcpy(g.h, y.ctypes.data_as(C.c_void_p), dy, C.c_size_t(8 * m), 2))
engine.check(L.fetigpu_synchronize(g.h))
print("y sha1", hashlib.sha1(y.tobytes()).hexdigest()[:16])
g.close()
