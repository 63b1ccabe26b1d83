"""C4 single-vector F-apply, a few launches only: the target of the ncu
captures of the dominant kernel (k_sym_gemv_tma / k_sym_gemv_scatter)."""
import ctypes as C
import os
import sys

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
engine.check(L.fetigpu_time_apply(g.h, xp, yp, 1, int(os.environ.get("REPS", "4")), 0, ms, C.byref(n)))
print(f"C4 apply {ms[0] * 1e3:.1f} us, dominant kernel {ms[1] * 1e3:.1f} us; apply_kernel "
      f"{g.stats()['apply_kernel']} ring {g.stats()['apply_ring']}", flush=True)
g.close()
