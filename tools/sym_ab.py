"""Same-process A/B of the C4 F-apply's dominant kernel: one context per
environment setting (the switches are read at build), timed alternately so
clock / power drift hits every variant alike.  Usage:
  python tools/sym_ab.py "FETIGPU_SYM_TMA=0" "FETIGPU_SYM_FLAGS=0" "" ..."""
import ctypes as C
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

variants = sys.argv[1:] or ["FETIGPU_SYM_TMA=0", ""]
prob = pb.config4()
L = engine.lib()
ctxs = []
for v in variants:
    kv = dict(x.split("=", 1) for x in v.split(",") if x)
    os.environ.update(kv)
    g = engine.FetiSystem(prob)
    for k in kv:
        del os.environ[k]
    m = g.m
    dx, dy = C.c_void_p(), C.c_void_p()
    engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m), C.byref(dx)))
    engine.check(L.fetigpu_device_alloc(g.h, C.c_size_t(8 * m), C.byref(dy)))
    xp, yp = C.cast(dx, C.POINTER(C.c_double)), C.cast(dy, C.POINTER(C.c_double))
    engine.check(L.fetigpu_fill_random(g.h, xp, C.c_size_t(m), C.c_ulonglong(7)))
    ctxs.append((v or "default", g, xp, yp, dy, [], []))
ms, n = (C.c_double * 3)(), C.c_int()
for rnd in range(int(os.environ.get("ROUNDS", "6"))):
    for name, g, xp, yp, dy, ta, tk in ctxs:
        engine.check(L.fetigpu_time_apply(g.h, xp, yp, 1, 60, 0, ms, C.byref(n)))
        if rnd:
            ta.append(ms[0] * 1e3)
            tk.append(ms[1] * 1e3)
for name, g, xp, yp, dy, ta, tk in ctxs:
    y = np.empty(g.m)
    engine.check(L.fetigpu_memcpy(g.h, y.ctypes.data_as(C.c_void_p), dy, C.c_size_t(8 * g.m), 2))
    engine.check(L.fetigpu_synchronize(g.h))
    st = g.stats()
    print(f"{name:40s} apply min {min(ta):6.1f} med {sorted(ta)[len(ta) // 2]:6.1f} us | kernel min {min(tk):6.1f} "
          f"med {sorted(tk)[len(tk) // 2]:6.1f} us = {st['main_kernel_bytes'] / min(tk) / 1e3:5.0f} GB/s | kernel "
          f"{st['apply_kernel']} ring {st['apply_ring']} | sha1 {hashlib.sha1(y.tobytes()).hexdigest()[:12]}", flush=True)
    g.close()
