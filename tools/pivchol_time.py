"""Standalone pivoted Cholesky (fetigpu_pivoted_cholesky, Alg. 1 line 9) on a
random PSD n x n matrix: best-of-10 host wall time per call (includes the
2 n^2 x 8-byte host copies) and a hash of (perm, L).  Variant switches are
read once per process (FETIGPU_PIVCHOL_CL1, FETIGPU_PIVCHOL_CLUSTER)."""
import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine  # noqa: E402

for n in [int(x) for x in (sys.argv[1:] or ["128", "512", "640"])]:
    rng = np.random.default_rng(n)
    X = rng.standard_normal((n, n)) * np.logspace(0, -3, n)
    A = X @ X.T
    best = 1e30
    for _ in range(10):
        t0 = time.perf_counter()
        p, L, r = engine.pivoted_cholesky(A)
        best = min(best, time.perf_counter() - t0)
    print(f"n {n}: rank {r}, {best * 1e3:.3f} ms per call, hash "
          f"{hashlib.sha1(p.tobytes() + L.tobytes()).hexdigest()[:12]}", flush=True)
