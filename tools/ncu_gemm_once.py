"""One DMMA GEMM launch for ncu (dla.cuh default tile): M x N x K NN."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine  # noqa: E402

M, N, K = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (2048, 2048, 8192)))
engine.dla_time_gemm(M, N, K, False, False, reps=1)
