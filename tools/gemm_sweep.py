"""DMMA GEMM tile-configuration sweep (csrc/dla.cuh, FETIGPU_GEMM_CFG):
python tools/gemm_sweep.py  (configurations of dla.cuh gemm_cfg)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1:   # child: one config
    sys.path.insert(0, ROOT)
    from paper_2111_11728_b200 import engine
    cfg = sys.argv[1]
    out = {"cfg": int(cfg)}
    for (M, N, K, ta, tb) in ((2048, 2048, 2048, 0, 0), (2048, 2048, 16384, 0, 0), (4096, 4096, 4096, 0, 0),
                              (2048, 4224, 4224, 0, 0), (8192, 2048, 2048, 0, 1), (2048, 2048, 8192, 1, 1)):
        ms = engine.dla_time_gemm(M, N, K, bool(ta), bool(tb), reps=5)
        out[f"{M}x{N}x{K}{'T' if ta else 'N'}{'T' if tb else 'N'}"] = round(2.0 * M * N * K / (ms * 1e-3) / 1e12, 2)
    print(json.dumps(out), flush=True)
else:
    env = dict(os.environ)
    for cfg in range(8):
        env["FETIGPU_GEMM_CFG"] = str(cfg)
        subprocess.run([sys.executable, __file__, str(cfg)], env=env)
