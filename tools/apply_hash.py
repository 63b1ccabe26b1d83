"""Bit-identity probe for kernel variants: sha1 of F x (fixed seeded x) and of
the recovered displacements for a few configurations."""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

cfgs = {"C1": pb.config1, "C2": pb.config2, "C3dp": lambda: pb.config3(method=pb.FETIDP), "C5": pb.config5, "C4": pb.config4}
for name in (sys.argv[1:] or list(cfgs)):
    g = engine.FetiSystem(cfgs[name]())
    x = np.random.default_rng(7).standard_normal(g.m)
    y = g.apply_F(x)
    z = g.apply_precond(x)
    print(name, hashlib.sha1(y.tobytes()).hexdigest()[:16], hashlib.sha1(z.tobytes()).hexdigest()[:16], flush=True)
    g.close()
