import sys, os, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2111_11728_b200 import engine, problems as pb
from oracle import pyoracle as po
for name, p in [('C3dp_s', pb.config3(method=1, sx=4, sy=2, n=8)), ('C3tf_s', pb.config3(method=0, sx=4, sy=2, n=8)), ('C4s', pb.config4(sx=4, sy=2, n=8))]:
    g = engine.FetiSystem(p); o = po.Oracle(p)
    rng = np.random.default_rng(0)
    d, _ = g.rhs()
    # low-energy directions: preconditioned residual-like vectors
    X = [g.apply_precond(rng.standard_normal(g.m)) for _ in range(2)] + [rng.standard_normal(g.m) for _ in range(2)]
    if p.method == 0: X = [g.project(x) for x in X]
    for lab, F in (('gpu', g.apply_F), ('oracle', o.apply_F)):
        out = []
        for a, b in ((0, 1), (2, 3), (0, 2)):
            x, y = X[a], X[b]
            Fx, Fy = F(x), F(y)
            out.append(abs(x @ Fy - y @ Fx) / np.sqrt(abs(x @ Fx) * abs(y @ Fy)))
        print(name, lab, ['%.2e' % v for v in out])
    g.close()
