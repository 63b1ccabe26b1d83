"""Writes the golden fixtures used by tests/.

spec_examples.json: the known answers on this path that the reference's
SPEC.md states (file:line cited per entry) and SURVEY.md Appendix B derives
from the reference code; transcribed here, not computed.

oracle_small.npz: outputs of the CPU oracle on small seeded cases (the
reference itself does not build here), so the GPU tests can
also run against a frozen fixture.  Regenerate with
    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

SPEC = {
    "simp_modulus": {"cite": "SPEC.md:110-112",
                     "cases": [[1.0, 1.0], [0.0, 1e-9], [0.5, 0.125000000875]]},
    "q4_row0_nu03": {"cite": "SURVEY.md App. B (fem.cpp:44-84)",
                     "values": [0.494505494505494, 0.178571428571429, -0.302197802197802,
                                -0.013736263736264, -0.247252747252747, -0.178571428571429,
                                0.054945054945055, 0.013736263736264]},
    "q4_eigs_nu03": {"cite": "SURVEY.md App. B / SPEC.md:121",
                     "nonzero": [0.4945054945, 0.4945054945, 0.7692307692, 0.7692307692, 1.4285714286]},
    "fixing_dofs": {"cite": "SURVEY.md App. B (linalg.cpp:146-175)",
                    "n": [16, 32, 48, 64], "rule": "{0, 1, 2n(n+1)}"},
    "mbb_geometry": {"cite": "SPEC.md:197,611; PAPER.md:411; SURVEY.md 6 (10,972 = T-FETI interface rows; "
                             "the two pinned corner nodes add 4 Dirichlet rows)",
                     "total_dofs": 184512, "tfeti_iface": 10972, "tfeti_m": 10976, "fetidp_m": 9976,
                     "fetidp_nc": 234},
    "corners": {"cite": "SPEC.md:231-233", "cases": [[2, 2, 18], [1, 2, 12], [12, 8, 234]]},
    "config_sizes": {"cite": "SURVEY.md App. A",
                     "C1": {"m": 418, "iface": 350}, "C2": {"m": 3224, "nc": 80},
                     "C3": {"tfeti_m": 15736, "fetidp_m": 14384, "nc": 302},
                     "C4": {"m": 504000, "nc": 4224}, "C5": {"m": 91744, "nc": 1118}},
    "pivoted_cholesky": {"cite": "SPEC.md:49-51",
                         "identity3": {"rank": 3, "perm": [0, 1, 2]},
                         "vvT_122": {"rank": 1, "first_pivot": 1}},
    "k_scaling": {"cite": "SPEC.md:249-251",
                  "pair": [1.0, 1e6, 1e6 / (1.0 + 1e6)],
                  "cross4": [[1.0, 1.0, 1e3, 1e3], 1e3 / (1.0 + 1.0 + 1e3 + 1e3)]},
}


def main():
    with open(os.path.join(HERE, "spec_examples.json"), "w") as f:
        json.dump(SPEC, f, indent=1)
    from oracle import pyoracle
    from paper_2111_11728_b200 import problems as pb
    out = {}
    for name, prob in (("c1s", pb.config1(sx=4, sy=2, n=8)), ("c2s", pb.config2(sx=4, sy=2, n=8))):
        o = pyoracle.Oracle(prob)
        X = np.random.default_rng(2024).standard_normal((o.m, 2))
        out[name + "_x"] = X
        out[name + "_Fx"] = np.stack([o.apply_F(X[:, c]) for c in range(2)], axis=1)
        out[name + "_d"] = o.rhs()[0]
        for dirs in (1, 2):
            lam, tr = o.solve(tol=1e-8, max_it=500, directions=dirs)
            out[f"{name}_iters{dirs}"] = np.array(tr["iterations"])
            out[f"{name}_kept{dirs}"] = tr["kept"]
        out[name + "_u"] = o.recover(lam)
    np.savez_compressed(os.path.join(HERE, "oracle_small.npz"), **out)


if __name__ == "__main__":
    main()
