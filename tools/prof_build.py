"""C4 device build only (profiling driver)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_11728_b200 import engine, problems as pb  # noqa: E402

g = engine.FetiSystem(pb.config4())
s = g.stats()
print("build_ms", s["build_ms"], "nd_ms", s["nd_ms"], "slot_ms", s["slot_ms"])
