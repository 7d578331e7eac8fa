"""Kernel-time census of one solve_poisson call (run under ncu --metrics gpu__time_duration.sum)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05052_b200 import tgfem  # noqa: E402

m = tgfem.generate_grid("tri3", [1.0, 1.0], [300, 300])
r = tgfem.solve_poisson(m)
print("iters", r["iterations"])
