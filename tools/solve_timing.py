"""Phase timing of tgfem.solve_poisson on the GPU (assembly, boundary, condensation, BiCGSTAB)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05052_b200 import engine, tgfem  # noqa: E402

for kind, ext, div in [("tri3", [1.0, 1.0], [300, 300]), ("tet4", [1.0, 1.0, 1.0], [40, 40, 40])]:
    m = tgfem.generate_grid(kind, ext, div)
    tgfem.solve_poisson(m)
    t = [time.perf_counter()]
    dm = m._device()
    r = m._routing(1, segments=False)
    K, F, _ = engine.assemble(dm, r, diffusion=1.0, sources=[1.0])
    torch.cuda.synchronize(); t.append(time.perf_counter())
    b = m.boundary_nodes
    t.append(time.perf_counter())
    cond = engine.Condensed(r, K, F, b, np.zeros(b.size))
    torch.cuda.synchronize(); t.append(time.perf_counter())
    u, rep = engine.solve_condensed(cond)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(kind, div, "assemble %.1f boundary %.1f condense %.1f solve %.1f ms, iters %d, us/iter %.1f"
          % (d[0], d[1], d[2], d[3], rep["iterations"], d[3] * 1e3 / max(1, rep["iterations"])))

# the public entry, repeated
for kind, ext, div in [("tri3", [1.0, 1.0], [300, 300])]:
    m = tgfem.generate_grid(kind, ext, div)
    for i in range(3):
        t0 = time.perf_counter()
        res = tgfem.solve_poisson(m)
        print("solve_poisson call", i, "%.1f ms" % ((time.perf_counter() - t0) * 1e3), res["iterations"])
