"""Run one C2/C2a assembly with TGK_FUSED_TRACE and summarise the per-block phase timeline."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
w = sys.argv[1] if len(sys.argv) > 1 else "c2a"
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/trace.bin"
import torch
from paper_2602_05052_b200 import engine, tgfem
m = tgfem.generate_grid("tet4", [1, 1, 1], [100, 100, 100])
dm = engine.DeviceMesh("tet4", m.nodes, m.elements)
r = engine.Routing(dm, 1)
kw = dict(sources=[1.0], with_mass=(w == "c2"))
for _ in range(3):
    engine.assemble(dm, r, **kw)
torch.cuda.synchronize()
os.environ["TGK_FUSED_TRACE"] = out
engine.assemble(dm, r, **kw)
torch.cuda.synchronize()
t = np.fromfile(out, dtype=np.int64).reshape(-1, 8)
start, pro, a, b, epi, sm, nch, end = t.T
span = end.max() - start.min()
print(f"{w}: blocks {len(t)}, kernel span {span} cycles = {span/1.965e3:.1f} us @1.965GHz")
dur = end - start
print(f"block duration mean {dur.mean():.0f} cyc; prologue {pro.mean():.0f}, phaseA {a.mean():.0f} ({a.mean()/nch.mean():.0f}/chunk), phaseB {b.mean():.0f} ({b.mean()/nch.mean():.0f}/chunk), epilogue {epi.mean():.0f}; chunks/block {nch.mean():.2f}")
per_sm = np.bincount(sm, minlength=148)
print(f"blocks per SM: min {per_sm.min()} max {per_sm.max()}; sum of block durations per SM / span = {np.bincount(sm, weights=dur).mean()/span:.2f} (avg concurrency)")
