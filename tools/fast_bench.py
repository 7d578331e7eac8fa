"""Quick device timing of the fused assembly modes (exact vs fast) on the bench
configurations; CUDA events on the launching stream, median of N after warm-up.
Usage: python tools/fast_bench.py [c2a c2 c1 ...] [--reps 20]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import port  # noqa: E402
from paper_2602_05052_b200 import engine  # noqa: E402

CFG = {
    "c1": ("tri3", [256, 256], dict(sources=[1.0]), 11.6e6),
    "c2a": ("tet4", [100, 100, 100], dict(sources=[1.0]), 634.66e6),
    "c2": ("tet4", [100, 100, 100], dict(sources=[1.0], with_mass=True), 756.34e6),
    "c5": ("tet4", [256, 256, 256], dict(sources=[1.0]), 10.62e9),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", nargs="*", default=["c2a", "c2", "c1"])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--modes", default="fast,exact")
    a = ap.parse_args()
    peak = 6537.6
    for name in a.cfg:
        kind, div, kw, alg = CFG[name]
        nodes, elems = port.generate_grid(kind, [1.0] * len(div), div)
        m = engine.DeviceMesh(kind, nodes, elems)
        r = engine.Routing(m, 1)
        E = elems.shape[0]
        K = torch.empty(r.nnz, dtype=torch.float64, device="cuda")
        F = torch.empty(r.N, dtype=torch.float64, device="cuda")
        M = torch.empty(r.nnz, dtype=torch.float64, device="cuda") if kw.get("with_mass") else None
        for mode in a.modes.split(","):
            engine.assemble(m, r, mode=mode, out=(K, F, M), **kw)  # plan build
            torch.cuda.synchronize()
            ts = []
            for i in range(a.reps + 3):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(400000)  # back up the queue: host overhead stays off the clock
                s.record()
                engine.assemble(m, r, mode=mode, out=(K, F, M), **kw)
                e.record()
                e.synchronize()
                if i >= 3:
                    ts.append(s.elapsed_time(e))
            t = float(np.median(ts))
            print(f"{name:4s} {mode:5s} E={E} median {t*1e3:8.1f} us  best {min(ts)*1e3:8.1f} us  "
                  f"{E/t/1e6:7.2f} G elem/s  frac {alg/(t*1e-3)/1e9/peak:.3f}", flush=True)


if __name__ == "__main__":
    main()
