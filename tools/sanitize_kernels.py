"""One small launch of every hot kernel, for compute-sanitizer:

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_kernels.py

k_fast_scalar (K16 / KS32 / S16 formats, nodal load), k_fast_elast (constant
and per-element fields), k_fused_scalar (R = 64,
128, 256), k_fused_elast2, k_batched_entries, k_adjoint_groups, the
materialised Stage I/II drop-ins; each result is checked against the oracle
so a silent corruption under the tool also fails."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import port  # noqa: E402
from paper_2602_05052_b200 import engine, meshgen  # noqa: E402


def close(a, b, what, exact=True):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    s = np.abs(b).max() if b.size else 0.0
    err = np.abs(a - b).max() if b.size else 0.0
    ok = err == 0.0 if exact else err <= 1e-12 * s + 1e-14 * s
    print(f"  {what:40s} max|d| {err:.2e} {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        raise SystemExit(f"{what}: mismatch")


def main():
    torch.cuda.set_device(0)
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [6, 5, 7])
    E, Nn = elems.shape[0], nodes.shape[0]
    m = engine.DeviceMesh("tet4", nodes, elems)
    r = engine.Routing(m, 1)
    pr = port.Routing(Nn, port.dofmap("tet4", elems, 1))
    rho = 0.5 + np.random.default_rng(3).random(E)
    nod = 0.5 + np.random.default_rng(4).random(Nn)
    cases = [dict(sources=[1.0]), dict(sources=[1.0], with_mass=True),
             dict(diffusion=("nodal", nod), sources=[("nodal", nod)]),
             dict(problem="mass", diffusion=("element", rho))]
    print("k_fast_scalar", flush=True)
    for kw in cases:
        kw = dict(kw)
        problem = kw.pop("problem", "poisson")
        K, F, M = engine.assemble(m, r, kind=problem, mode="fast", **kw)
        Kr, Fr, Mr = port.assemble("tet4", nodes, elems, pr, problem=problem, **kw)
        close(K, Kr, f"fast {problem} {sorted(kw)} K", exact=False)
        close(F, Fr, "  F", exact=False)
    print("k_fused_scalar", flush=True)
    for R in ["64", "128", "256"]:
        os.environ["TGK_FUSED_R"] = R
        r2 = engine.Routing(m, 1)
        K, F, M = engine.assemble(m, r2, sources=[1.0], with_mass=True, diffusion=("element", rho))
        Kr, Fr, Mr = port.assemble("tet4", nodes, elems, pr, sources=[1.0], with_mass=True,
                                   diffusion=("element", rho))
        close(K, Kr, f"exact R={R} K")
        close(M, Mr, f"exact R={R} M")
    os.environ.pop("TGK_FUSED_R", None)
    print("k_fused_elast2", flush=True)
    rv = engine.Routing(m, 3)
    prv = port.Routing(Nn * 3, port.dofmap("tet4", elems, 3))
    K, F, _ = engine.assemble(m, rv, kind="elasticity", lam=0.5769230769230769, mu=0.38461538461538464,
                              sources=[1.0, 1.0, 1.0])
    Kr, Fr, _ = port.assemble("tet4", nodes, elems, prv, problem="elasticity", lam=0.5769230769230769,
                              mu=0.38461538461538464, sources=[1.0, 1.0, 1.0])
    close(K, Kr, "elasticity K")
    close(F, Fr, "elasticity F")
    print("k_fast_elast", flush=True)
    lam_e = 0.3 + np.random.default_rng(5).random(E)
    for kw in [dict(lam=0.5769230769230769, mu=0.38461538461538464, sources=[1.0, 1.0, 1.0]),
               dict(lam=("element", lam_e), mu=("element", rho), sources=[("element", rho), 1.0, 0.5])]:
        K, F, _ = engine.assemble(m, rv, kind="elasticity", mode="fast", **kw)
        Kr, Fr, _ = port.assemble("tet4", nodes, elems, prv, problem="elasticity", **kw)
        close(K, Kr, f"fast elasticity {'element' if isinstance(kw['lam'], tuple) else 'const'} K", exact=False)
        close(F, Fr, "  F", exact=False)
    print("k_batched_entries / k_adjoint_groups", flush=True)
    tn, te = meshgen.unstructured_tri(24)
    tm = engine.DeviceMesh("tri3", tn, te)
    tr = engine.Routing(tm, 1)
    tpr = port.Routing(tn.shape[0], port.dofmap("tri3", te, 1))
    B = 5
    rb = meshgen.batch_fields(B, te.shape[0])
    Kb, Fb = engine.assemble_batched(tm, tr, rb, source=1.0)
    for b in range(B):
        Kr, _, _ = port.assemble("tri3", tn, te, tpr, diffusion=("element", rb[b]), sources=[1.0])
        close(Kb[b], Kr, f"batched field {b}")
    lam = np.stack([np.random.default_rng(20 + b).random(tn.shape[0]) - 0.5 for b in range(B)])
    U = np.stack([np.random.default_rng(30 + b).random(tn.shape[0]) - 0.5 for b in range(B)])
    adj = engine.adjoint_gather(tm, tr, lam, U, degree=1)
    K0 = port.local("tri3", tn, te, 1, port.DIFFUSION, np.ones(te.shape[0]))
    dm = port.dofmap("tri3", te, 1)
    for b in range(B):
        close(adj[b], port.adjoint_gather(dm, K0, lam[b], U[b]), f"adjoint field {b}")
    torch.cuda.synchronize()
    print("all kernels ran clean", flush=True)


if __name__ == "__main__":
    main()
