"""Benchmark of the fused P1 assembly hot path (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--workload c2] [--impl reference]

A step is one tg::assemble-equivalent pass (Map fused with Reduce) over the
workload's mesh.  Default workload = BASELINE.json configs[1] ("C2"): 3D Poisson
P1 tet stiffness + mass + load on the unit-cube Kuhn grid 100^3 (6,000,000
tets), fp64.  Under torchrun each rank owns a z-slab of 100 cube layers of a
100 x 100 x (100 N) grid (row-owning partition, halo elements recomputed, no
data-path collective) -> weak scaling, results bitwise identical to one GPU.

value     = assembled elements / s over all ranks, inputs resident in HBM
            (device time, CUDA events on the launching stream, max over ranks)
e2e       = the same metric through the host-buffer C-ABI call (tgk_assemble):
            per step H2D of the mesh (pinned host -> device) and D2H of K, M, F
roofline  = algorithmic bytes / measured step time vs the
            measured HBM copy peak (MEASURED_PEAKS.json)
cpu_baseline = the reference library (oracle/_ref, compiled from the reference
            sources) on the box's host cores, bounded sample, rank 0 only
--impl reference runs that reference CPU implementation as the timed arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "assembled elements/sec and achieved HBM GB/s (% roofline) at 1/2/4/8 B200 vs CPU ref"
UNIT = "elements/s"

WORKLOADS = {
    # name: (kind, divisions per rank, problem kwargs, description)
    "c2": ("tet4", (100, 100, 100), dict(sources=[1.0], with_mass=True),
           "C2: 3D Poisson P1 tet K+M+F, unit-cube Kuhn 100^3 (6M tets), fp64, Q=4"),
    "c2a": ("tet4", (100, 100, 100), dict(sources=[1.0]),
            "C2a: 3D Poisson P1 tet K+F, unit-cube Kuhn 100^3 (6M tets), fp64, Q=1"),
    "c1": ("tri3", (256, 256), dict(sources=[1.0]),
           "C1: 2D Poisson P1 K+F, unit square 256x256 (131k tris), fp64"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def alg_bytes(kind, E, Nn, nnz, with_mass, has_f):
    """SURVEY.md 8(d) algorithmic bytes: connectivity E*k*4 + coordinates N*d*8
    + slot map E*k^2*4 + CSR values nnz*8 per matrix + load N*8."""
    k = 4 if kind == "tet4" else 3
    d = 3 if kind == "tet4" else 2
    b = E * k * 4 + Nn * d * 8 + E * k * k * 4 + nnz * 8 * (2 if with_mass else 1)
    if has_f:
        b += Nn * 8
    compulsory = b - E * k * k * 4
    return b, compulsory


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def slab_mesh(kind, div, rank, world):
    """Rank `rank`'s z-slab of the global grid div[0] x div[1] x (div[2]*world):
    cube layers [z0-1, z1) (one halo layer below for rank > 0), coordinates and
    connectivity bit-identical to the global tg::generate_grid arrays.
    Returns (nodes, elems, owned node range [lo, hi), global element offset)."""
    from paper_2602_05052_b200 import tgfem
    if world == 1:
        m = tgfem.generate_grid(kind, [1.0] * len(div), list(div))
        return m.nodes, m.elements, 0, m.node_count(), 0
    nx, ny, nzr = div
    nz = nzr * world
    z0, z1 = rank * nzr, (rank + 1) * nzr
    zl = z0 - 1 if rank > 0 else 0
    # the global grid restricted to cube layers [zl, z1): generate the full-size
    # index pattern on a local grid and shift (Kuhn split is translation invariant)
    loc = tgfem.generate_grid(kind, [1.0, 1.0, 1.0], [nx, ny, z1 - zl])
    hz = 1.0 / nz
    nodes = loc.nodes.copy()
    layer = (nx + 1) * (ny + 1)
    kz = np.repeat(np.arange(zl, z1 + 1, dtype=np.int64), layer)
    nodes[:, 2] = kz * hz                 # same expression as mesh.cpp:139 (kz * hz)
    nodes[:, 0] = loc.nodes[:, 0]
    nodes[:, 1] = loc.nodes[:, 1]
    own_lo = (z0 - zl) * layer
    own_hi = (z1 - zl) * layer + (layer if rank == world - 1 else 0)
    return nodes, loc.elements, own_lo, own_hi, zl * nx * ny * 6


def cpu_reference_time(kind, divs, problem_kw, steps, warmup, threads=0):
    """Reference tg::assemble (oracle/_ref) on the host: returns (E, seconds list)."""
    from oracle import ref
    ref.set_threads(threads)
    m = ref.Mesh.grid(kind, [1.0] * len(divs), list(divs))
    r = ref.Routing(m, 1)
    times = []
    for i in range(warmup + steps):
        *_, secs = ref.assemble(m, r, timing=True, **problem_kw)
        if i >= warmup:
            times.append(secs)
    return m.E, times


def effective_cores():
    return os.cpu_count() or 1


def run_reference(args):
    """--impl reference: the reference's CPU implementation (compiled from its sources)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    kind, div, kw, desc = WORKLOADS[args.workload]
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtgref.so not built"}))
        return
    sample = tuple(args.ref_sample) if args.ref_sample else ((50, 50, 50) if kind == "tet4" else div)
    E, times = cpu_reference_time(kind, sample, kw, args.steps, args.warmup)
    mean = statistics.mean(times)
    value = E / mean
    cores = ref.thread_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc, "sample": f"{kind} Kuhn {'x'.join(map(str, sample))} ({E} elements) "
                   "per step (bounded sample of the workload)", "parallelism": f"{cores} host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"tg::assemble on {kind} {'x'.join(map(str, sample))}, {E} elements, "
                                   f"mean of {args.steps}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="exact", choices=["exact", "fast"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample", type=int, nargs="*", default=None)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    from paper_2602_05052_b200 import engine
    from paper_2602_05052_b200 import _native as N

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    kind, div, kw, desc = WORKLOADS[args.workload]
    if kind != "tet4" and world > 1:
        raise SystemExit("multi-GPU slabs are defined for the tet4 workloads")

    # ---------------- setup (not timed): mesh, routing, fused plan
    t0 = time.time()
    nodes, elems, own_lo, own_hi, _ = slab_mesh(kind, div, rank, world)
    mesh = engine.DeviceMesh(kind, nodes, elems)
    routing = engine.Routing(mesh, 1)
    if world > 1:
        N.check(N.lib().tgk_routing_set_owned_rows(routing._h, own_lo, own_hi))
    import ctypes as C
    nb, nh, nrec, pbytes = (C.c_int64() for _ in range(4))
    R = 128 if kw.get("with_mass") else 256  # rows per block of the fused kernel variant
    N.check(N.lib().tgk_routing_plan_stats(routing._h, R, C.byref(nb), C.byref(nh), C.byref(nrec),
                                           C.byref(pbytes)))
    setup_s = time.time() - t0
    E_own = 6 * div[0] * div[1] * div[2] if kind == "tet4" else 2 * div[0] * div[1]
    with_mass = kw.get("with_mass", False)
    has_f = bool(kw.get("sources"))
    p, keep = engine.make_problem("poisson", mode=args.mode, **kw)
    dev = torch.device("cuda", local_rank)
    K = torch.empty(routing.nnz, dtype=torch.float64, device=dev)
    F = torch.empty(routing.N, dtype=torch.float64, device=dev)
    M = torch.empty(routing.nnz, dtype=torch.float64, device=dev) if with_mass else None
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    ptr = lambda t: None if t is None else C.c_void_p(t.data_ptr())  # noqa: E731

    def step():
        N.check(N.lib().tgk_assemble_async_d(C.byref(p), mesh._h, routing._h, ptr(K), ptr(F), ptr(M),
                                             ptr(bad), sp))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if int(bad.item()) != -1:
        raise SystemExit(f"element {bad.item()} has non-positive Jacobian determinant")

    # ---------------- timed region (device time)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    total_E = E_own * world
    value = total_E / (ms_per_step * 1e-3)

    # ---------------- e2e through the host-buffer C-ABI call
    e2e = None
    if args.e2e_steps > 0:
        h_nodes = torch.from_numpy(np.ascontiguousarray(nodes)).pin_memory()
        h_elems = torch.from_numpy(np.ascontiguousarray(elems)).pin_memory()
        hK = torch.empty(routing.nnz, dtype=torch.float64).pin_memory()
        hF = torch.empty(routing.N, dtype=torch.float64).pin_memory()
        hM = torch.empty(routing.nnz, dtype=torch.float64).pin_memory() if with_mass else None
        hp = N.Problem()
        C.memmove(C.addressof(hp), C.addressof(p), C.sizeof(p))
        hptr = lambda t: None if t is None else C.c_void_p(t.data_ptr())  # noqa: E731

        def e2e_step():
            N.check(N.lib().tgk_mesh_upload(mesh._h, hptr(h_nodes), hptr(h_elems), sp))
            N.check(N.lib().tgk_assemble(C.byref(hp), mesh._h, routing._h, hptr(hK), hptr(hF), hptr(hM)))

        e2e_step()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - w0) / args.e2e_steps
        if dist:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        h2d = h_nodes.numel() * 8 + h_elems.numel() * 8
        d2h = hK.numel() * 8 + hF.numel() * 8 + (hM.numel() * 8 if hM is not None else 0)
        e2e = {"value": total_E / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3,
               "path": "tgk_mesh_upload + tgk_assemble (host buffers, pinned)"}

    # ---------------- roofline of the fused kernel (the step is one fused launch)
    Nn = nodes.shape[0]
    own_nodes = own_hi - own_lo
    offs = routing.host_arrays(slot_of=False, segments=False)["offsets"]
    nnz_own = int(offs[own_hi] - offs[own_lo])
    ab, comp = alg_bytes(kind, E_own, own_nodes, nnz_own, with_mass, has_f)
    peak, peak_src = peaks()
    achieved = ab / (ms_per_step * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(f"{args.workload}_{args.mode}")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ref
            if ref.available():
                sample = (40, 40, 40) if kind == "tet4" else div
                Es, times = cpu_reference_time(kind, sample, kw, 3, 1)
                cpu = {"value": Es / min(times), "unit": UNIT, "cores": ref.thread_count(),
                       "kind": "reference",
                       "sample": f"tg::assemble (oracle/_ref, reference sources) on {kind} Kuhn "
                                 f"{'x'.join(map(str, sample))} = {Es} elements, best of 3"}
            else:
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                       "sample": "oracle/_ref/libtgref.so not present"}
        except Exception as exc:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"error: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "elements_per_gpu": E_own, "nnz_per_gpu": nnz_own,
                       "mode": args.mode,
                       "parallelism": "single GPU" if world == 1 else
                       f"{world} row-owning z-slabs (halo recompute, no data-path collective)",
                       "l2": "inputs larger than L2 (working set ~1 GB vs 126 MB L2)",
                       "fused_plan": {"rows_per_block": R, "blocks": nb.value, "halo_elements": nh.value,
                                      "recompute_factor": nh.value / max(1, elems.shape[0]),
                                      "records": nrec.value, "bytes": pbytes.value},
                       "setup_s": setup_s},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "alg_bytes": ab,
                         "compulsory_bytes": comp, "peak_source": peak_src,
                         "kernel": "k_fused_scalar (one launch per step)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
