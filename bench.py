"""Benchmark of the fused P1 assembly hot path (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--workload c2] [--impl reference]
                    [--dist-mode exchange|halo]

A step is one tg::assemble-equivalent pass (Map fused with Reduce) over the
workload's mesh.  Workloads (BASELINE.json configs):

  c2   (default, configs[1]) 3D Poisson P1 tet K+M+F, unit-cube Kuhn 100^3 per GPU
       (6,000,000 tets), fp64, Q=4; weak scaling: rank r owns a z-slab of 100
       cube layers of a 100 x 100 x (100 N) grid
  c2a  the same mesh, K+F at Q=1 (the north-star target case)
  c1   (configs[0]) 2D Poisson P1 K+F, unit square 256x256 (131k tris)
  c3   (configs[2]) 3D linear elasticity (3x3 blocks), Kuhn 100^3 per GPU, K+F
  c4   (configs[3]) 256 per-element coefficient fields on the 2D unstructured
       C4 mesh (131k tris): batched K_b (+F) and the adjoint transpose gather;
       fields sharded across GPUs (strong scaling)
  c5   (configs[4]) Kuhn 256^3 (100.7M tets) split into N z-slabs (strong scaling)

Multi-GPU (tet4 scalar workloads): --dist-mode exchange (default) assembles
each rank's own elements and sums the interface node layer over NCCL
(paper_2602_05052_b200/dist.py); --dist-mode halo recomputes the halo layer
instead (no data-path collective, bitwise equal to one GPU).

value     = elements/s over all ranks, inputs resident in HBM (device time of
            the whole step, CUDA events on the launching stream, max over ranks)
e2e       = the same metric through the public C ABI with host buffers:
            H2D of the mesh from pinned memory, assembly, D2H of the outputs
roofline  = SURVEY.md 8(d) algorithmic bytes of the dominant kernel per launch
            / that kernel's event-timed duration, vs MEASURED_PEAKS.json
cpu_baseline = the reference library (oracle/_ref, compiled from the reference
            sources) on the box's host cores, bounded sample, rank 0 at N=1
--impl reference runs that reference CPU implementation as the timed arm.
"""
from __future__ import annotations

import argparse
import ctypes as C
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

# name: (kind, divisions per rank or global, problem kwargs, description, scaling)
WORKLOADS = {
    "c2": ("tet4", (100, 100, 100), dict(sources=[1.0], with_mass=True),
           "C2: 3D Poisson P1 tet K+M+F, unit-cube Kuhn 100^3 (6M tets) per GPU, fp64, Q=4", "weak"),
    "c2a": ("tet4", (100, 100, 100), dict(sources=[1.0]),
            "C2a: 3D Poisson P1 tet K+F, unit-cube Kuhn 100^3 (6M tets) per GPU, fp64, Q=1", "weak"),
    "c1": ("tri3", (256, 256), dict(sources=[1.0]),
           "C1: 2D Poisson P1 K+F, unit square 256x256 (131k tris), fp64, Q=1", "weak"),
    "c3": ("tet4", (100, 100, 100), None,
           "C3: 3D linear elasticity P1 tets (3x3 blocks), Kuhn 100^3 (6M tets) per GPU, E=1 nu=0.3, "
           "body force (1,1,1), K+F, fp64", "weak"),
    "c4": ("tri3", (256, 256), None,
           "C4: 256 per-element coefficient fields on the 2D unstructured C4 mesh (131,072 tris, "
           "jittered + random diagonals + permuted), batched K_b + F, with the adjoint transpose gather, fp64",
           "strong"),
    "c5": ("tet4", (256, 256, 256), dict(sources=[1.0]),
           "C5: 3D Poisson P1 tet K+F, Kuhn 256^3 (100.7M tets) partitioned into z-slabs, fp64, Q=1", "strong"),
    "rm": ("tri3", (1000, 500), None,
           "RM: the reduce_matrix drop-in (routing.cpp:109-132) on the reference's published reduction workload, "
           "TRI3 1000x500 over [1, 0.5] (E = 1e6; acceptance.cpp:677-689, 12.25 ms in proj/test_output.txt:24), fp64",
           "weak"),
}
C4_FIELDS = 256
LAME = (0.3 / (1.3 * 0.4), 1.0 / (2 * 1.3))  # lame_from_young(1, 0.3) (batch.cpp:353-357)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def alg_bytes(kind, E, Nn, nnz, with_mass, has_f, comps=1, vbytes=8):
    """SURVEY.md 8(d) algorithmic bytes: connectivity E*k*4 + coordinates N*d*8
    + slot map E*k^2*4 + CSR values nnz*8 per matrix + load N_dof*8
    (+ scalar row_ptr (N+1)*4 for vector problems); vbytes=4 for the fp32 outputs."""
    k = 4 if kind == "tet4" else 3
    d = 3 if kind == "tet4" else 2
    b = E * k * 4 + Nn * d * 8 + E * k * k * 4 + nnz * vbytes * (2 if with_mass else 1)
    if has_f:
        b += Nn * comps * vbytes
    if comps > 1:
        b += (Nn + 1) * 4
    return b, b - E * k * k * 4


def ncu_traffic(workload, kernel=None):
    """dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel per launch, from the
    committed ncu --set full capture of this workload (profiles/traffic.json) when it captured
    `kernel` (the one this run times), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            e = json.load(f).get(workload, {})
        if kernel and kernel not in e.get("kernel", ""):
            return None
        return e.get("bytes")
    except Exception:
        return None


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (NVML, ~1 ms
    period; nvidia-smi fallback)."""

    def __init__(self, index):
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._ready = threading.Event()  # set once the sampler is initialised (NVML init can take ~100 ms)
        self._t = None

    def _run_nvml(self):
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        names = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "sw_power_cap": 0x4}
        self._ready.set()
        while not self._stop.is_set():
            self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            self.mx.append(mx)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            for n, bit in names.items():
                if r & bit:
                    self.reasons.add(n)
            time.sleep(0.001)

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        self._ready.set()
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip().split(",")
                self.sm.append(float(out[0]))
                self.mx.append(float(out[1]))
                for i, n in enumerate(names):
                    if out[2 + i].strip().lower().startswith("active"):
                        self.reasons.add(n)
            except Exception:
                pass
            self._stop.wait(0.05)

    def _run(self):
        try:
            self._run_nvml()
        except Exception:
            self._run_smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._ready.wait(timeout=10)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx),
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


# ------------------------------------------------------------------ reference (CPU) arm
def cpu_reference_time(kind, divs, problem_kw, steps, warmup, threads=0):
    """Reference tg::assemble (oracle/_ref) on the host: returns (E, seconds list)."""
    from oracle import ref
    ref.set_threads(threads)
    m = ref.Mesh.grid(kind, [1.0] * len(divs), list(divs))
    r = ref.Routing(m, 3 if problem_kw.get("problem") == "elasticity" else 1)
    times = []
    for i in range(warmup + steps):
        *_, secs = ref.assemble(m, r, timing=True, **problem_kw)
        if i >= warmup:
            times.append(secs)
    return m.E, times


def cpu_reference_rm(steps, warmup, threads=0):
    """reduce_matrix of the reference (routing.cpp:109-132) on the RM workload, the unit-coefficient
    local stiffness of the reference's own Stage I as input (acceptance.cpp:677-689)."""
    from oracle import ref
    ref.set_threads(threads)
    m = ref.Mesh.grid("tri3", [1.0, 0.5], [1000, 500])
    r = ref.Routing(m, 1)
    K_local = ref.local(m, 1, 0, np.ones(m.E))
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        r.reduce_matrix(K_local)
        if i >= warmup:
            times.append(time.perf_counter() - t0)
    return m.E, times


def cpu_reference_c4(steps, warmup, fields=4, threads=0):
    """B x (per-element evaluate + local_stiffness_diffusion + reduce_matrix) (+F) of the reference on
    the C4 mesh, `fields` fields per step (a bounded sample of the 256-field batch)."""
    from oracle import ref
    from paper_2602_05052_b200 import meshgen
    ref.set_threads(threads)
    nodes, elems = meshgen.unstructured_tri(256)
    m = ref.Mesh.from_arrays("tri3", nodes, elems)
    r = ref.Routing(m, 1)
    rho = meshgen.batch_fields(fields, elems.shape[0])
    times = []
    for i in range(warmup + steps):
        t = 0.0
        for b in range(fields):
            *_, secs = ref.assemble(m, r, diffusion=("element", rho[b]), sources=[1.0] if b == 0 else [],
                                    timing=True)
            t += secs
        if i >= warmup:
            times.append(t)
    return elems.shape[0] * fields, times


def ref_problem_kw(workload):
    kind, div, kw, desc, _ = WORKLOADS[workload]
    if workload == "c3":
        return dict(problem="elasticity", lam=LAME[0], mu=LAME[1], sources=[1.0, 1.0, 1.0])
    return dict(kw or {})


# Reference-arm / cpu_baseline meshes: the workload's own configuration for
# C1, C2 and C2a (same-config ratio; ~4 s per CPU step at 100^3 on 16
# cores), bounded samples for C3 (the reference routing of the 3-DoF 100^3
# mesh takes minutes single-threaded) and C5 (100.7M tets need > 100 GB of
# host RAM in the reference's materialised Stage I).
REF_SAMPLE = {"c2": (100, 100, 100), "c2a": (100, 100, 100), "c1": (256, 256), "c3": (30, 30, 30),
              "c5": (64, 64, 64), "rm": (1000, 500)}


def e2e_pipelined(ctx, N, L, engine, kind, nodes, elems, p, with_mass, h_nodes, h_elems, fK, fF, fM, steps,
                  comps=1):
    """Seconds per step of repeated host-to-host assembly with the copies of consecutive steps overlapped
    (two device buffer sets, upload / compute / download streams); every step still moves its inputs
    H2D and its results D2H.  None if it cannot run."""
    torch = ctx.torch
    try:
        meshes = [engine.DeviceMesh(kind, nodes, elems) for _ in range(2)]
        routs = [engine.Routing(m, comps) for m in meshes]
        nnz, n = routs[0].nnz, routs[0].N
        bufs = [dict(K=torch.empty(nnz, dtype=torch.float64, device=ctx.dev),
                     F=torch.empty(n, dtype=torch.float64, device=ctx.dev),
                     M=torch.empty(nnz, dtype=torch.float64, device=ctx.dev) if with_mass else None,
                     bad=torch.full((1,), -1, dtype=torch.int64, device=ctx.dev)) for _ in range(2)]
        s_up, s_cmp, s_dn = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        ev_up = [torch.cuda.Event() for _ in range(2)]
        ev_cmp = [torch.cuda.Event() for _ in range(2)]
        ev_dn = [torch.cuda.Event() for _ in range(2)]

        def step(i):
            j = i & 1
            b = bufs[j]
            s_up.wait_event(ev_cmp[j])  # step i-2's assembly no longer reads mesh j
            N.check(L.tgk_mesh_upload_async(meshes[j]._h, ptr(h_nodes), ptr(h_elems), C.c_void_p(s_up.cuda_stream)))
            ev_up[j].record(s_up)
            s_cmp.wait_event(ev_up[j])
            s_cmp.wait_event(ev_dn[j])  # step i-2's download of buffer set j is done
            if comps == 1:
                N.check(L.tgk_assemble_async_d(C.byref(p), meshes[j]._h, routs[j]._h, ptr(b["K"]), ptr(b["F"]),
                                               ptr(b["M"]), ptr(b["bad"]), C.c_void_p(s_cmp.cuda_stream)))
            else:  # vector problems: the device entry (checks its flags on its stream)
                N.check(L.tgk_assemble_d(C.byref(p), meshes[j]._h, routs[j]._h, ptr(b["K"]), ptr(b["F"]), None,
                                         C.c_void_p(s_cmp.cuda_stream)))
            ev_cmp[j].record(s_cmp)
            s_dn.wait_event(ev_cmp[j])
            with torch.cuda.stream(s_dn):
                fK.copy_(b["K"], non_blocking=True)
                fF.copy_(b["F"], non_blocking=True)
                if fM is not None:
                    fM.copy_(b["M"], non_blocking=True)
            ev_dn[j].record(s_dn)

        for i in range(4):  # plans, certification, warm-up
            step(i)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for i in range(steps):
            step(i)
        torch.cuda.synchronize()
        for m in meshes:  # the uploads' range checks (accumulated on the device), inside the timed region
            N.check(L.tgk_mesh_upload_check(m._h))
        dt = (time.perf_counter() - w0) / steps
        if any(int(b["bad"].item()) != -1 for b in bufs):
            return None
        return dt
    except Exception:
        return None


def c1_graph_time(ctx, launch, steps):
    """C1: the same assembly captured `steps` times into one CUDA
    graph on a side stream and replayed; ms per assembly from CUDA events.  The
    launch-overhead-free time of a small mesh (reported in config, not as value)."""
    torch = ctx.torch
    try:
        gs = torch.cuda.Stream()
        sp = C.c_void_p(gs.cuda_stream)
        with torch.cuda.stream(gs):
            for _ in range(3):
                launch(sp)
        gs.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            for _ in range(steps):
                launch(sp)
        g.replay()
        gs.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        with torch.cuda.stream(gs):
            e0.record(gs)
            for _ in range(reps):
                g.replay()
            e1.record(gs)
        gs.synchronize()
        return {"ms_per_step": e0.elapsed_time(e1) / (reps * steps), "assemblies_per_graph": steps}
    except Exception as exc:  # capture unsupported here: say why, keep the bench line
        return {"error": str(exc)[:200]}


def run_reference(args):
    """--impl reference: the reference's CPU implementation (compiled from its sources)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    kind, div, kw, desc, scaling = WORKLOADS[args.workload]
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtgref.so not built"}))
        return
    if args.workload == "c4":
        E, times = cpu_reference_c4(args.steps, args.warmup)
        sample = f"C4 mesh, 4 of the 256 coefficient fields per step ({E} element-fields)"
    elif args.workload == "rm":
        E, times = cpu_reference_rm(args.steps, args.warmup)
        sample = f"reduce_matrix on tri3 1000x500 ({E} elements) per step (the workload itself)"
    else:
        smp = tuple(args.ref_sample) if args.ref_sample else REF_SAMPLE[args.workload]
        E, times = cpu_reference_time(kind, smp, ref_problem_kw(args.workload), args.steps, args.warmup)
        sample = f"{kind} Kuhn {'x'.join(map(str, smp))} ({E} elements) per step"
    mean = statistics.mean(times)
    value = E / mean
    cores = ref.thread_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc, "sample": sample + " (bounded sample of the workload)",
                   "parallelism": f"{cores} host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"tg::assemble, {sample}, mean of {args.steps}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def cpu_baseline_line(workload):
    try:
        from oracle import ref
        if not ref.available():
            return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                    "sample": "oracle/_ref/libtgref.so not present"}
        if workload == "c4":
            E, times = cpu_reference_c4(2, 1)
            sample = f"tg::assemble per field on the C4 mesh, 4 fields ({E} element-fields), best of 2"
        elif workload == "rm":
            E, times = cpu_reference_rm(5, 1)
            sample = f"reduce_matrix (oracle/_ref) on tri3 1000x500 = {E} elements, best of 5"
        else:
            kind = WORKLOADS[workload][0]
            smp = REF_SAMPLE.get(workload)
            E, times = cpu_reference_time(kind, smp, ref_problem_kw(workload), 3, 1)
            sample = (f"tg::assemble (oracle/_ref, reference sources) on {kind} Kuhn {'x'.join(map(str, smp))} "
                      f"= {E} elements, best of 3")
        return {"value": E / min(times), "unit": UNIT, "cores": ref.thread_count(), "kind": "reference",
                "sample": sample}
    except Exception as exc:  # reported, never fatal
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"error: {exc}"}


# ------------------------------------------------------------------ our arm
class Ctx:
    def __init__(self, args):
        import torch
        self.torch = torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local_rank)
        self.dev = torch.device("cuda", self.local_rank)
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group("nccl", device_id=self.dev)
            self.dist = dist
        self.stream = torch.cuda.current_stream()
        self.sp = C.c_void_p(self.stream.cuda_stream)

    def barrier(self):
        if self.dist:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, x):
        if not self.dist:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def timed(self, step, steps, clocks=None):
        """Device time (ms) of `steps` calls of step(), CUDA events on the stream, max over ranks."""
        torch = self.torch
        self.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(self.stream)
        for _ in range(steps):
            step()
        ev1.record(self.stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        self.barrier()
        return self.max_over_ranks(ms)


def ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def ramp(step, ctx, seconds=0.3):
    """Untimed extra warm-up until `seconds` of back-to-back GPU work: after a
    long host-side setup (plan builds) the SM clocks have dropped, and a few
    sub-millisecond warm-up steps do not bring them back before the timed region."""
    t0 = time.perf_counter()
    n = 1
    while time.perf_counter() - t0 < seconds:
        for _ in range(n):
            step()
        ctx.torch.cuda.synchronize()
        n = min(2 * n, 256)


def run_scalar(args, ctx, N):
    """c1 / c2 / c2a / c5: fused scalar assembly; tet4 meshes split into z-slabs."""
    torch = ctx.torch
    from paper_2602_05052_b200 import dist as D, engine, tgfem
    kind, div, kw, desc, scaling = WORKLOADS[args.workload]
    world, rank = ctx.world, ctx.rank
    t0 = time.time()
    if kind == "tet4":
        per = tuple(div) if scaling == "weak" else (div[0], div[1], div[2] // world)
        if scaling == "strong" and div[2] % world:
            raise SystemExit(f"{args.workload}: {div[2]} cube layers do not split into {world} slabs")
        s = D.slab(per, rank, world, args.dist_mode if world > 1 else "halo")
        nodes, elems = D.slab_mesh(s)
        parallelism = ("single GPU" if world == 1 else
                       f"{world} row-owning z-slabs, " + ("own elements + NCCL interface-layer exchange"
                                                          if s.mode == "exchange" else
                                                          "halo recompute (no data-path collective)"))
    else:
        if world > 1:
            parallelism = f"{world} independent replicas (2D mesh not partitioned)"
        else:
            parallelism = "single GPU"
        m = tgfem.generate_grid(kind, [1.0] * len(div), list(div))
        nodes, elems, s = m.nodes, m.elements, None
    mesh = engine.DeviceMesh(kind, nodes, elems)
    routing = engine.Routing(mesh, 1)
    L = N.lib()
    if s is not None and world > 1:
        N.check(L.tgk_routing_set_owned_rows(routing._h, s.own_lo, s.calc_hi))
        if s.mode == "exchange":
            N.check(L.tgk_routing_set_element_range(routing._h, s.elem_lo, s.elem_hi))
    nb, nh, nrec, pbytes = (C.c_int64() for _ in range(4))
    # rows per block of the fused kernel (fused.cu fused_rows_per_block: 64 below 4 x 128 x #SMs rows)
    n_rows_own = (s.calc_hi - s.own_lo) if (s is not None and world > 1) else nodes.shape[0]
    R_plan = 64 if (kw.get("with_mass") or
                    n_rows_own < 128 * 4 * torch.cuda.get_device_properties(ctx.dev).multi_processor_count) else 128
    N.check(L.tgk_routing_plan_stats(routing._h, R_plan, C.byref(nb), C.byref(nh), C.byref(nrec), C.byref(pbytes)))
    setup_s = time.time() - t0
    with_mass = kw.get("with_mass", False)
    has_f = bool(kw.get("sources"))
    p, keep = engine.make_problem("poisson", mode=args.mode, **kw)
    f32 = args.precision == "f32"
    vdt = torch.float32 if f32 else torch.float64
    K = torch.zeros(routing.nnz, dtype=vdt, device=ctx.dev)
    F = torch.zeros(routing.N, dtype=vdt, device=ctx.dev)
    M = torch.zeros(routing.nnz, dtype=vdt, device=ctx.dev) if with_mass else None
    bad = torch.empty(1, dtype=torch.int64, device=ctx.dev)
    row_ptr = routing.host_arrays(slot_of=False, segments=False)["offsets"]
    exchange = s is not None and world > 1 and s.mode == "exchange"
    ev_k0, ev_k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def kernel():
        if f32:
            N.check(L.tgk_assemble_f32_d(C.byref(p), mesh._h, routing._h, ptr(K), ptr(F), ptr(M), ptr(bad), ctx.sp))
        else:
            N.check(L.tgk_assemble_async_d(C.byref(p), mesh._h, routing._h, ptr(K), ptr(F), ptr(M), ptr(bad), ctx.sp))

    def step():
        kernel()
        if exchange:
            D.exchange_interface(K, F, row_ptr, s, D.gpu_combine, ctx.dist)
            if M is not None:
                z = torch.zeros_like(F)
                D.exchange_interface(M, z, row_ptr, s, D.gpu_combine, ctx.dist)

    bad.fill_(-1)
    for _ in range(args.warmup):
        step()
    ramp(step, ctx)
    torch.cuda.synchronize()
    if int(bad.item()) != -1:
        raise SystemExit(f"element {bad.item()} has non-positive Jacobian determinant")
    with ClockSampler(ctx.local_rank) as clocks:
        ms = ctx.timed(step, args.steps)
        # kernel-only duration (roofline): event pair around the fused launches
        # alone, median of three passes of `steps` launches
        trials = []
        for _ in range(3):
            ctx.barrier()
            ev_k0.record(ctx.stream)
            for _ in range(args.steps):
                kernel()
            ev_k1.record(ctx.stream)
            torch.cuda.synchronize()
            trials.append(ev_k0.elapsed_time(ev_k1) / args.steps)
    ms_kernel = sorted(trials)[1]
    ms_per_step = ms / args.steps
    other = None  # the other fp64 mode's kernel time on the same inputs (both modes reported)
    if not f32:
        q, keep_q = engine.make_problem("poisson", mode="exact" if args.mode == "fast" else "fast", **kw)
        qK, qF = torch.empty_like(K), torch.empty_like(F)
        qM = torch.empty_like(M) if M is not None else None

        def kernel_other():
            N.check(L.tgk_assemble_async_d(C.byref(q), mesh._h, routing._h, ptr(qK), ptr(qF), ptr(qM), ptr(bad),
                                           ctx.sp))
        for _ in range(2):
            kernel_other()
        ctx.barrier()
        ev_k0.record(ctx.stream)
        for _ in range(args.steps):
            kernel_other()
        ev_k1.record(ctx.stream)
        torch.cuda.synchronize()
        other = ev_k0.elapsed_time(ev_k1) / args.steps
        del qK, qF, qM
    graph = None
    if args.workload == "c1" and not f32 and world == 1:
        graph = c1_graph_time(ctx, lambda sp: N.check(L.tgk_assemble_async_d(
            C.byref(p), mesh._h, routing._h, ptr(K), ptr(F), ptr(M), ptr(bad), sp)), args.steps)
    if kind == "tet4":
        E_own = 6 * s.div[0] * s.div[1] * s.div[2]
        own_rows = (s.own_lo, s.own_hi)
    else:
        E_own = elems.shape[0]
        own_rows = (0, nodes.shape[0])
    total_E = E_own * world
    value = total_E / (ms_per_step * 1e-3)

    # e2e through the C ABI with host buffers
    e2e = None
    if args.e2e_steps > 0 and not f32:
        h_nodes = torch.from_numpy(np.ascontiguousarray(nodes)).pin_memory()
        h_elems = torch.from_numpy(np.ascontiguousarray(elems)).pin_memory()
        o0, o1 = own_rows
        kk0, kk1 = int(row_ptr[o0]), int(row_ptr[o1])
        hK = torch.empty(kk1 - kk0, dtype=torch.float64).pin_memory()
        hF = torch.empty(o1 - o0, dtype=torch.float64).pin_memory()
        hM = torch.empty(kk1 - kk0, dtype=torch.float64).pin_memory() if with_mass else None
        if world == 1:
            fK = torch.empty(routing.nnz, dtype=torch.float64).pin_memory()
            fF = torch.empty(routing.N, dtype=torch.float64).pin_memory()
            fM = torch.empty(routing.nnz, dtype=torch.float64).pin_memory() if with_mass else None
            hp = N.Problem()
            C.memmove(C.addressof(hp), C.addressof(p), C.sizeof(p))

            def e2e_step():  # host buffers in, host buffers out: tgk_assemble copies inside
                N.check(L.tgk_mesh_upload(mesh._h, ptr(h_nodes), ptr(h_elems), ctx.sp))
                N.check(L.tgk_assemble(C.byref(hp), mesh._h, routing._h, ptr(fK), ptr(fF), ptr(fM)))
            d2h = (fK.numel() + fF.numel() + (fM.numel() if fM is not None else 0)) * 8
            path = "tgk_mesh_upload + tgk_assemble (host buffers, pinned)"
        else:
            def e2e_step():
                N.check(L.tgk_mesh_upload(mesh._h, ptr(h_nodes), ptr(h_elems), ctx.sp))
                step()
                hK.copy_(K[kk0:kk1], non_blocking=True)
                hF.copy_(F[o0:o1], non_blocking=True)
                if hM is not None:
                    hM.copy_(M[kk0:kk1], non_blocking=True)
                torch.cuda.current_stream().synchronize()
            d2h = (hK.numel() + hF.numel() + (hM.numel() if hM is not None else 0)) * 8
            path = "tgk_mesh_upload + tgk_assemble_async_d + NCCL exchange + D2H of owned rows (pinned)"
        e2e_step()
        ctx.barrier()
        w0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = ctx.max_over_ranks((time.perf_counter() - w0) / args.e2e_steps)
        e2e = {"value": total_E / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h_nodes.numel() * 8 + h_elems.numel() * 8),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3, "path": path}
        if world == 1:
            pipe = e2e_pipelined(ctx, N, L, engine, kind, nodes, elems, p, with_mass, h_nodes, h_elems, fK, fF, fM,
                                 args.e2e_steps)
            if pipe is not None:
                e2e["sync_drop_in"] = {"value": e2e["value"], "ms_per_step": e2e["ms_per_step"], "path": path}
                e2e.update(value=total_E / pipe, ms_per_step=pipe * 1e3,
                           path="repeated assembly through the public async API: per step tgk_mesh_upload_async "
                                "(pinned H2D of nodes + int64 connectivity, narrowed and range-checked on the "
                                "device) -> tgk_assemble_async_d -> D2H of K(, M), F into pinned host buffers; two "
                                "device buffer sets on three streams so step i's D2H overlaps step i+1's H2D and "
                                "compute; the range checks read back once after the steps (tgk_mesh_upload_check) "
                                "inside the timed region (sync_drop_in: the blocking tgk_assemble)")

    # roofline of the fused kernel (per launch, kernel-only events)
    Nn = own_rows[1] - own_rows[0]
    nnz_own = int(row_ptr[own_rows[1]] - row_ptr[own_rows[0]])
    ab, comp = alg_bytes(kind, E_own, Nn, nnz_own, with_mass, has_f, vbytes=4 if f32 else 8)
    peak, peak_src = peaks()
    achieved = ab / (ms_kernel * 1e-3) / 1e9
    launches = args.steps * (1 + (2 * (2 if with_mass else 1) if exchange and s.receives_down else 0))
    fast = args.mode == "fast" and not f32
    mode_desc = ("fast (TGK_MODE_FAST: CSR pattern bit-exact, values within |dv| <= 1e-12|v_ref| + 1e-14 max|v_ref| "
                 "of the reference, bitwise deterministic; tests/test_gpu_fast.py)" if fast else
                 "exact (bit-identical to the reference)" if not f32 else "fp32 (|dv| <= 1e-5|v| + 1e-7 max|v|)")
    fplan = None
    if fast:
        fr, fb, fh, fe, fw, fby = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        if L.tgk_routing_fast_plan_info(routing._h, C.byref(fr), C.byref(fb), C.byref(fh), C.byref(fe), C.byref(fw),
                                        C.byref(fby)) == 0:
            fplan = {"rows_per_block": fr.value, "blocks": fb.value, "halo_elements": fh.value,
                     "recompute_factor": fh.value / max(1, E_own), "entries": fe.value, "item_words": fw.value,
                     "bytes": fby.value}
    config = {"workload": desc, "elements_per_gpu": E_own, "nnz_per_gpu": nnz_own, "mode": mode_desc,
              "parallelism": parallelism,
              "l2": "inputs larger than L2 (working set > 126 MB L2)" if ab > 2e8 else
                    "working set below L2 size (C1 parity config; no flush between steps)",
              "exact_plan": {"rows_per_block": R_plan, "blocks": nb.value, "halo_elements": nh.value,
                             "recompute_factor": nh.value / max(1, elems.shape[0]), "records": nrec.value,
                             "bytes": pbytes.value},
              "setup_s": setup_s, "kernel_ms": ms_kernel}
    if fplan is not None:
        config["fast_plan"] = fplan
    if other is not None:
        config["other_mode_kernel_ms"] = {("exact" if fast else "fast"): other}
    if graph is not None:
        config["cuda_graph"] = graph
    return dict(value=value, ms_per_step=ms_per_step, scaling=scaling, config=config, e2e=e2e,
                gpu_launches=launches, clocks=clocks.summary(),
                roofline={"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                          "frac": achieved / peak, "traffic": ncu_traffic(args.workload, "k_fast_scalar" if fast else "k_fused_scalar") if world == 1 else None,
                          "alg_bytes": ab, "compulsory_bytes": comp,
                          "peak_source": peak_src,
                          "kernel": ("k_fast_scalar" if fast else "k_fused_scalar") + " (one launch per step)",
                          "kernel_ms": ms_kernel})


def run_elasticity(args, ctx, N):
    """c3: 3D linear elasticity (materialised Stage I + Stage II kernels; replicas for N > 1)."""
    torch = ctx.torch
    from paper_2602_05052_b200 import engine, tgfem
    kind, div, _, desc, scaling = WORKLOADS["c3"]
    t0 = time.time()
    m = tgfem.generate_grid(kind, [1.0] * 3, list(div))
    mesh = engine.DeviceMesh(kind, m.nodes, m.elements)
    routing = engine.Routing(mesh, 3)
    setup_s = time.time() - t0
    p, keep = engine.make_problem("elasticity", lam=LAME[0], mu=LAME[1], sources=[1.0, 1.0, 1.0], mode=args.mode)
    K = torch.empty(routing.nnz, dtype=torch.float64, device=ctx.dev)
    F = torch.empty(routing.N, dtype=torch.float64, device=ctx.dev)
    L = N.lib()

    def step():
        N.check(L.tgk_assemble_d(C.byref(p), mesh._h, routing._h, ptr(K), ptr(F), None, ctx.sp))

    for _ in range(args.warmup):
        step()
    ramp(step, ctx)
    with ClockSampler(ctx.local_rank) as clocks:
        ms = ctx.timed(step, args.steps)
    ms_per_step = ms / args.steps
    # the other fp64 mode on the same inputs (both modes reported)
    q, keep_q = engine.make_problem("elasticity", lam=LAME[0], mu=LAME[1], sources=[1.0, 1.0, 1.0],
                                    mode="exact" if args.mode == "fast" else "fast")
    qK, qF = torch.empty_like(K), torch.empty_like(F)

    def step_other():
        N.check(L.tgk_assemble_d(C.byref(q), mesh._h, routing._h, ptr(qK), ptr(qF), None, ctx.sp))
    step_other()
    other_ms = ctx.timed(step_other, max(3, args.steps // 4)) / max(3, args.steps // 4)
    del qK, qF
    E = m.element_count()
    value = E * ctx.world / (ms_per_step * 1e-3)
    ab, comp = alg_bytes(kind, E, m.node_count(), routing.nnz, False, True, comps=3)
    peak, peak_src = peaks()
    achieved = ab / (ms_per_step * 1e-3) / 1e9
    e2e = None
    if args.e2e_steps > 0:
        hK = np.empty(routing.nnz)
        hF = np.empty(routing.N)
        h_nodes = torch.from_numpy(np.ascontiguousarray(m.nodes)).pin_memory()
        h_elems = torch.from_numpy(np.ascontiguousarray(m.elements)).pin_memory()
        hp = N.Problem()
        C.memmove(C.addressof(hp), C.addressof(p), C.sizeof(p))

        def e2e_step():
            N.check(L.tgk_mesh_upload(mesh._h, ptr(h_nodes), ptr(h_elems), ctx.sp))
            N.check(L.tgk_assemble(C.byref(hp), mesh._h, routing._h, hK.ctypes.data, hF.ctypes.data, None))
        e2e_step()
        ctx.barrier()
        w0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        e2e_s = ctx.max_over_ranks((time.perf_counter() - w0) / args.e2e_steps)
        e2e = {"value": E * ctx.world / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(h_nodes.numel() * 8 + h_elems.numel() * 8),
               "d2h_bytes_per_step": int((hK.size + hF.size) * 8), "ms_per_step": e2e_s * 1e3,
               "path": "tgk_mesh_upload + tgk_assemble (host buffers)"}
        if ctx.world == 1:
            fK = torch.empty(routing.nnz, dtype=torch.float64).pin_memory()
            fF = torch.empty(routing.N, dtype=torch.float64).pin_memory()
            pipe = e2e_pipelined(ctx, N, L, engine, kind, m.nodes, m.elements, p, False, h_nodes, h_elems, fK, fF,
                                 None, args.e2e_steps, comps=3)
            if pipe is not None:
                e2e["sync_drop_in"] = {"value": e2e["value"], "ms_per_step": e2e["ms_per_step"], "path": e2e["path"]}
                e2e.update(value=E / pipe, ms_per_step=pipe * 1e3,
                           path="repeated assembly through the public API: per step tgk_mesh_upload (pinned H2D) -> "
                                "tgk_assemble_d -> D2H of K, F into pinned host buffers; two device buffer sets on "
                                "three streams so step i's D2H overlaps step i+1's H2D and compute (sync_drop_in: "
                                "the blocking tgk_assemble into pageable buffers)")
    fast = args.mode == "fast"
    config = {"workload": desc, "elements_per_gpu": E, "nnz_per_gpu": routing.nnz,
              "mode": ("fast (TGK_MODE_FAST: within |dv| <= 1e-12|v_ref| + 1e-14 max|v_ref|, deterministic; "
                       "tests/test_gpu_fast.py)" if fast else "exact (bit-identical to the reference)"),
              "parallelism": "single GPU" if ctx.world == 1 else f"{ctx.world} independent replicas",
              "path": ("fast elasticity kernel (fast.cu k_fast_elast)" if fast else
                       "fused row-block elasticity kernel (fused_elast.cu)") + ": one launch per step",
              "l2": "inputs larger than L2", "setup_s": setup_s,
              "other_mode_kernel_ms": {("exact" if fast else "fast"): other_ms}}
    return dict(value=value, ms_per_step=ms_per_step, scaling=scaling, config=config, e2e=e2e,
                gpu_launches=args.steps, clocks=clocks.summary(),
                roofline={"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                          "frac": achieved / peak, "traffic": ncu_traffic("c3", "k_fast_elast" if fast else "k_fused_elast") if ctx.world == 1 else None,
                          "alg_bytes": ab, "compulsory_bytes": comp, "peak_source": peak_src,
                          "kernel": ("k_fast_elast" if fast else "k_fused_elast2") + " (one launch per step)"})


def run_reduce(args, ctx, N):
    """rm: the materialised Stage II drop-in tgk_reduce_matrix_d (k_segment_reduce) on the reference's
    published reduction workload; input = the unit-coefficient local stiffness (E x 3 x 3) in HBM."""
    torch = ctx.torch
    from paper_2602_05052_b200 import engine, tgfem
    kind, div, _, desc, scaling = WORKLOADS["rm"]
    t0 = time.time()
    m = tgfem.generate_grid(kind, [1.0, 0.5], list(div))
    mesh = engine.DeviceMesh(kind, m.nodes, m.elements)
    routing = engine.Routing(mesh, 1, segments=True)
    E, Nn = m.element_count(), m.node_count()
    local = engine.local_stiffness_diffusion(mesh, 1, torch.ones(E, dtype=torch.float64, device=ctx.dev))
    vals = torch.empty(routing.nnz, dtype=torch.float64, device=ctx.dev)
    setup_s = time.time() - t0
    L = N.lib()

    def step():
        N.check(L.tgk_reduce_matrix_d(routing._h, ptr(local), ptr(vals), ctx.sp))

    for _ in range(args.warmup):
        step()
    ramp(step, ctx)
    with ClockSampler(ctx.local_rank) as clocks:
        ms = ctx.timed(step, args.steps)
    ms_per_step = ms / args.steps
    value = E * ctx.world / (ms_per_step * 1e-3)
    nnz = routing.nnz
    # algorithmic bytes: segment offsets + slots + the gathered local values + the CSR values written
    ab = (nnz + 1) * 4 + E * 9 * 4 + E * 9 * 8 + nnz * 8
    peak, peak_src = peaks()
    achieved = ab / (ms_per_step * 1e-3) / 1e9
    e2e = None
    if args.e2e_steps > 0:
        h_local = torch.empty(local.shape, dtype=torch.float64).pin_memory()
        h_local.copy_(local)
        h_vals = torch.empty(nnz, dtype=torch.float64).pin_memory()

        def e2e_step():  # host K_local in, host CSR values out (the reference's calling pattern)
            local.copy_(h_local, non_blocking=True)
            step()
            h_vals.copy_(vals, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        e2e_step()
        w0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        e2e_s = ctx.max_over_ranks((time.perf_counter() - w0) / args.e2e_steps)
        e2e = {"value": E * ctx.world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h_local.numel() * 8),
               "d2h_bytes_per_step": int(nnz * 8), "ms_per_step": e2e_s * 1e3,
               "path": "pinned H2D of K_local (E x 9) + tgk_reduce_matrix_d + D2H of the CSR values"}
    config = {"workload": desc, "elements": E, "nnz": nnz, "mode": "exact (bit-identical)",
              "parallelism": "single GPU" if ctx.world == 1 else f"{ctx.world} independent replicas",
              "l2": "inputs larger than L2 (72 MB K_local + 13 MB segments + 28 MB values ~ L2 size; not flushed)",
              "reference_published_ms": 12.25, "setup_s": setup_s}
    return dict(value=value, ms_per_step=ms_per_step, scaling=scaling, config=config, e2e=e2e,
                gpu_launches=args.steps, clocks=clocks.summary(),
                roofline={"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                          "frac": achieved / peak, "traffic": ncu_traffic("rm", "k_segment_reduce") if ctx.world == 1 else None, "alg_bytes": ab,
                          "peak_source": peak_src, "kernel": "k_segment_reduce (one launch per step)",
                          "kernel_ms": ms_per_step})


def run_batched(args, ctx, N):
    """c4: batched per-element coefficient fields + adjoint gather; fields sharded across ranks."""
    torch = ctx.torch
    from paper_2602_05052_b200 import engine, meshgen
    _, _, _, desc, scaling = WORKLOADS["c4"]
    t0 = time.time()
    nodes, elems = meshgen.unstructured_tri(256)
    E, Nn = elems.shape[0], nodes.shape[0]
    mesh = engine.DeviceMesh("tri3", nodes, elems)
    routing = engine.Routing(mesh, 1)
    from paper_2602_05052_b200 import dist as D
    b0, b1 = D.field_shard(C4_FIELDS, ctx.rank, ctx.world)
    Bl = b1 - b0
    rho_h = np.stack([0.5 + np.random.default_rng(1000 + b).random(E) for b in range(b0, b0 + Bl)])
    lam_h = np.stack([np.random.default_rng(2000 + b).random(Nn) - 0.5 for b in range(b0, b0 + Bl)])
    U_h = np.stack([np.random.default_rng(3000 + b).random(Nn) - 0.5 for b in range(b0, b0 + Bl)])
    rho = torch.from_numpy(rho_h).to(ctx.dev)
    lam = torch.from_numpy(lam_h).to(ctx.dev)
    U = torch.from_numpy(U_h).to(ctx.dev)
    K = torch.empty(Bl, routing.nnz, dtype=torch.float64, device=ctx.dev)
    F = torch.empty(Nn, dtype=torch.float64, device=ctx.dev)
    dr = torch.empty(Bl, E, dtype=torch.float64, device=ctx.dev)
    setup_s = time.time() - t0
    L = N.lib()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]

    mode = engine.MODES[args.mode]  # both modes run k_batched_entries (bit-identical; fast variants were slower)
    kname = "k_batched_entries"

    def k_batched():
        N.check(L.tgk_assemble_batched_d(mesh._h, routing._h, Bl, ptr(rho), 1.0, ptr(K), ptr(F), mode, ctx.sp))

    def k_adjoint():
        N.check(L.tgk_adjoint_gather_d(mesh._h, routing._h, Bl, ptr(lam), ptr(U), ptr(dr), 1, ctx.sp))

    def step():
        k_batched()
        k_adjoint()

    for _ in range(args.warmup):
        step()
    ramp(step, ctx)
    with ClockSampler(ctx.local_rank) as clocks:
        ms = ctx.timed(step, args.steps)
        ctx.barrier()
        ev[0].record(ctx.stream)
        for _ in range(args.steps):
            k_batched()
        ev[1].record(ctx.stream)
        for _ in range(args.steps):
            k_adjoint()
        ev[2].record(ctx.stream)
        torch.cuda.synchronize()
    ms_b = ev[0].elapsed_time(ev[1]) / args.steps
    ms_a = ev[1].elapsed_time(ev[2]) / args.steps
    ms_per_step = ms / args.steps
    value = E * C4_FIELDS / (ms_per_step * 1e-3)  # element-fields per second, all ranks
    # batched K_b: connectivity + coordinates + slot map + B*nnz*8 + B*E*8 (rho) + N*8 (F)
    ab_b = E * 3 * 4 + Nn * 2 * 8 + E * 9 * 4 + Bl * routing.nnz * 8 + Bl * E * 8 + Nn * 8
    ab_a = E * 3 * 4 + Nn * 2 * 8 + E * 9 * 4 + Bl * (2 * Nn * 8 + E * 8)
    peak, peak_src = peaks()
    ach_b = ab_b / (ms_b * 1e-3) / 1e9
    ach_a = ab_a / (ms_a * 1e-3) / 1e9
    e2e = None
    if args.e2e_steps > 0:
        h_rho = torch.from_numpy(rho_h).pin_memory()
        h_lam = torch.from_numpy(lam_h).pin_memory()
        h_U = torch.from_numpy(U_h).pin_memory()
        hK = torch.empty(Bl, routing.nnz, dtype=torch.float64).pin_memory()
        hdr = torch.empty(Bl, E, dtype=torch.float64).pin_memory()
        hF = torch.empty(Nn, dtype=torch.float64).pin_memory()

        def e2e_step():
            rho.copy_(h_rho, non_blocking=True)
            lam.copy_(h_lam, non_blocking=True)
            U.copy_(h_U, non_blocking=True)
            step()
            hK.copy_(K, non_blocking=True)
            hF.copy_(F, non_blocking=True)
            hdr.copy_(dr, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        e2e_step()
        ctx.barrier()
        w0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        e2e_s = ctx.max_over_ranks((time.perf_counter() - w0) / args.e2e_steps)
        sync_s = e2e_s
        # pipelined repetition: two device buffer sets on upload / compute / download streams
        try:
            sets = [dict(rho=torch.empty_like(rho), lam=torch.empty_like(lam), U=torch.empty_like(U),
                         K=torch.empty_like(K), F=torch.empty_like(F), dr=torch.empty_like(dr)) for _ in range(2)]
            s_up, s_cmp, s_dn = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
            ev_up, ev_cmp, ev_dn = ([torch.cuda.Event() for _ in range(2)] for _ in range(3))

            def pipe_step(i):
                j = i & 1
                b = sets[j]
                s_up.wait_event(ev_cmp[j])
                with torch.cuda.stream(s_up):
                    b["rho"].copy_(h_rho, non_blocking=True)
                    b["lam"].copy_(h_lam, non_blocking=True)
                    b["U"].copy_(h_U, non_blocking=True)
                ev_up[j].record(s_up)
                s_cmp.wait_event(ev_up[j])
                s_cmp.wait_event(ev_dn[j])
                sp = C.c_void_p(s_cmp.cuda_stream)
                N.check(L.tgk_assemble_batched_d(mesh._h, routing._h, Bl, ptr(b["rho"]), 1.0, ptr(b["K"]),
                                                 ptr(b["F"]), mode, sp))
                N.check(L.tgk_adjoint_gather_d(mesh._h, routing._h, Bl, ptr(b["lam"]), ptr(b["U"]), ptr(b["dr"]),
                                               1, sp))
                ev_cmp[j].record(s_cmp)
                s_dn.wait_event(ev_cmp[j])
                with torch.cuda.stream(s_dn):
                    hK.copy_(b["K"], non_blocking=True)
                    hF.copy_(b["F"], non_blocking=True)
                    hdr.copy_(b["dr"], non_blocking=True)
                ev_dn[j].record(s_dn)

            for i in range(3):
                pipe_step(i)
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            for i in range(args.e2e_steps):
                pipe_step(i)
            torch.cuda.synchronize()
            e2e_s = ctx.max_over_ranks((time.perf_counter() - w0) / args.e2e_steps)
            del sets
        except Exception:
            pass
        e2e = {"value": E * C4_FIELDS / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int((h_rho.numel() + h_lam.numel() + h_U.numel()) * 8),
               "d2h_bytes_per_step": int((hK.numel() + hF.numel() + hdr.numel()) * 8),
               "ms_per_step": e2e_s * 1e3,
               "path": "per step: pinned H2D of rho/lambda/U + tgk_assemble_batched_d + tgk_adjoint_gather_d + D2H of "
                       "K_b, F, drho; two device buffer sets on upload / compute / download streams so consecutive "
                       "steps' copies overlap (sync_drop_in: one stream, no overlap)",
               "sync_drop_in": {"value": E * C4_FIELDS / sync_s, "ms_per_step": sync_s * 1e3}}
    config = {"workload": desc, "fields_per_gpu": Bl, "elements": E, "nnz": routing.nnz,
              "metric_unit_note": "element-fields/s (E x 256 per step)",
              "parallelism": "single GPU" if ctx.world == 1 else f"{ctx.world} GPUs, fields sharded (no collective)",
              "l2": "outputs larger than L2 (K_b 943 MB per step)", "setup_s": setup_s,
              "mode": "exact kernels in both modes (bit-identical)", "batched_ms": ms_b, "adjoint_ms": ms_a,
              "adjoint_roofline": {"achieved": ach_a, "frac": ach_a / peak, "alg_bytes": ab_a}}
    return dict(value=value, ms_per_step=ms_per_step, scaling=scaling, config=config, e2e=e2e,
                gpu_launches=args.steps * 2, clocks=clocks.summary(),
                roofline={"bound": "hbm", "achieved": ach_b, "peak": peak, "unit": "GB/s",
                          "frac": ach_b / peak, "traffic": ncu_traffic("c4", kname) if ctx.world == 1 else None,
                          "alg_bytes": ab_b, "peak_source": peak_src,
                          "kernel": f"{kname} (one launch per step, all fields)", "kernel_ms": ms_b})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--dist-mode", default="exchange", choices=["exchange", "halo"])
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"],
                    help="f32: the fp32 variant of the fused scalar kernel (tgk_assemble_f32_d)")
    ap.add_argument("--mode", default="fast", choices=["fast", "exact"],
                    help="fp64 arithmetic mode of the scalar workloads (TGK_MODE_FAST / TGK_MODE_EXACT)")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample", type=int, nargs="*", default=None)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    from paper_2602_05052_b200 import _native as N
    ctx = Ctx(args)
    if args.workload == "c3":
        r = run_elasticity(args, ctx, N)
    elif args.workload == "c4":
        r = run_batched(args, ctx, N)
    elif args.workload == "rm":
        r = run_reduce(args, ctx, N)
    else:
        r = run_scalar(args, ctx, N)
    cpu = None
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_line(args.workload)
    if ctx.rank == 0:
        line = {
            "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": ctx.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
            "scaling": r["scaling"], "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
            "config": r["config"], "roofline": r["roofline"], "cpu_baseline": cpu, "e2e": r["e2e"],
            "gpu_launches": r["gpu_launches"], "clocks": r["clocks"],
        }
        print(json.dumps(line))
    if ctx.dist:
        ctx.dist.destroy_process_group()


if __name__ == "__main__":
    main()
