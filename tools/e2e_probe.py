"""Where does the C2 end-to-end step go?  The pipelined bench step (tgk_mesh_upload
+ tgk_assemble_async_d + D2H on three streams) vs the same with the mesh upload
done as async torch copies (no host sync inside the upload)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import port  # noqa: E402
from paper_2602_05052_b200 import _native as N, engine  # noqa: E402

L = N.lib()
nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [100, 100, 100])
p, keep = engine.make_problem("poisson", 1.0, sources=[1.0], with_mass=True, mode="fast")
dev = torch.device("cuda:0")
h_nodes = torch.from_numpy(nodes).pin_memory()
h_elems = torch.from_numpy(elems).pin_memory()
meshes = [engine.DeviceMesh("tet4", nodes, elems) for _ in range(2)]
routs = [engine.Routing(m, 1) for m in meshes]
nnz, n = routs[0].nnz, routs[0].N
fK = torch.empty(nnz, dtype=torch.float64).pin_memory()
fM = torch.empty(nnz, dtype=torch.float64).pin_memory()
fF = torch.empty(n, dtype=torch.float64).pin_memory()
bufs = [dict(K=torch.empty(nnz, dtype=torch.float64, device=dev), M=torch.empty(nnz, dtype=torch.float64, device=dev),
             F=torch.empty(n, dtype=torch.float64, device=dev), bad=torch.full((1,), -1, dtype=torch.int64, device=dev),
             st=torch.empty(elems.size, dtype=torch.int64, device=dev)) for _ in range(2)]
views = []
for m in meshes:
    dn, de = C.c_void_p(), C.c_void_p()
    N.check(L.tgk_mesh_info(m._h, None, None, None, C.byref(dn), C.byref(de)))
    views.append((dn.value, de.value))
s_up, s_cmp, s_dn = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
ev_up, ev_cmp, ev_dn = ([torch.cuda.Event() for _ in range(2)] for _ in range(3))
ptr = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731


def step(i, mode):
    j = i & 1
    b = bufs[j]
    s_up.wait_event(ev_cmp[j])
    if mode == "abi":
        N.check(L.tgk_mesh_upload(meshes[j]._h, ptr(h_nodes), ptr(h_elems), C.c_void_p(s_up.cuda_stream)))
    elif mode == "abi_async":
        N.check(L.tgk_mesh_upload_async(meshes[j]._h, ptr(h_nodes), ptr(h_elems), C.c_void_p(s_up.cuda_stream)))
    elif mode == "nodes_only":  # connectivity resident: coordinates only (lower bound of the H2D side)
        N.check(L.tgk_mesh_upload_async(meshes[j]._h, ptr(h_nodes), None, C.c_void_p(s_up.cuda_stream)))
    else:  # async copies + narrowing on the stream, no host sync
        N.check(L.tgk_copy_d2d(C.c_void_p(views[j][0]), ptr(h_nodes), h_nodes.numel() * 8, C.c_void_p(s_up.cuda_stream)))
        with torch.cuda.stream(s_up):
            b["st"].copy_(h_elems.view(-1), non_blocking=True)
            conn = torch.from_dlpack(b["st"])  # placeholder to keep the shape
            tmp = b["st"].to(torch.int32)
        N.check(L.tgk_copy_d2d(C.c_void_p(views[j][1]), ptr(tmp), tmp.numel() * 4, C.c_void_p(s_up.cuda_stream)))
    ev_up[j].record(s_up)
    s_cmp.wait_event(ev_up[j])
    s_cmp.wait_event(ev_dn[j])
    N.check(L.tgk_assemble_async_d(C.byref(p), meshes[j]._h, routs[j]._h, ptr(b["K"]), ptr(b["F"]), ptr(b["M"]),
                                   ptr(b["bad"]), C.c_void_p(s_cmp.cuda_stream)))
    ev_cmp[j].record(s_cmp)
    s_dn.wait_event(ev_cmp[j])
    with torch.cuda.stream(s_dn):
        fK.copy_(b["K"], non_blocking=True)
        fF.copy_(b["F"], non_blocking=True)
        fM.copy_(b["M"], non_blocking=True)
    ev_dn[j].record(s_dn)


for mode in ["abi", "async", "abi_async", "nodes_only", "abi_async"]:
    for i in range(4):
        step(i, mode)
    torch.cuda.synchronize()
    w = time.perf_counter()
    for i in range(20):
        step(i, mode)
    torch.cuda.synchronize()
    print(mode, "ms/step %.3f" % ((time.perf_counter() - w) / 20 * 1e3))

# the narrowing kernel alone (tgk_mesh_upload_async with nodes=None, elements resident in pinned memory)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st = torch.cuda.current_stream()
for _ in range(2):
    N.check(L.tgk_mesh_upload_async(meshes[0]._h, None, ptr(h_elems), C.c_void_p(st.cuda_stream)))
torch.cuda.synchronize()
ev0.record(st)
for _ in range(10):
    N.check(L.tgk_mesh_upload_async(meshes[0]._h, None, ptr(h_elems), C.c_void_p(st.cuda_stream)))
ev1.record(st)
torch.cuda.synchronize()
print("upload_async(elems) ms %.3f" % (ev0.elapsed_time(ev1) / 10))
d_elems = torch.from_numpy(elems.reshape(-1)).to(dev)
ev0.record(st)
for _ in range(10):
    h_tmp = d_elems.to(torch.int32)
ev1.record(st)
torch.cuda.synchronize()
print("torch narrow only ms %.3f" % (ev0.elapsed_time(ev1) / 10))
