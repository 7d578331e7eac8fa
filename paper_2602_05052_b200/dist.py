"""Multi-GPU assembly of one Kuhn grid by row-owning z-slabs.

One process per GPU.  Kuhn element ids are cube-major with x fastest, then y,
then z (generate_grid, mesh.cpp:134-150) and node ids are x-fastest, so a
contiguous range of cube layers is a z-slab and a node layer is a contiguous
range of CSR rows.  Rank r of `world` owns cube layers [z0, z1) and the node
layers [z0, z1) (the last rank also owns the top layer).  Two modes:

``exchange`` (default; the north star's NCCL interface reduction)
    the local mesh is the slab extended by one cube layer on each side, so its
    CSR rows for node layers z0..z1 are exactly the global rows; the fused
    kernel assembles only the rank's own elements (tgk_routing_set_element_range)
    into rows z0..z1.  The top node layer z1 then holds the partial fold of the
    rank's elements and is sent to rank r+1, which adds it in front of its own
    partial for that layer (lower elements first: a fixed order, deterministic;
    equal to the single-GPU fold within rounding).  One
    ncclSend/ncclRecv pair per neighbour (torch.distributed P2P over NCCL).
``halo``
    the local mesh is the slab plus one cube layer below; every element
    incident to an owned row is assembled locally (halo recompute): no data-path
    collective, rows bitwise equal to the single-GPU result (the ablation).

The host logic here is device-agnostic (torch.distributed with nccl on GPUs,
gloo on CPU for the multi-process tests); the interface sum runs in libtgk's
``tgk_interface_combine_d`` on the GPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Slab:
    rank: int
    world: int
    div: tuple          # (nx, ny, layers per rank)
    mode: str
    zl: int             # local mesh = global cube layers [zl, zh)
    zh: int
    z0: int             # own cube layers [z0, z1)
    z1: int
    layer: int          # nodes per node layer
    own_lo: int         # owned node rows, local numbering
    own_hi: int
    calc_hi: int        # rows assembled locally: [own_lo, calc_hi)
    elem_lo: int        # own elements, local numbering
    elem_hi: int
    elem_offset: int    # global id of local element 0
    node_offset: int    # global id of local node 0

    @property
    def sends_up(self):
        return self.mode == "exchange" and self.rank < self.world - 1

    @property
    def receives_down(self):
        return self.mode == "exchange" and self.rank > 0

    @property
    def top_rows(self):
        """Local rows of the upper interface node layer (partial, sent to rank+1)."""
        return (self.own_hi, self.own_hi + self.layer)

    @property
    def bottom_rows(self):
        """Local rows of the lower interface node layer (owned, completed with rank-1's partial)."""
        return (self.own_lo, self.own_lo + self.layer)


def slab(div, rank, world, mode="exchange"):
    nx, ny, nzr = (int(x) for x in div)
    if mode not in ("exchange", "halo"):
        raise ValueError(f"unknown slab mode {mode!r}")
    z0, z1 = rank * nzr, (rank + 1) * nzr
    zl = z0 - 1 if rank > 0 else 0
    zh = z1 + 1 if (mode == "exchange" and rank < world - 1) else z1
    layer = (nx + 1) * (ny + 1)
    cubes = nx * ny
    own_lo = (z0 - zl) * layer
    own_hi = (z1 - zl) * layer + (layer if rank == world - 1 else 0)
    calc_hi = own_hi + (layer if (mode == "exchange" and rank < world - 1) else 0)
    if mode == "exchange":
        elem_lo, elem_hi = (z0 - zl) * cubes * 6, (z1 - zl) * cubes * 6
    else:
        elem_lo, elem_hi = 0, (zh - zl) * cubes * 6
    return Slab(rank, world, (nx, ny, nzr), mode, zl, zh, z0, z1, layer, own_lo, own_hi, calc_hi,
                elem_lo, elem_hi, zl * cubes * 6, zl * layer)


def slab_mesh(s: Slab):
    """Node coordinates and connectivity of the local mesh, bit-identical to the
    corresponding rows of the global tg::generate_grid arrays."""
    from . import tgfem
    nx, ny, nzr = s.div
    nz = nzr * s.world
    loc = tgfem.generate_grid("tet4", [1.0, 1.0, 1.0], [nx, ny, s.zh - s.zl])
    nodes = loc.nodes.copy()
    kz = np.repeat(np.arange(s.zl, s.zh + 1, dtype=np.int64), s.layer)
    nodes[:, 2] = kz * (1.0 / nz)  # same expression as mesh.cpp:139 (kz * hz)
    # Kuhn connectivity is translation invariant in z: the local pattern is the global one shifted
    return nodes, loc.elements


def exchange_interface(K, F, row_ptr, s: Slab, combine, dist, group=None):
    """Send the top interface layer's partial values up, receive the lower
    neighbour's partial for the bottom layer and fold it in front of ours:
    values[bottom] = recv + values[bottom] (via ``combine(recv, values_slice)``).
    K, F: this rank's value arrays (torch tensors on the P2P device);
    row_ptr: host int64 array of the local CSR offsets."""
    import torch
    ops = []
    send = recv = None
    if s.sends_up:
        lo, hi = s.top_rows
        send = torch.cat([K[int(row_ptr[lo]):int(row_ptr[hi])], F[lo:hi]]).contiguous()
        ops.append(dist.P2POp(dist.isend, send, s.rank + 1, group))
    if s.receives_down:
        lo, hi = s.bottom_rows
        n = int(row_ptr[hi] - row_ptr[lo]) + (hi - lo)
        recv = torch.empty(n, dtype=K.dtype, device=K.device)
        ops.append(dist.P2POp(dist.irecv, recv, s.rank - 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if recv is not None:
        lo, hi = s.bottom_rows
        nk = int(row_ptr[hi] - row_ptr[lo])
        combine(recv[:nk], K[int(row_ptr[lo]):int(row_ptr[hi])])
        combine(recv[nk:], F[lo:hi])
    return (0 if send is None else send.numel() * 8) + (0 if recv is None else recv.numel() * 8)


def field_shard(B, rank, world):
    """Batched coefficient fields (C4) shard trivially: rank r
    assembles fields [b0, b1) — contiguous, balanced to within one field, no
    collective (every field's K_b, adjoint row drho_b is independent)."""
    if B < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("field_shard: bad arguments")
    return rank * B // world, (rank + 1) * B // world


def gpu_combine(lower, values):
    """values = lower + values on the GPU (libtgk tgk_interface_combine_d)."""
    import ctypes as C
    import torch
    from ._native import check, lib
    check(lib().tgk_interface_combine_d(C.c_void_p(lower.data_ptr()), C.c_void_p(values.data_ptr()),
                                        values.numel(), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
