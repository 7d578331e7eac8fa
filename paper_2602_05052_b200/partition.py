"""Row-owning partitions of ANY mesh for multi-GPU assembly.

The z-slabs of dist.py rely on the Kuhn grid's numbering; this partitioner
takes an arbitrary mesh (e.g. a permuted unstructured gmsh mesh):

* nodes are ordered along a Morton curve of their coordinates and cut into
  ``world`` contiguous chunks: part p OWNS those rows (compact in space =>
  short interfaces);
* an element is owned by the lowest part among its nodes ("element ownership
  by minimum row"), so every element is assembled by exactly one rank;
* rank p's local mesh = every element touching a p-owned node (ascending
  global element id, owned elements first in exchange mode), local nodes =
  p's owned nodes first (ascending global id) then the others: the owned rows
  are the local row range [0, n_own) (tgk_routing_set_owned_rows), the owned
  elements the range [0, e_own) (tgk_routing_set_element_range).

Two modes, as dist.py:

``halo``      every element touching an owned row is assembled locally (halo
              recompute); no data-path collective; every owned row bitwise
              equal to the single-GPU result (the local element order keeps
              the global ascending order, the reference fold order).
``exchange``  each rank assembles only its owned elements into all of its
              local rows; the ghost rows' partials are sent to their owners,
              one send/recv pair per neighbouring part (torch.distributed P2P:
              NCCL on GPUs, gloo in the CPU tests), and added after the owner's
              own partial in ascending source-rank order (deterministic; equal
              to one GPU within the SURVEY.md 8(c) tolerance).

Everything here is host-side index bookkeeping (numpy); the assembly is the
library's fused kernels, the interface sum a deterministic index_add per
neighbour.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def morton_keys(nodes):
    """Morton code of each node (21 bits per axis in 3D, 32 in 2D), like plan.cpp morton_order."""
    nodes = np.asarray(nodes, dtype=np.float64)
    d = nodes.shape[1]
    lo = nodes.min(axis=0)
    span = float((nodes.max(axis=0) - lo).max()) or 1.0
    bits = 21 if d == 3 else 32
    q = ((nodes - lo) * (((1 << bits) - 1) / span)).astype(np.uint64)
    key = np.zeros(nodes.shape[0], dtype=np.uint64)
    for b in range(bits):
        for c in range(d):
            key |= ((q[:, c] >> np.uint64(b)) & np.uint64(1)) << np.uint64(b * d + c)
    return key


@dataclass
class Part:
    rank: int
    world: int
    mode: str
    nodes_g: np.ndarray      # local -> global node id (owned first)
    elems_g: np.ndarray      # local -> global element id
    n_own: int               # owned rows: local [0, n_own)
    e_own: int               # assembled elements: local [0, e_own) (all local elements in halo mode)
    nodes: np.ndarray        # local coordinates
    elems: np.ndarray        # local connectivity (local node ids)
    offsets: np.ndarray = None   # local CSR pattern (host), for the exchange maps
    cols: np.ndarray = None
    send: dict = field(default_factory=dict)   # q -> (K positions, F rows) sent to q, local numbering
    recv: dict = field(default_factory=dict)   # q -> (K positions, F rows) received from q

    @property
    def exchange(self):
        return self.mode == "exchange"


def csr_pattern(n_nodes, elems):
    """Sorted-unique neighbour lists of a mesh (the pattern of build_routing, routing.cpp:17-36)."""
    k = elems.shape[1]
    rows = np.repeat(elems, k, axis=1).reshape(-1)
    cols = np.tile(elems, (1, k)).reshape(-1)
    key = np.unique(rows.astype(np.int64) * n_nodes + cols)
    r, c = key // n_nodes, key % n_nodes
    offsets = np.zeros(n_nodes + 1, dtype=np.int64)
    np.add.at(offsets, r + 1, 1)
    return np.cumsum(offsets), c


def partition(nodes, elems, world, mode="exchange"):
    """All `world` parts of a mesh (each rank uses parts[rank])."""
    if mode not in ("exchange", "halo"):
        raise ValueError(f"unknown partition mode {mode!r}")
    nodes = np.asarray(nodes, dtype=np.float64)
    elems = np.asarray(elems, dtype=np.int64)
    N, E = nodes.shape[0], elems.shape[0]
    order = np.argsort(morton_keys(nodes), kind="stable")
    part_of = np.empty(N, dtype=np.int64)
    part_of[order] = np.arange(N) * world // N
    owner = part_of[elems].min(axis=1)
    parts = []
    for p in range(world):
        own_nodes = np.nonzero(part_of == p)[0]                      # ascending global id
        touch = np.nonzero((part_of[elems] == p).any(axis=1))[0]    # ascending global element id
        if mode == "exchange":
            mine = touch[owner[touch] == p]
            elems_g = np.concatenate([mine, touch[owner[touch] != p]])
            e_own = mine.size
        else:
            elems_g, e_own = touch, touch.size
        others = np.setdiff1d(np.unique(elems[elems_g]), own_nodes)
        nodes_g = np.concatenate([own_nodes, others])
        g2l = np.full(N, -1, dtype=np.int64)
        g2l[nodes_g] = np.arange(nodes_g.size)
        parts.append(Part(p, world, mode, nodes_g, elems_g, own_nodes.size, e_own, nodes[nodes_g],
                          g2l[elems[elems_g]]))
    if mode == "exchange":
        _exchange_maps(parts, part_of)
    return parts


def _exchange_maps(parts, part_of):
    """Per neighbour pair: the ghost-row entries rank p sends to their owner q
    (positions in p's local K and F) and where q adds them (positions in q's)."""
    for pt in parts:
        pt.offsets, pt.cols = csr_pattern(pt.nodes_g.size, pt.elems)
    for p, pt in enumerate(parts):
        ghost = np.arange(pt.n_own, pt.nodes_g.size)
        gowner = part_of[pt.nodes_g[ghost]]
        for q in np.unique(gowner):
            q = int(q)
            qt = parts[q]
            rows = ghost[gowner == q]
            # sent entries: every position of those local rows, row-major
            pos = np.concatenate([np.arange(pt.offsets[r], pt.offsets[r + 1]) for r in rows])
            grow = np.repeat(pt.nodes_g[rows], np.diff(pt.offsets)[rows])
            gcol = pt.nodes_g[pt.cols[pos]]
            # the owner's positions of the same (global row, global column) pairs
            g2l_q = {int(g): i for i, g in enumerate(qt.nodes_g)}
            qrow = np.array([g2l_q[int(g)] for g in grow], dtype=np.int64)
            qcol = np.array([g2l_q[int(g)] for g in gcol], dtype=np.int64)
            qpos = np.empty(qrow.size, dtype=np.int64)
            for i, (r, c) in enumerate(zip(qrow, qcol)):
                lo, hi = qt.offsets[r], qt.offsets[r + 1]
                j = lo + np.searchsorted(qt.cols[lo:hi], c)
                assert j < hi and qt.cols[j] == c, "ghost entry missing from the owner's row"
                qpos[i] = j
            qrows_f = np.array([g2l_q[int(g)] for g in pt.nodes_g[rows]], dtype=np.int64)
            pt.send[q] = (pos, rows)
            qt.recv[p] = (qpos, qrows_f)


def exchange(part: Part, K, F, dist, group=None):
    """Send the ghost rows' partial values to their owners, receive the
    neighbours' partials for the owned rows and add them after this rank's own
    partial, in ascending source-rank order (deterministic).  K, F: this rank's
    local value tensors (torch; GPU with NCCL, CPU with gloo).  Returns the bytes moved."""
    import torch
    if not part.exchange:
        return 0
    ops, bufs, moved = [], {}, 0
    for q, (pos, rows) in sorted(part.send.items()):
        pos_t = torch.as_tensor(pos, device=K.device)
        rows_t = torch.as_tensor(rows, device=K.device)
        buf = torch.cat([K.index_select(0, pos_t), F.index_select(0, rows_t)]).contiguous()
        ops.append(dist.P2POp(dist.isend, buf, q, group))
        moved += buf.numel() * buf.element_size()
    for p, (qpos, qrows) in sorted(part.recv.items()):
        buf = torch.empty(qpos.size + qrows.size, dtype=K.dtype, device=K.device)
        bufs[p] = buf
        ops.append(dist.P2POp(dist.irecv, buf, p, group))
        moved += buf.numel() * buf.element_size()
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for p in sorted(bufs):  # ascending source rank: a fixed association
        qpos, qrows = part.recv[p]
        buf = bufs[p]
        K.index_add_(0, torch.as_tensor(qpos, device=K.device), buf[:qpos.size])  # unique positions per source
        F.index_add_(0, torch.as_tensor(qrows, device=K.device), buf[qpos.size:])
    return moved
