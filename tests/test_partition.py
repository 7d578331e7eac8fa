"""CPU, gloo world_size 2 and 3: the general row-owning partitioner
(paper_2602_05052_b200/partition.py) on permuted unstructured meshes.

Each rank assembles its part with the CPU oracle exactly as the GPU path does
(owned rows = local [0, n_own); exchange mode: only its owned elements, ghost
rows sent to their owners with the real partition.exchange over
torch.distributed), and the owned rows are compared entry by entry — mapped
back to global (row, column) — with the single-process assembly: halo mode
bit-identical, exchange mode within the SURVEY.md 8(c) tolerance.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port
from paper_2602_05052_b200 import meshgen
from paper_2602_05052_b200 import partition as P
from tests._util import assert_bitwise, assert_scaled_close


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mesh(kind):
    if kind == "tri3":
        return meshgen.unstructured_tri(40)
    nodes, elems = port.generate_grid("tet4", [1.0, 1.0, 1.0], [6, 5, 7])
    rng = np.random.default_rng(8)
    pn = rng.permutation(nodes.shape[0])
    inv = np.argsort(pn)
    return nodes[pn], inv[elems][rng.permutation(elems.shape[0])]


def _local_assembly(kind, pt):
    """The rank's local assembly (oracle): exchange mode folds only elements [0, e_own)."""
    r = port.Routing(pt.nodes.shape[0], port.dofmap(kind, pt.elems, 1))
    E = pt.elems.shape[0]
    Kl = port.local(kind, pt.nodes, pt.elems, 1, port.DIFFUSION, np.ones(E))
    Fl = port.local(kind, pt.nodes, pt.elems, 1, port.LOAD, np.ones(E))
    Kl[pt.e_own:] = 0.0
    Fl[pt.e_own:] = 0.0
    return r, r.reduce_matrix(Kl.reshape(-1)), r.reduce_vector(Fl.reshape(-1))


def _worker(rank, world, port_, kind, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nodes, elems = _mesh(kind)
        pt = P.partition(nodes, elems, world, mode)[rank]
        r, K, F = _local_assembly(kind, pt)
        if mode == "exchange":
            assert np.array_equal(r.offsets, pt.offsets) and np.array_equal(r.cols, pt.cols)
        Kt, Ft = torch.from_numpy(K.copy()), torch.from_numpy(F.copy())
        moved = P.exchange(pt, Kt, Ft, dist)
        q.put((rank, pt.nodes_g, pt.n_own, r.offsets, r.cols, Kt.numpy(), Ft.numpy(), moved))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", ["tri3", "tet4"])
@pytest.mark.parametrize("mode", ["exchange", "halo"])
def test_general_partition_matches_single_process(world, kind, mode):
    nodes, elems = _mesh(kind)
    gr = port.Routing(nodes.shape[0], port.dofmap(kind, elems, 1))
    Kg, Fg, _ = port.assemble(kind, nodes, elems, gr, sources=[1.0])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_, kind, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    covered = np.zeros(nodes.shape[0], bool)
    for rank, nodes_g, n_own, offs, cols, K, F, moved in sorted(res, key=lambda t: t[0]):
        assert (moved > 0) == (mode == "exchange")
        got, want = [], []
        for lr in range(n_own):
            g = nodes_g[lr]
            assert not covered[g]
            covered[g] = True
            lc = nodes_g[cols[offs[lr]:offs[lr + 1]]]
            gcols = gr.cols[gr.offsets[g]:gr.offsets[g + 1]]
            assert np.array_equal(np.sort(lc), gcols), "owned row pattern differs from the global row"
            gpos = gr.offsets[g] + np.searchsorted(gcols, lc)
            got.append(K[offs[lr]:offs[lr + 1]])
            want.append(Kg[gpos])
        got_k, want_k = np.concatenate(got), np.concatenate(want)
        got_f, want_f = F[:n_own], Fg[nodes_g[:n_own]]
        if mode == "halo":
            assert_bitwise(got_k, want_k, f"rank {rank} K")
            assert_bitwise(got_f, want_f, f"rank {rank} F")
        else:
            assert_scaled_close(got_k, want_k, what=f"rank {rank} K")
            assert_scaled_close(got_f, want_f, what=f"rank {rank} F")
    assert covered.all(), "every row is owned by exactly one rank"
