"""CPU, world_size 2 (gloo): the multi-GPU slab logic of paper_2602_05052_b200/dist.py.

Each rank builds its slab of a global Kuhn grid exactly as bench.py does on the
GPUs, computes its partial assembly with the CPU oracle (its own elements
only, folded into the extended-mesh CSR rows), runs the real
exchange_interface over torch.distributed (gloo here, NCCL on the GPUs) and
compares the owned rows with the single-process oracle result: interior rows
bit-identical, interface rows within the SURVEY.md 8(c) tolerance (the fold
association changes there: lower slab's partial + upper slab's partial).
Also checks the halo-recompute mode (no exchange) is bitwise exact.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port
from paper_2602_05052_b200 import dist as D
from tests._util import assert_bitwise, assert_scaled_close


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partial(nodes, elems, s, with_mass):
    """Oracle assembly of this rank's own elements into the local (extended) CSR rows."""
    r = port.Routing(nodes.shape[0], port.dofmap("tet4", elems, 1))
    deg = 2 if with_mass else 1
    own = np.zeros(elems.shape[0], bool)
    own[s.elem_lo:s.elem_hi] = True
    Kl = port.local("tet4", nodes, elems, deg, port.DIFFUSION, np.ones(elems.shape[0] * (4 if deg == 2 else 1)))
    Fl = port.local("tet4", nodes, elems, deg, port.LOAD, np.ones(elems.shape[0] * (4 if deg == 2 else 1)))
    Kl[~own] = 0.0
    Fl[~own] = 0.0
    K = r.reduce_matrix(Kl.reshape(-1))
    F = r.reduce_vector(Fl.reshape(-1))
    return r, K, F


def _worker(rank, world, port_, div, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = D.slab(div, rank, world, mode)
        nodes, elems = D.slab_mesh(s)
        if mode == "exchange":
            r, K, F = _partial(nodes, elems, s, False)
        else:
            r = port.Routing(nodes.shape[0], port.dofmap("tet4", elems, 1))
            K, F, _ = port.assemble("tet4", nodes, elems, r, sources=[1.0])
        Kt, Ft = torch.from_numpy(K.copy()), torch.from_numpy(F.copy())

        def cpu_combine(lower, values):  # the GPU path runs tgk_interface_combine_d
            values.copy_(lower + values)

        nbytes = D.exchange_interface(Kt, Ft, r.offsets, s, cpu_combine, dist)
        lo, hi = s.own_lo, s.own_hi
        q.put((rank, s.node_offset + lo, s.node_offset + hi, r.offsets[lo:hi + 1] - r.offsets[lo],
               Kt.numpy()[r.offsets[lo]:r.offsets[hi]].copy(), Ft.numpy()[lo:hi].copy(), nbytes))
    finally:
        dist.destroy_process_group()


def _run(div, world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_, div, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("mode", ["exchange", "halo"])
def test_two_rank_slabs_match_single_process(mode):
    div = (3, 2, 2)  # per rank: 3 x 2 cubes, 2 cube layers
    world = 2
    out = _run(div, world, mode)
    nodes, elems = port.generate_grid("tet4", [1.0] * 3, [3, 2, 2 * world])
    r = port.Routing(nodes.shape[0], port.dofmap("tet4", elems, 1))
    K, F, _ = port.assemble("tet4", nodes, elems, r, sources=[1.0])
    layer = 4 * 3
    covered = 0
    for rank, g0, g1, offs, Kr, Fr, nbytes in out:
        assert np.array_equal(offs, r.offsets[g0:g1 + 1] - r.offsets[g0]), "row pattern of the slab"
        Kg = K[r.offsets[g0]:r.offsets[g1]]
        Fg = F[g0:g1]
        if mode == "halo" or rank == 0:
            assert_bitwise(Kr, Kg, f"rank {rank} K")
            assert_bitwise(Fr, Fg, f"rank {rank} F")
            if mode == "halo":
                assert nbytes == 0
        else:
            # interface layer (first node layer of rank 1): lower + upper partial
            n_if = int(offs[layer])
            assert_scaled_close(Kr[:n_if], Kg[:n_if], what="interface K")
            assert_scaled_close(Fr[:layer], Fg[:layer], what="interface F")
            assert_bitwise(Kr[n_if:], Kg[n_if:], "interior K")
            assert_bitwise(Fr[layer:], Fg[layer:], "interior F")
            assert nbytes > 0
        covered += g1 - g0
    assert covered == nodes.shape[0]


def test_slab_partition_covers_grid():
    for world in (1, 2, 4, 8):
        div = (4, 3, 2)
        rows = 0
        elems = 0
        for rank in range(world):
            s = D.slab(div, rank, world, "exchange")
            assert s.own_hi - s.own_lo == (div[2] + (rank == world - 1)) * s.layer
            assert s.elem_hi - s.elem_lo == 6 * div[0] * div[1] * div[2]
            assert s.sends_up == (rank < world - 1) and s.receives_down == (rank > 0)
            rows += s.own_hi - s.own_lo
            elems += s.elem_hi - s.elem_lo
        assert rows == (div[0] + 1) * (div[1] + 1) * (div[2] * world + 1)
        assert elems == 6 * div[0] * div[1] * div[2] * world


def _field_worker(rank, world, port_, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_05052_b200 import meshgen
        nodes, elems = meshgen.unstructured_tri(16)
        B = 7
        b0, b1 = D.field_shard(B, rank, world)
        rho = meshgen.batch_fields(B, elems.shape[0])[b0:b1]
        r = port.Routing(nodes.shape[0], port.dofmap("tri3", elems, 1))
        K = np.stack([port.assemble("tri3", nodes, elems, r, diffusion=("element", rho[i]))[0]
                      for i in range(b1 - b0)]) if b1 > b0 else np.zeros((0, r.nnz))
        # gather the shards (the bench needs no collective; this only checks the union)
        sizes = [None] * world
        dist.all_gather_object(sizes, (b0, b1))
        out = [None] * world
        dist.all_gather_object(out, K)
        if rank == 0:
            q.put((sizes, np.concatenate(out)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_c4_field_sharding_covers_every_field_once(world):
    """C4 field sharding (dist.field_shard, bench.py c4): contiguous disjoint
    shards covering all fields; the gathered per-field assemblies equal the
    single-process batch bit for bit."""
    from paper_2602_05052_b200 import meshgen
    nodes, elems = meshgen.unstructured_tri(16)
    B = 7
    rho = meshgen.batch_fields(B, elems.shape[0])
    r = port.Routing(nodes.shape[0], port.dofmap("tri3", elems, 1))
    want = np.stack([port.assemble("tri3", nodes, elems, r, diffusion=("element", rho[b]))[0] for b in range(B)])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_field_worker, args=(rk, world, port_, q)) for rk in range(world)]
    for p in procs:
        p.start()
    sizes, got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sizes[0][0] == 0 and sizes[-1][1] == B
    assert all(sizes[i][1] == sizes[i + 1][0] for i in range(world - 1))
    assert_bitwise(got, want, "sharded fields")
