"""Multi-rank host logic on CPU (gloo, world size 2, 3, 4 and 8 -- the last two on
the bench's 4- and 8-GPU weak-scaling meshes, 1920 and 3840 macros): macro partition,
owner-computes rows, ghost blocks and the exchange plan of libhhg, built in
plan-only contexts (no CUDA) and checked end to end: every requested node id
arrives from its owner (hhg_plan_check), and the owned unknowns of all ranks
add up to the oracle's unknown count exactly."""
import os
import socket

import numpy as np
import pytest

import synth
from oracle import geometry as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mesh_args, L, out_q, part="contig"):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_1608_06473_b200 as hhg
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mesh = synth.shell_mesh(0.55, 1.0, *mesh_args)
        hhg.set_torch_transport(host_only=True)
        if part == "rcb":  # the bench's partition: whole radial columns
            from paper_1608_06473_b200.partition import partition_rcb
            owner = partition_rcb(mesh.vertices, mesh.tets, world)
        else:  # radial-layer-friendly contiguous split, but not aligned to layers
            owner = (np.arange(mesh.nt) * world) // mesh.nt
        ctx = hhg.Ctx.from_mesh(mesh, L, rank=rank, nranks=world, owner=owner)
        res = {}
        for lev in range(2, L + 1):
            res[lev] = (ctx.plan_info(lev), ctx.plan_check(lev))
        out_q.put((rank, res))
        ctx.close()
    except Exception as e:  # pragma: no cover
        out_q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mesh_args,L,part", [(2, (0, 2), 4, "contig"), (3, (0, 1), 3, "contig"),
                                                      (2, (1, 1), 3, "contig"), (4, (2, 2), 2, "contig"),
                                                      (8, (2, 4), 2, "contig"), (3, (0, 2), 3, "rcb"),
                                                      (4, (2, 2), 2, "rcb"), (8, (2, 4), 2, "rcb")])
def test_partition_plan_consistent(world, mesh_args, L, part):
    import torch.multiprocessing as mp
    import __graft_entry__ as ge
    ge.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mesh_args, L, q, part)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(results[r], str), results[r]
    mesh = synth.shell_mesh(0.55, 1.0, *mesh_args)
    for lev in range(2, L + 1):
        num = G.Numbering(mesh, 2 ** lev)
        owned = sum(results[r][lev][0]["owned"] for r in range(world))
        assert owned == int(num.unknown_mask.sum())
        sends = sum(results[r][lev][0]["send"] for r in range(world))
        recvs = sum(results[r][lev][0]["recv"] for r in range(world))
        assert sends == recvs > 0
        for r in range(world):
            assert results[r][lev][1] == 0          # no mismatched ids
            assert results[r][lev][0]["blocks"] > results[r][lev][0]["local_macros"]
