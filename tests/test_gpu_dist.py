"""Multi-rank apply / residual / GS through the C-ABI: 2 or 4 ranks as processes
sharing cuda:0, exchanging ghost values through the library's host transport
(torch.distributed gloo; the NCCL transport moves the same buffers).  The
assembled result must match the single-process oracle to 1e-12."""
import os
import socket

import numpy as np
import pytest

import synth
from oracle import fem, geometry as G, solvers, surrogate as S

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mesh_args, L, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_1608_06473_b200 as hhg
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        mesh = synth.shell_mesh(0.55, 1.0, *mesh_args)
        hhg.set_torch_transport(host_only=False)
        owner = (np.arange(mesh.nt) * world) // mesh.nt
        ctx = hhg.Ctx.from_mesh(mesh, L, rank=rank, nranks=world, owner=owner)
        ctx.fit(2)
        n_local, n_owned, n_global = ctx.layout(L)
        g = np.arange(n_global)
        num = G.Numbering(mesh, 2 ** L)
        u = synth.uniform_pm1(0, g) * num.unknown_mask
        f = synth.uniform_pm1(1, g) * num.unknown_mask
        du, df, dy, dr = ctx.zeros(L), ctx.zeros(L), ctx.zeros(L), ctx.zeros(L)
        ctx.scatter_global(L, torch.from_numpy(u).cuda(), du)
        ctx.scatter_global(L, torch.from_numpy(f).cuda(), df)
        ctx.apply(L, du, dy)
        nrm = ctx.residual(L, du, df, dr, norm=True)
        ctx.gs_sweep(L, du, df, 2)
        torch.cuda.synchronize()
        out = {}
        for name, vec in (("y", dy), ("r", dr), ("u", du)):
            part = torch.from_numpy(ctx.gather_global(L, vec))
            dist.all_reduce(part)  # each entry owned by exactly one rank
            out[name] = part.numpy()
        out["norm"] = nrm
        out["owned"] = n_owned
        out_q.put((rank, out))
        ctx.close()
    except Exception as e:  # pragma: no cover
        import traceback
        out_q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mesh_args,L", [(2, (0, 2), 3), (2, (0, 2), 4), (4, (0, 2), 3)])
def test_two_ranks_match_oracle(world, mesh_args, L):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mesh_args, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    mesh = synth.shell_mesh(0.55, 1.0, *mesh_args)
    num = G.Numbering(mesh, 2 ** L)
    Lt, _, _ = S.surrogate_operator(mesh, L, 2, num=num)
    g = np.arange(num.n_total)
    u = synth.uniform_pm1(0, g) * num.unknown_mask
    f = synth.uniform_pm1(1, g) * num.unknown_mask
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    assert sum(res[r]["owned"] for r in range(world)) == int(num.unknown_mask.sum())
    assert rel(res[0]["y"], solvers.apply(Lt, num, u)) < 1e-12
    r_ref = solvers.residual(Lt, num, u, f)
    assert rel(res[0]["r"], r_ref) < 1e-12
    for r in range(world):
        assert abs(res[r]["norm"] - np.linalg.norm(r_ref)) < 1e-12 * np.linalg.norm(r_ref)
    u2 = solvers.GS(Lt, num).sweep(u.copy(), f, 2)
    assert rel(res[0]["u"], u2) < 1e-12


def _vworker(rank, world, port, mesh_args, L, cycles, out_q, part="contig"):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_1608_06473_b200 as hhg
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        mesh = synth.shell_mesh(0.55, 1.0, *mesh_args)
        hhg.set_torch_transport(host_only=False)
        owner = (hhg.partition_rcb(mesh.vertices, mesh.tets, world) if part == "rcb"
                 else (np.arange(mesh.nt) * world) // mesh.nt)
        ctx = hhg.Ctx.from_mesh(mesh, L, rank=rank, nranks=world, owner=owner)
        ctx.fit(2)
        n_local, n_owned, n_global = ctx.layout(L)
        g = np.arange(n_global)
        num = G.Numbering(mesh, 2 ** L)
        u = synth.uniform_pm1(7, g) * num.unknown_mask
        f = synth.uniform_pm1(8, g) * num.unknown_mask
        du, df = ctx.zeros(L), ctx.zeros(L)
        ctx.scatter_global(L, torch.from_numpy(u).cuda(), du)
        ctx.scatter_global(L, torch.from_numpy(f).cuda(), df)
        hist = ctx.vcycle(L, du, df, n_cycles=cycles)
        torch.cuda.synchronize()
        part = torch.from_numpy(ctx.gather_global(L, du))
        dist.all_reduce(part)
        out_q.put((rank, {"hist": hist, "u": part.numpy()}))
        ctx.close()
    except Exception:  # pragma: no cover
        import traceback
        out_q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mesh_args,L,cycles,world,part", [((0, 2), 4, 3, 2, "contig"), ((0, 2), 4, 2, 3, "rcb"),
                                                               ((0, 2), 4, 2, 3, "contig"), ((0, 2), 3, 1, 3, "rcb"),
                                                               ((0, 2), 3, 1, 2, "rcb")])
def test_two_rank_vcycle_matches_oracle(mesh_args, L, cycles, world, part):
    """V(3,3) with the macros split over 2 ranks (restriction partials of
    shared coarse nodes summed across ranks, prolongation re-synced): residual
    history and iterate agree with the single-process oracle to 1e-10."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_vworker, args=(r, world, port, mesh_args, L, cycles, q, part))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    mesh = synth.shell_mesh(0.55, 1.0, *mesh_args)
    H = solvers.Hierarchy(mesh, L, 2, 2)
    num = H.num[L]
    g = np.arange(num.n_total)
    u0 = synth.uniform_pm1(7, g) * num.unknown_mask
    f = synth.uniform_pm1(8, g) * num.unknown_mask
    u_ref, hist_ref = H.solve(u0.copy(), f, cycles)
    for r in range(world):
        assert np.all(np.abs(res[r]["hist"] - hist_ref) <= 1e-10 * hist_ref), (r, res[r]["hist"], hist_ref)
    rel = np.linalg.norm(res[0]["u"] - u_ref) / np.linalg.norm(u_ref)
    assert rel < 1e-10


def _bworker(rank, world, port, mesh_args, L, out_q, part):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_1608_06473_b200 as hhg
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        mesh = synth.shell_mesh(0.55, 1.0, *mesh_args)
        if world > 1:
            hhg.set_torch_transport(host_only=False)
            owner = (hhg.partition_rcb(mesh.vertices, mesh.tets, world) if part == "rcb"
                     else (np.arange(mesh.nt) * world) // mesh.nt)
            ctx = hhg.Ctx.from_mesh(mesh, L, rank=rank, nranks=world, owner=owner)
        else:
            ctx = hhg.Ctx.from_mesh(mesh, L)
        ctx.fit(2)
        n_local, n_owned, n_global = ctx.layout(L)
        g = np.arange(n_global)
        num = G.Numbering(mesh, 2 ** L)
        u = synth.uniform_pm1(0, g) * num.unknown_mask
        f = synth.uniform_pm1(1, g) * num.unknown_mask
        du, df, dy, dr = ctx.zeros(L), ctx.zeros(L), ctx.zeros(L), ctx.zeros(L)
        ctx.scatter_global(L, torch.from_numpy(u).cuda(), du)
        ctx.scatter_global(L, torch.from_numpy(f).cuda(), df)
        ctx.apply(L, du, dy)
        nrm = ctx.residual(L, du, df, dr, norm=True)
        ug = du.clone()
        ctx.gs_sweep(L, ug, df, 2)
        hist = ctx.vcycle(L, du, df, n_cycles=2)
        torch.cuda.synchronize()
        out = {"norm": nrm, "hist": hist}
        for name, vec in (("y", dy), ("r", dr), ("ug", ug), ("uv", du)):
            v = torch.from_numpy(ctx.gather_global(L, vec))
            if world > 1:
                dist.all_reduce(v)  # each entry owned by exactly one rank (+0.0 elsewhere: exact)
            out[name] = v.numpy()
        out_q.put((rank, out))
        ctx.close()
    except Exception:  # pragma: no cover
        import traceback
        out_q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _run(world, mesh_args, L, part):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bworker, args=(r, world, port, mesh_args, L, q, part)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    return res


@pytest.mark.parametrize("part", ["rcb", "contig"])
def test_results_bitwise_identical_across_rank_counts(part):
    """apply, residual and GS sweeps give BITWISE the same
    vectors on 1, 2, 3 and 4 ranks (every node's arithmetic is partition-
    independent: volume rows per macro, lower-primitive rows at their owner
    from the same stored rows); the residual norm and the V(3,3) history
    (sums over rank partials) agree to 1e-14 / 1e-12 and the V-cycle iterate
    to 1e-12."""
    mesh_args, L = (0, 2), 4
    ref = _run(1, mesh_args, L, part)[0]
    for world in (2, 3, 4):
        res = _run(world, mesh_args, L, part)
        for r in range(world):
            o = res[r]
            for name in ("y", "r", "ug"):
                assert np.array_equal(o[name], ref[name]), (world, r, name, np.abs(o[name] - ref[name]).max())
            assert abs(o["norm"] - ref["norm"]) <= 1e-14 * ref["norm"], (world, o["norm"], ref["norm"])
            assert np.all(np.abs(o["hist"] - ref["hist"]) <= 1e-12 * ref["hist"]), (world, o["hist"], ref["hist"])
            rel = np.linalg.norm(o["uv"] - ref["uv"]) / np.linalg.norm(ref["uv"])
            assert rel < 1e-12, (world, rel)


@pytest.mark.parametrize("env", [{"HHG_OVERLAP": "0"}, {"HHG_GS_KERNEL": "wide4"}, {"HHG_GS_KERNEL": "passes"}])
def test_rank_results_independent_of_overlap_and_gs_kernel(env, monkeypatch):
    """The exchange/compute overlap (on by default) and the choice of volume GS
    kernel do not change a single bit: 2 ranks with the overlap off, or with the
    single-pass wavefront / the colour-pass kernels, reproduce the 1-rank
    default vectors exactly."""
    mesh_args, L = (0, 2), 4
    ref = _run(1, mesh_args, L, "rcb")[0]
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    res = _run(2, mesh_args, L, "rcb")
    for r in range(2):
        for name in ("y", "r", "ug"):
            assert np.array_equal(res[r][name], ref[name]), (env, r, name)
