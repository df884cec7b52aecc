#!/usr/bin/env python
"""Benchmark: surrogate stencil apply + multicolour GS sweep (fp64) on B200.

Metric (BASELINE.json): "GLUP/s surrogate stencil apply + GS sweep (fp64) at
1/2/4/8 B200; % HBM roofline".  One step = one surrogate apply y = L~u plus
one full multicolour GS sweep on u (every unknown updated once by each), i.e.
2 * n_unknowns lattice updates per step.

Workload at N = 1: BASELINE config 4's per-GPU weak-scaling load -- the
480-macro shell (t=1, n_r=2), L = 7, q = 2 LSQP (j = 2), 167,117,310 unknowns,
inputs (1.4 GB per vector) far larger than L2.

`--impl reference` times the CPU oracle (oracle/) on a bounded sample of the
same workload on the host cores (the reference arm for this paper-only tier).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GLUP/s surrogate stencil apply + GS sweep (fp64) at 1/2/4/8 B200; % HBM roofline"
UNIT = "GLUP/s"
# fp64 floor of the apply: 45 DFMA per volume unknown (15 weights x 2 + 15,
# SURVEY 8(d)); peak measured by tools/peak_fp64.cu on a B200 at 1965 MHz
DFMA_PER_UNKNOWN = 45
DFMA_PER_S = 148 * 58.8 * 1965e6


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--t", type=int, default=1, help="icosahedral refinements")
    p.add_argument("--nr", type=int, default=2, help="radial layers")
    p.add_argument("--L", type=int, default=7)
    p.add_argument("--q", type=int, default=2)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extras", action="store_true")
    p.add_argument("--transport", default="nccl", choices=["nccl", "host"],
                   help="multi-rank exchange: NCCL (production) or host/gloo (functional check of the "
                        "multi-rank path with several ranks sharing one GPU)")
    return p.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
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
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi samples"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------
# CPU oracle leg (cpu_baseline and --impl reference)
# ----------------------------------------------------------------------------
def oracle_sample(L, q, n_macros=1):
    """The oracle on a bounded sample of the workload: the first `n_macros`
    macros of the same shell at the same level, as a stand-alone mesh with all
    outer faces Dirichlet.  Returns (n_unknowns, step_fn)."""
    import numpy as np

    import synth
    from oracle import geometry as G, solvers, surrogate as S
    sh = synth.shell_mesh(0.55, 1.0, 1, 2)
    tets = sh.tets[:n_macros]
    vids = np.unique(tets)
    remap = {int(v): i for i, v in enumerate(vids)}
    t2 = np.vectorize(remap.get)(tets)
    mesh = synth.MacroMesh(sh.vertices[vids], sh.radius[vids], t2, np.ones_like(t2, dtype=np.uint8))
    num = G.Numbering(mesh, 2 ** L)
    t_setup = time.perf_counter()
    Lt, _, _ = S.surrogate_operator(mesh, L, q, num=num)
    oracle_sample.setup_s = time.perf_counter() - t_setup  # FEM sampling + LSQP fit + CSR assembly
    gs = solvers.GS(Lt, num)
    g = np.arange(num.n_total)
    u = synth.uniform_pm1(0, g) * num.unknown_mask
    f = synth.uniform_pm1(1, g) * num.unknown_mask
    n_unk = int(num.unknown_mask.sum())

    def step():
        y = solvers.apply(Lt, num, u)
        gs.sweep(u.copy(), f)
        return y
    return n_unk, step, f"oracle (scipy CSR SpMV + colour-step GS) on {n_macros} macro(s) of the 480-macro shell at L={L}"


def workload(a, ws):
    """(t, n_r, workload string) of the bench configuration at ws GPUs --
    weak scaling (BASELINE config 4): ~480 macros per GPU;
    1: t=1 n_r=2 (480), 2: t=1 n_r=4 (960), 4: t=2 n_r=2 (1920), 8: t=2 n_r=4 (3840)."""
    t, nr = a.t, a.nr
    if ws > 1 and (a.t, a.nr) == (1, 2):
        t, nr = {2: (1, 4), 4: (2, 2), 8: (2, 4)}.get(ws, (1, 2 * ws))
    nt = 60 * 4 ** t * nr
    return t, nr, f"shell t={t} n_r={nr} ({nt} macros) L={a.L} q={a.q} LSQP j=2, apply + 1 GS sweep"


def run_reference(a):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    L = min(a.L, 7)
    n_unk, step, sample = oracle_sample(L, a.q, 1)
    for _ in range(max(a.warmup, 0)):
        step()
    ts = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    t = sum(ts) / len(ts)
    value = 2 * n_unk / t / 1e9
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": workload(a, ws)[2], "sample": sample},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------
# GPU leg
# ----------------------------------------------------------------------------
def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import numpy as np
    import torch

    import paper_1608_06473_b200 as hhg
    import synth

    ws, rank, local = dist_env()
    host_tr = a.transport == "host"
    if host_tr:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        if host_tr:
            dist.init_process_group("gloo")
            hhg.set_torch_transport()
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    rdev = torch.device("cpu") if host_tr else dev  # device of the reduction tensors
    stream = torch.cuda.current_stream(dev)
    L, q = a.L, a.q
    t_ref, nr_ref, workload_str = workload(a, ws)
    mesh = synth.shell_mesh(0.55, 1.0, t_ref, nr_ref)
    t0 = time.time()
    if ws > 1:
        # one process per GPU; the library's ghost exchange runs over NCCL;
        # RCB partition of the radial columns (whole columns per rank, 480 macros
        # each, 144 cut faces per GPU at 8 GPUs -- half the contiguous split's)
        owner = hhg.partition_rcb(mesh.vertices, mesh.tets, ws)
        if host_tr:
            ctx = hhg.Ctx.from_mesh(mesh, L, stream=stream.cuda_stream, rank=rank, nranks=ws, owner=owner)
        else:
            nid = [hhg.nccl_unique_id() if rank == 0 else None]  # the library's own NCCL creates the id
            dist.broadcast_object_list(nid, src=0)
            ctx = hhg.Ctx.from_mesh(mesh, L, stream=stream.cuda_stream, rank=rank, nranks=ws, owner=owner,
                                    nccl_id=nid[0])
    else:
        ctx = hhg.Ctx.from_mesh(mesh, L, stream=stream.cuda_stream)
    ctx.fit(q, "lsqp", 2)
    torch.cuda.synchronize()
    t_setup = time.time() - t0
    n_local, n_owned, n_global = ctx.layout(L)
    n_owned_total = n_owned
    if ws > 1:
        tt = torch.tensor([float(n_owned)], device=rdev)
        dist.all_reduce(tt)
        n_owned_total = int(tt.item())
    # inputs: seeded U[-1,1] on canonical ids (generated on the host once)
    unk = np.ones(n_global, dtype=bool)
    g = np.arange(n_global, dtype=np.int64)
    u_g = synth.uniform_pm1(0, g)
    f_g = synth.uniform_pm1(1, g)
    del g, unk
    u = ctx.zeros(L)
    f = ctx.zeros(L)
    y = ctx.zeros(L)
    ctx.scatter_global(L, torch.from_numpy(u_g).to(dev), u)
    ctx.scatter_global(L, torch.from_numpy(f_g).to(dev), f)
    del u_g, f_g
    torch.cuda.synchronize()

    def step():
        ctx.apply(L, u, y)
        ctx.gs_sweep(L, u, f, 1)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.kernel_launches
    ctx.profile(True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(a.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    ctx.profile(False)
    launches = ctx.kernel_launches - launches0
    ms = ev0.elapsed_time(ev1) / a.steps
    if dist:
        tt = torch.tensor([ms], device=rdev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    lups_step = 2 * n_owned_total
    value = lups_step / (ms * 1e-3) / 1e9
    prof = ctx.profile_read()
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    # dominant kernel: volume kernels; algorithmic bytes per volume unknown:
    # apply 16 B (u in, y out), GS 24 B (u in, f in, u out) -- SURVEY 8(d)
    nt_local = ctx.plan_info(L)["local_macros"] if ws > 1 else ctx.nt  # this rank's macros (timed kernels)
    nvol = nt_local * ((2 ** L - 1) * (2 ** L - 2) * (2 ** L - 3) // 6)
    va_ms, va_n = prof["vol_apply"]
    vg_ms, vg_n = prof["vol_gs"]
    roof = None
    if va_n:
        # dominant volume kernel; algorithmic bytes per volume unknown:
        # apply 16 B (u in, y out), GS sweep 24 B (u, f in; u out) -- one apply and
        # one sweep per step, whatever the number of launches they take
        dom = max(("vol_apply", va_ms, 16, va_n), ("vol_gs", vg_ms, 24, vg_n), key=lambda t: t[1])
        name, tot_ms, bpu, n_launch = dom
        achieved = nvol * bpu * a.steps / (tot_ms * 1e-3) / 1e9
        kname = "k_gs_items" if name == "vol_gs" else "k_vol_march"
        traffic, tsrc = None, None
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[kname]
            traffic, tsrc = tr["bytes"], tr["source"]
        except Exception:
            pass
        roof = {"kernel": "k_gs_items (4-colour GS sweep)" if name == "vol_gs" else "k_vol_march (apply)",
                "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "traffic_source": tsrc,
                "algorithmic_bytes_per_launch": nvol * bpu,
                "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)",
                "bytes_per_unknown": bpu, "units_per_launch": nvol * a.steps // max(n_launch, 1),
                "launches": n_launch, "avg_launch_ms": tot_ms / max(n_launch, 1),
                "share_of_step": tot_ms / (ms * a.steps),
                "apply_frac": nvol * 16 * a.steps / (va_ms * 1e-3) / 1e9 / hbm,
                "gs_frac": (nvol * 24 * a.steps / (vg_ms * 1e-3) / 1e9 / hbm) if vg_n else None}
        # the apply is HBM- AND fp64-bound: 16 B and 45 DFMA per
        # volume unknown; its roofline time is the larger of the two floors
        t_apply = va_ms * 1e-3 / a.steps
        t_hbm = nvol * 16 / (hbm * 1e9)
        t_fp64 = nvol * DFMA_PER_UNKNOWN / (DFMA_PER_S * (clk.summary().get("sm_mhz") or 1965.0) / 1965.0)
        roof["apply_roofline"] = {"bound": "fp64" if t_fp64 > t_hbm else "hbm", "t_hbm_ms": t_hbm * 1e3,
                                  "t_fp64_ms": t_fp64 * 1e3, "t_measured_ms": t_apply * 1e3,
                                  "frac": max(t_hbm, t_fp64) / t_apply,
                                  "fp64_peak_dfma_per_s": DFMA_PER_S,
                                  "fp64_peak_source": "tools/peak_fp64.cu on a B200 (58.8 DFMA/clk/SM at 1965 MHz)"}
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
            roof["fp64_pipe_pct"] = {k: v.get("fp64_pipe_pct") for k, v in tr.items()
                                     if isinstance(v, dict) and v.get("fp64_pipe_pct") is not None}
        except Exception:
            pass
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": workload_str, "unknowns": n_owned_total,
                      "macros_per_gpu": mesh.nt // ws,
                      "parallelism": (f"RCB radial-column macro partition over {ws} ranks, "
                                      + ("host (gloo) ghost exchange, ranks sharing a GPU: functional check, "
                                         "not a performance number" if host_tr else "NCCL ghost exchange"))
                      if ws > 1 else "1 GPU",
                      "l2": "inputs larger than L2 (1 vector = %.2f GB)" % (n_local * 8 / 1e9),
                      "setup_s": round(t_setup, 2)},
           "gpu_launches": launches,
           "roofline": roof,
           "clocks": clk.summary(),
           "profile_ms": prof}
    if not a.no_extras:
        # every rank takes part (apply / GS / V-cycle are collectives over the
        # ranks' ghost exchange); times are the max over ranks
        def tmax(x):
            if not dist:
                return x
            tt = torch.tensor([float(x)], device=rdev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            return float(tt.item())
        ee = e2e(ctx, L, u, f, y, a, n_owned_total, tmax)
        cmp = comparisons(ctx, L, u, f, y, n_owned_total, tmax)
        if rank == 0:
            out["e2e"] = ee
            out["comparisons"] = cmp
            if ws == 1:
                out["comparisons"].update(other_configs(stream, q))
    if rank == 0 and not a.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(L, q)
        if ws == 1:
            out["cpu_baseline"]["parity_of_timed_step"] = step_parity(ctx, mesh, L, q, u, f, y, step)
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()


def e2e(ctx, L, u, f, y, a, n_owned, tmax):
    """Same metric through the C-ABI with HOST buffers: the library stages
    u (apply), u and f (GS) host->device and y, u device->host every step."""
    import torch
    hu = u.cpu().pin_memory()
    hf = f.cpu().pin_memory()
    hy = torch.empty_like(hu).pin_memory()
    step = lambda: (ctx.apply(L, hu.numpy(), hy.numpy()), ctx.gs_sweep(L, hu.numpy(), hf.numpy(), 1))
    step()
    torch.cuda.synchronize()
    n = max(1, min(a.steps, 5))
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    torch.cuda.synchronize()
    t = tmax((time.perf_counter() - t0) / n)
    nb = hu.numel() * 8
    return {"value": 2 * n_owned / t / 1e9, "unit": UNIT, "h2d_bytes_per_step": 3 * nb,
            "d2h_bytes_per_step": 2 * nb, "ms_per_step": t * 1e3}


def comparisons(ctx, L, u, f, y, n_owned, tmax):
    """Per-operation rates on the same workload: surrogate
    residual and GS sweep alone; comparison operators (a11/a12): element-wise
    on-the-fly FEM apply and constant-stencil (affine) apply, GLUP/s."""
    import torch
    res = {}
    r = torch.empty_like(y)
    uu = u.clone()
    for name, fn, reps in (("surrogate_residual", lambda: ctx.residual(L, u, f, r), 5),
                           ("surrogate_gs_sweep", lambda: ctx.gs_sweep(L, uu, f, 1), 5)):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = tmax(e0.elapsed_time(e1) / reps)
        res[name] = {"ms": ms, "glups": n_owned / (ms * 1e-3) / 1e9}
    del r, uu
    for op, reps in (("surrogate", 5), ("const", 5), ("fem", 2)):
        ctx.apply(L, u, y, op=op)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            ctx.apply(L, u, y, op=op)
        e1.record()
        torch.cuda.synchronize()
        ms = tmax(e0.elapsed_time(e1) / reps)
        res[f"{op}_apply"] = {"ms": ms, "glups": n_owned / (ms * 1e-3) / 1e9}
    # BASELINE config 5 on this GPU's mesh: V(3,3) cycles, levels 2..L, surrogate
    # GS smoother on every level, 50 CG iterations at L = 2 (u, f ~ U[-1,1]).
    uu = u.clone()
    ff = f.clone()
    ctx.vcycle(L, uu, ff, n_cycles=1)
    torch.cuda.synchronize()
    uu.copy_(u)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ncyc = 3
    e0.record()
    hist = ctx.vcycle(L, uu, ff, n_cycles=ncyc)
    e1.record()
    torch.cuda.synchronize()
    rates = [hist[i + 1] / hist[i] for i in range(ncyc) if hist[i] > 0]
    res["vcycle_V33"] = {"ms_per_cycle": tmax(e0.elapsed_time(e1) / ncyc), "levels": f"2..{L}",
                         "residual_history": [float(h) for h in hist],
                         "reduction_per_cycle": [float(r) for r in rates]}
    # double discretisation: surrogate smoother, element-wise
    # FEM residual on every level; history = exact-operator residual
    uu.copy_(u)
    e0.record()
    hist = ctx.vcycle(L, uu, ff, n_cycles=ncyc, residual_op="fem")
    e1.record()
    torch.cuda.synchronize()
    res["vcycle_V33_DD"] = {"ms_per_cycle": tmax(e0.elapsed_time(e1) / ncyc), "levels": f"2..{L}",
                            "residual_history": [float(h) for h in hist]}
    return res


def other_configs(stream, q):
    """BASELINE configs 2 and 3 as context lines (1 GPU): config 2 = the single
    curved tet at L = 7 (333,375 unknowns, 2.7 MB per vector: L2-resident and
    launch-bound, reported as-is), apply + 1 GS sweep per step, and the same
    tet as a batch of 480 copies (160 M unknowns: the roofline-
    relevant single-tet number; every face Dirichlet, so volume kernels only);
    config 3 = the 480-macro shell at L = 6 (20.8 M unknowns), residual + 2 GS
    sweeps per step."""
    import numpy as np
    import torch

    import paper_1608_06473_b200 as hhg
    import synth
    res = {}
    for name, mesh, L, kind in (("config2_single_tet_L7", synth.single_tet(), 7, "apply+gs"),
                                ("config2_tet_batch480_L7", synth.tet_batch(480), 7, "apply+gs"),
                                ("config3_shell480_L6", synth.shell_mesh(0.55, 1.0, 1, 2), 6, "resid+2gs")):
        ctx = hhg.Ctx.from_mesh(mesh, L, stream=stream.cuda_stream)
        ctx.fit(q, "lsqp", 2)
        n_local, n_owned, n_global = ctx.layout(L)
        g = np.arange(n_global, dtype=np.int64)
        u, f, y = ctx.zeros(L), ctx.zeros(L), ctx.zeros(L)
        ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(0, g)).cuda(), u)
        ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(1, g)).cuda(), f)

        def step():
            if kind == "apply+gs":
                ctx.apply(L, u, y)
                ctx.gs_sweep(L, u, f, 1)
            else:
                ctx.residual(L, u, f, y)
                ctx.gs_sweep(L, u, f, 2)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        reps = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        lups = (2 if kind == "apply+gs" else 3) * n_owned
        res[name] = {"step": kind, "unknowns": n_owned, "ms_per_step": ms, "glups": lups / (ms * 1e-3) / 1e9,
                     "note": "L2-resident, launch-bound" if n_owned < 1e6 else "inputs larger than L2"}
        ctx.close()
    return res


def cpu_baseline_parallel(step, n_unk, sample, seconds=8.0):
    """The same oracle step run independently by one forked process per core
    of os.sched_getaffinity(0) (SciPy's SpMV is single-threaded): aggregate
    throughput of the host, reported beside the 1-core figure."""
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    ctx = mp.get_context("fork")
    q = ctx.Queue()

    def worker():
        n, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < seconds:
            step()
            n += 1
        q.put((n, time.perf_counter() - t0))
    procs = [ctx.Process(target=worker) for _ in range(cores)]
    for p in procs:
        p.start()
    res = [q.get(timeout=seconds * 20 + 120) for _ in procs]
    for p in procs:
        p.join()
    value = sum(2 * n_unk * n / t for n, t in res) / 1e9
    return {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": sample + f", one process per core, {seconds:.0f} s each"}


def step_parity(ctx, mesh, L, q, u, f, y, step):
    """Part of the oracle leg: one more bench step (apply + GS sweep) from a
    snapshot u0, and at sampled volume nodes of a few macros the oracle's own
    values (its LSQP fit of the node's macro; the GS update
    replayed on the node's dependency cone of interior volume nodes, DESIGN.md
    R13/R14): max |gpu - oracle| / (row magnitude)."""
    import numpy as np
    import torch
    try:
        from oracle import geometry as G, surrogate as S
        N = 2 ** L
        u0 = u.clone()
        step()
        torch.cuda.synchronize()
        num = G.Numbering(mesh, N)
        ug0, yg, ug1 = (np.asarray(ctx.gather_global(L, v)) for v in (u0, y, u))
        fg = np.asarray(ctx.gather_global(L, f))
        dirs = np.array(G.DIRS)
        rng = np.random.default_rng(2024)
        err_y, err_u, n = 0.0, 0.0, 0
        for T in rng.choice(mesh.nt, 3, replace=False):
            T = int(T)
            a_T = S.fit_macro(mesh, T, L, q, "lsqp", 2, blended=True)
            for _ in range(6):
                while True:
                    i, j, k = (int(x) for x in rng.integers(5, N - 5, 3))
                    if i + j + k <= N - 5:
                        break
                ijk = np.array([[i, j, k]])
                sw = S.eval_weights(a_T, ijk, N, q)[0]
                gI = int(num.gids(T, ijk)[0])
                un = ug0[num.gids(T, ijk + dirs)]
                err_y = max(err_y, abs(yg[gI] - float(np.dot(sw, un))) / float(np.abs(sw * un).sum()))
                memo = {}

                def new_value(p):
                    if p in memo:
                        return memo[p]
                    c = (p[0] + 2 * p[1] + 3 * p[2]) % 4
                    pp = np.array([p])
                    s2 = S.eval_weights(a_T, pp, N, q)[0]
                    acc = mag = 0.0
                    for w in range(15):
                        if w == 7:
                            continue
                        qn = (p[0] + dirs[w][0], p[1] + dirs[w][1], p[2] + dirs[w][2])
                        c2 = (qn[0] + 2 * qn[1] + 3 * qn[2]) % 4
                        v = new_value(qn)[0] if c2 < c else ug0[int(num.gids(T, np.array([qn]))[0])]
                        acc += s2[w] * v
                        mag += abs(s2[w] * v)
                    g = int(num.gids(T, pp)[0])
                    memo[p] = ((fg[g] - acc) / s2[7], (abs(fg[g]) + mag) / abs(s2[7]))
                    return memo[p]
                ref, scale = new_value((i, j, k))
                err_u = max(err_u, abs(ug1[gI] - ref) / scale)
                n += 1
        return {"nodes": n, "macros": 3, "apply_max_rel_err": err_y, "gs_max_rel_err": err_u,
                "tolerance": 1e-12, "how": "sampled volume nodes >= 5 steps from their macro boundary"}
    except Exception as e:  # pragma: no cover
        return {"failed": str(e)}


def cpu_baseline(L, q):
    try:
        n_unk, step, sample = oracle_sample(min(L, 7), q, 1)
        step()
        ts = []
        t_end = time.time() + 15
        while time.time() < t_end or len(ts) < 2:
            t0 = time.perf_counter()
            step()
            ts.append(time.perf_counter() - t0)
        t = statistics.median(ts)
        out = {"value": 2 * n_unk / t / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": sample + f", {len(ts)} reps, median",
               # the oracle's setup of the sample macro (FEM node
               # sampling, LSQP fit, CSR assembly of its operator) next to the
               # library's whole setup (config.setup_s: mesh, lattice, fit of
               # every macro; PAPER.md:1205-1214 Table setup)
               "setup_s_per_macro": round(getattr(oracle_sample, "setup_s", float("nan")), 2)}
        out["all_cores"] = cpu_baseline_parallel(step, n_unk, sample)
        return out
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": f"failed: {e}"}


if __name__ == "__main__":
    main()
