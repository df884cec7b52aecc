"""Cycle accounting of the single-pass GS kernel (hhg_gs_prof) on the bench
workload: where the first thread of every CTA spends a wavefront step.

usage: python tools/gsprof.py [t] [n_r] [L] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1608_06473_b200 as hhg
import synth

if os.environ.get("KB_LIB"):  # variant build of the library (tools/build_variant.py)
    hhg.LIB_PATH = os.path.abspath(os.environ["KB_LIB"])


def main():
    t = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    nr = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    L = int(sys.argv[3]) if len(sys.argv) > 3 else 7
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
    mesh = synth.shell_mesh(0.55, 1.0, t, nr)
    ctx = hhg.Ctx.from_mesh(mesh, L)
    ctx.fit(2)
    n_local, n_owned, n_global = ctx.layout(L)
    g = np.arange(n_global)
    u, f = ctx.zeros(L), ctx.zeros(L)
    ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(0, g)).cuda(), u)
    ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(1, g)).cuda(), f)
    ctx.gs_sweep(L, u, f, 1)
    ctx.gs_prof(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.gs_sweep(L, u, f, reps)
    e1.record()
    torch.cuda.synchronize()
    c = ctx.gs_prof(True, read=True).astype(np.float64)
    ctx.gs_prof(False)
    if os.environ.get("KB_ITEMS"):  # default k_gs_items sweep (instrumented instantiation): thread 0's cycles per phase
        tag = os.environ.get("KB_TAG", "items")
        items, steps = c[7] / reps, c[6] / reps
        print(f"{tag}: {e0.elapsed_time(e1) / reps:.3f} ms/sweep, items {items:.0f}, passes {4 * items:.0f}, "
              f"steps/pass {steps / max(4 * items, 1):.1f}")
        names = ["item fetch+setup", "flag wait", "start bar.sync", "pass march", "end bar.sync"]
        tot = sum(c[x] for x in range(5))
        for x, n in enumerate(names):
            print(f"   {n:17s} {c[x] / reps / max(4 * items, 1):9.0f} cyc/pass  {100 * c[x] / max(tot, 1):5.1f} %")
        ctx.close()
        return
    steps = c[6]
    names = ["plane wait", "node update", "halo wait", "progress", "barrier", "post-barrier"]
    tot = c[:6].sum()
    tag = os.environ.get("KB_TAG", os.environ.get("HHG_GS_KERNEL", "default"))
    print(f"{tag}: {e0.elapsed_time(e1) / reps:.3f} ms/sweep (whole call), items {c[7] / reps:.0f}, "
          f"steps/item {steps / max(c[7], 1):.1f}, cycles/step {tot / max(steps, 1):.0f}, "
          f"failed halo polls/step/CTA {c[8] / max(steps, 1):.1f}")
    for x, n in enumerate(names):
        print(f"   {n:13s} {c[x] / max(steps, 1):8.0f} cyc/step  {100 * c[x] / max(tot, 1):5.1f} %")
    ctx.close()


if __name__ == "__main__":
    main()
