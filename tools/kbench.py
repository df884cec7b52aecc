"""Kernel-level timing of the volume/face passes (development tool, not the bench).

usage: python tools/kbench.py [t] [n_r] [L] [reps]
Prints, per operation, the device time of the whole call and of each kernel
class (hhg_profile: 0 volume apply/resid, 1 volume GS, 2 lower-primitive rows,
3 other), CUDA events on the library stream, inputs > L2.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1608_06473_b200 as hhg
import synth

if os.environ.get("KB_LIB"):  # variant build of the library (tools/prof/*.so)
    hhg.LIB_PATH = os.path.abspath(os.environ["KB_LIB"])


def main():
    t = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    nr = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    L = int(sys.argv[3]) if len(sys.argv) > 3 else 7
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    mesh = synth.shell_mesh(0.55, 1.0, t, nr)
    ctx = hhg.Ctx.from_mesh(mesh, L)
    ctx.fit(2)
    n_local, n_owned, n_global = ctx.layout(L)
    g = np.arange(n_global)
    u, f, y = ctx.zeros(L), ctx.zeros(L), ctx.zeros(L)
    ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(0, g)).cuda(), u)
    ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(1, g)).cuda(), f)
    torch.cuda.synchronize()
    ops = {
        "apply": lambda: ctx.apply(L, u, y),
        "resid": lambda: ctx.residual(L, u, f, y),
        "const": lambda: ctx.apply(L, u, y, op="const"),
        "gs": lambda: ctx.gs_sweep(L, u, f, 1),
    }
    sel = os.environ.get("KB_OPS", "apply,resid,const,gs").split(",")
    tag = os.environ.get("KB_TAG", "")
    for name in sel:
        fn = ops[name]
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ctx.profile(True)
        ctx.profile_read()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        prof = ctx.profile_read()
        ctx.profile(False)
        parts = " ".join(f"{k}={v[0] / reps:.3f}" for k, v in prof.items() if v[1])
        print(f"{tag} {name}: {ms:.3f} ms/call  {n_owned / ms / 1e6:.1f} GLUP/s  [{parts}]", flush=True)
    if os.environ.get("KB_CHECK"):  # fingerprint of one GS sweep from the seeded start (variant cross-check)
        ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(0, g)).cuda(), u)
        ctx.gs_sweep(L, u, f, 2)
        ug = np.asarray(ctx.gather_global(L, u), dtype=np.float64)
        print(f"{tag} check: sum={ug.sum():.17e} sumsq={np.dot(ug, ug):.17e}", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
