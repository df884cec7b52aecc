"""Small driver for ncu captures: one ctx, a few calls of one operation.

usage: python tools/prof_run.py [apply|resid|gs|const|fem] [t] [n_r] [L] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1608_06473_b200 as hhg
import synth


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "apply"
    t = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    nr = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    L = int(sys.argv[4]) if len(sys.argv) > 4 else 7
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
    mesh = synth.shell_mesh(0.55, 1.0, t, nr)
    ctx = hhg.Ctx.from_mesh(mesh, L)
    ctx.fit(2)
    n_local, n_owned, n_global = ctx.layout(L)
    g = np.arange(n_global)
    u, f, y = ctx.zeros(L), ctx.zeros(L), ctx.zeros(L)
    ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(0, g)).cuda(), u)
    ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(1, g)).cuda(), f)
    for _ in range(reps):
        if what == "apply":
            ctx.apply(L, u, y)
        elif what == "const":
            ctx.apply(L, u, y, op="const")
        elif what == "fem":
            ctx.apply(L, u, y, op="fem")
        elif what == "resid":
            ctx.residual(L, u, f, y)
        elif what == "gs":
            ctx.gs_sweep(L, u, f, 1)
    torch.cuda.synchronize()
    print("ok", what, n_owned)


if __name__ == "__main__":
    main()
