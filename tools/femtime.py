"""Time the FEM (on-the-fly) vs surrogate apply on the 480-macro L7 shell."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_1608_06473_b200 as hhg
m = synth.shell_mesh(0.55, 1.0, 1, 2); L = int(sys.argv[1]) if len(sys.argv) > 1 else 7
ctx = hhg.Ctx.from_mesh(m, L); ctx.fit(2)
n_local, n_owned, n_global = ctx.layout(L)
u, y = ctx.zeros(L), ctx.zeros(L)
ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(0, np.arange(n_global))).cuda(), u)
for op in ("fem", "surrogate", "const"):
    ctx.apply(L, u, y, op=op); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): ctx.apply(L, u, y, op=op)
    e1.record(); torch.cuda.synchronize()
    print(op, "apply ms", e0.elapsed_time(e1) / 5, flush=True)
