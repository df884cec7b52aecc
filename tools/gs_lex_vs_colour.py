"""Lexicographic vs 4-colour GS on the 480-macro shell, L = 7: time per sweep and V(3,3) convergence per cycle."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, paper_1608_06473_b200 as hhg, synth
m = synth.shell_mesh(0.55, 1.0, 1, 2); L = 7
ctx = hhg.Ctx.from_mesh(m, L); ctx.fit(2)
nl, no, ng = ctx.layout(L)
g = np.arange(ng)
u0, f = ctx.zeros(L), ctx.zeros(L)
ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(0, g)).cuda(), u0)
ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(1, g)).cuda(), f)
for lex in (False, True):
    u = u0.clone()
    ctx.gs_sweep(L, u, f, 1, lexicographic=lex); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): ctx.gs_sweep(L, u, f, 1, lexicographic=lex)
    e1.record(); torch.cuda.synchronize()
    sweep_ms = e0.elapsed_time(e1) / 5
    u = u0.clone()
    ctx.vcycle(L, u, f, n_cycles=1, lexicographic=lex); torch.cuda.synchronize()
    u = u0.clone()
    e0.record()
    hist = ctx.vcycle(L, u, f, n_cycles=6, lexicographic=lex)
    e1.record(); torch.cuda.synchronize()
    print("lex" if lex else "colour", "sweep ms", sweep_ms, "vcycle ms/cycle", e0.elapsed_time(e1) / 6, "rates", [round(float(hist[i+1]/hist[i]), 3) for i in range(6)], flush=True)
