"""BASELINE config 5 on ONE GPU: V(3,3) cycles on the 3840-macro shell (t=2, n_r=4),
levels 2..L, surrogate GS smoother, 50 CG at L=2; u0, f ~ U[-1,1] (seeded).
Also times apply + GS sweep on that mesh (config 4's 8-GPU load on one GPU).
usage: python tools/vcycle_big.py [L] [cycles]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1608_06473_b200 as hhg
import synth

L = int(sys.argv[1]) if len(sys.argv) > 1 else 7
ncyc = int(sys.argv[2]) if len(sys.argv) > 2 else 3
mesh = synth.shell_mesh(0.55, 1.0, 2, 4)
t0 = time.time()
ctx = hhg.Ctx.from_mesh(mesh, L)
ctx.fit(2, "lsqp", 2)
torch.cuda.synchronize()
t_setup = time.time() - t0
n_local, n_owned, n_global = ctx.layout(L)
u, f, y = ctx.zeros(L), ctx.zeros(L), ctx.zeros(L)
chunk = 1 << 26
ug = torch.empty(n_global, dtype=torch.float64, device="cuda")
fg = torch.empty(n_global, dtype=torch.float64, device="cuda")
for s in range(0, n_global, chunk):
    g = np.arange(s, min(s + chunk, n_global))
    ug[s:s + len(g)] = torch.from_numpy(synth.uniform_pm1(0, g))
    fg[s:s + len(g)] = torch.from_numpy(synth.uniform_pm1(1, g))
ctx.scatter_global(L, ug, u)
ctx.scatter_global(L, fg, f)
del ug, fg
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    ctx.apply(L, u, y); ctx.gs_sweep(L, u, f, 1)
e0.record()
for _ in range(3):
    ctx.apply(L, u, y); ctx.gs_sweep(L, u, f, 1)
e1.record(); torch.cuda.synchronize()
ms_step = e0.elapsed_time(e1) / 3
uu = u.clone()
ctx.vcycle(L, uu, f, n_cycles=1)
torch.cuda.synchronize()
uu.copy_(u)
e0.record()
hist = ctx.vcycle(L, uu, f, n_cycles=ncyc)
e1.record(); torch.cuda.synchronize()
vc_ms = e0.elapsed_time(e1) / ncyc
# double discretisation (surrogate smoother, element-wise FEM residual on every level)
uu.copy_(u)
e0.record()
hist_dd = ctx.vcycle(L, uu, f, n_cycles=ncyc, residual_op="fem")
e1.record(); torch.cuda.synchronize()
dd_ms = e0.elapsed_time(e1) / ncyc
out = {"mesh": "shell t=2 n_r=4 (3840 macros)", "L": L, "unknowns": n_owned, "setup_s": round(t_setup, 2),
       "apply_plus_gs_ms": ms_step, "glups": 2 * n_owned / (ms_step * 1e-3) / 1e9,
       "vcycle_ms": vc_ms, "vcycle_dd_ms": dd_ms, "dd_residual_history": [float(h) for h in hist_dd],
       "residual_history": [float(h) for h in hist],
       "reduction_per_cycle": [float(hist[i + 1] / hist[i]) for i in range(ncyc)],
       "gpu_mem_gb": torch.cuda.max_memory_allocated() / 1e9}
print(json.dumps(out), flush=True)
