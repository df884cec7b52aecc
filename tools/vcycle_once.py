"""One V(3,3) cycle on the 480-macro shell at L = 7 (for ncu launch lists of the multigrid kernels)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, paper_1608_06473_b200 as hhg, synth
if os.environ.get("KB_LIB"): hhg.LIB_PATH = os.path.abspath(os.environ["KB_LIB"])
m = synth.shell_mesh(0.55, 1.0, 1, 2); L = 7
ctx = hhg.Ctx.from_mesh(m, L); ctx.fit(2)
nl, no, ng = ctx.layout(L)
u, f = ctx.zeros(L), ctx.zeros(L)
g = np.arange(ng)
ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(0, g)).cuda(), u)
ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(1, g)).cuda(), f)
ctx.vcycle(L, u, f, n_cycles=1)
torch.cuda.synchronize()
