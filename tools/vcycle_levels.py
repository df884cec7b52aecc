"""Per-level cost of the V(3,3) cycle on the 480-macro shell: time one cycle
from level Lt down to L = 2 for Lt = 3..7 (differences = cost of level Lt),
plus the profile split of the full cycle (development tool)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1608_06473_b200 as hhg
import synth

L = int(sys.argv[1]) if len(sys.argv) > 1 else 7
mesh = synth.shell_mesh(0.55, 1.0, 1, 2)
ctx = hhg.Ctx.from_mesh(mesh, L)
ctx.fit(2)
for Lt in range(3, L + 1):
    n_local, n_owned, n_global = ctx.layout(Lt)
    g = np.arange(n_global)
    u, f = ctx.zeros(Lt), ctx.zeros(Lt)
    ctx.scatter_global(Lt, torch.from_numpy(synth.uniform_pm1(0, g)).cuda(), u)
    ctx.scatter_global(Lt, torch.from_numpy(synth.uniform_pm1(1, g)).cuda(), f)
    ctx.vcycle(Lt, u, f, n_cycles=1)
    torch.cuda.synchronize()
    ctx.profile(True)
    ctx.profile_read()
    l0 = ctx.kernel_launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.vcycle(Lt, u, f, n_cycles=2)
    e1.record()
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile(False)
    parts = " ".join(f"{k}={v[0] / 2:.2f}" for k, v in prof.items() if v[1])
    tprof = e0.elapsed_time(e1) / 2
    lpc = (ctx.kernel_launches - l0) / 2
    ctx.vcycle(Lt, u, f, n_cycles=2)  # unprofiled (HHG_VCYCLE_GRAPH=1: captures the graph)
    e0.record()
    ctx.vcycle(Lt, u, f, n_cycles=3)  # unprofiled (replays the cached graph with HHG_VCYCLE_GRAPH=1)
    e1.record()
    torch.cuda.synchronize()
    t3 = e0.elapsed_time(e1) / 3
    print(f"levels 2..{Lt}: eager {tprof:.2f} ms/cycle (profiled), unprofiled {t3:.2f} ms/cycle, "
          f"launches/cycle {lpc:.0f}  [{parts}]",
          flush=True)
