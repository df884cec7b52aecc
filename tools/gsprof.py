"""Cycle breakdown of the quad GS kernel (instrumented build tools/prof/libhhg_prof.so)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1608_06473_b200 as hhg
hhg.LIB_PATH = os.path.join(ROOT, "tools", "prof", "libhhg_prof.so")
import numpy as np, torch, synth
os.environ.setdefault("HHG_GS_KERNEL", "items")
mesh = synth.shell_mesh(0.55, 1.0, 1, 2)
L = 7
ctx = hhg.Ctx.from_mesh(mesh, L)
ctx.fit(2)
n_local, n_owned, n_global = ctx.layout(L)
g = np.arange(n_global)
u, f = ctx.zeros(L), ctx.zeros(L)
ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(0, g)).cuda(), u)
ctx.scatter_global(L, torch.from_numpy(synth.uniform_pm1(1, g)).cuda(), f)
lib = hhg.lib()
buf = (ctypes.c_ulonglong * 12)()
ctx.gs_sweep(L, u, f, 1); torch.cuda.synchronize(); lib.hhg_gs_prof_read(buf)
ctx.gs_sweep(L, u, f, 1); torch.cuda.synchronize(); lib.hhg_gs_prof_read(buf)
v = list(buf)
tot = v[3]
if os.environ["HHG_GS_KERNEL"] == "quad":
    print("CTA-cycles total %.3e, data-wait %.1f%%, barrier %.1f%%, item-start %.1f%%, quads %d, cycles/quad/CTA %.0f" % (
        tot, 100 * v[0] / tot, 100 * v[1] / tot, 100 * v[2] / tot, v[4], tot / max(v[4], 1)))
else:
    print("items: CTA-cycles total %.3e: flag waits %.1f%%, passes %.1f%% (of which refill issue %.1f%%, "
          "quad waits %.1f%%, node compute %.1f%%, refill barrier %.1f%%, pass start %.1f%%, final waits %.1f%%, "
          "end barrier %.1f%%), item setup %.1f%%" % (
              tot, 100 * v[0] / tot, 100 * v[1] / tot, 100 * v[2] / tot, 100 * v[5] / tot, 100 * v[6] / tot,
              100 * v[7] / tot, 100 * v[8] / tot, 100 * v[9] / tot, 100 * v[10] / tot, 100 * v[4] / tot))
