"""Discretisation-error study of PAPER.md Sec. 4.1 / Table hHstudy
on the synthetic shells, solved on the GPU through the C-ABI.

Model problem -Laplace(u) = f on the shell r1 = 0.55 < r < 1, homogeneous
Dirichlet, exact solution u = (r - r1)(r - r2) sin(10x) sin(4y) sin(7z)
(PAPER.md:826-830), lumped right-hand side f_I = f(x_I) sum_{T ∋ I} |T| / 4
(oracle.fem.rhs_lumped, R20).  Error e = ||u_h - u(x_I)|| in the
lumped-mass discrete L2 norm sqrt(sum_I m_I e_I^2) over the unknowns.

  FEM:        u_h = CG on the exact (on-the-fly, element-wise) operator, run as a
              V-cycle whose coarsest level is the finest (hhg_vcycle L_coarse = L).
  LSQP/IPOLY: 10 V(3,3) cycles with the surrogate operator.
  LSQP2-DD:   10 V(3,3) cycles, surrogate smoother, exact residual.
  LSQP2-F:    10 V(3,3) cycles with surrogate face rows as well.

The paper's macro mesh is unknown: absolute values are context ("parity
unpinned"), the trends are the result (quadratic FEM convergence; surrogate
errors follow FEM until a plateau that drops with H and q).

usage: python tests/accuracy_study.py [out.txt]   (a few minutes on one B200)

Test infrastructure (it uses the oracle for the lumped right-hand side and
the node coordinates), kept under tests/ as the oracle rules require.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1608_06473_b200 as hhg
import synth
from oracle import fem, geometry as G

R1, R2 = 0.55, 1.0


def u_exact(x, y, z):
    r = np.sqrt(x * x + y * y + z * z)
    return (r - R1) * (r - R2) * np.sin(10 * x) * np.sin(4 * y) * np.sin(7 * z)


def f_exact(x, y, z):
    """-Laplace(u) for u = g(r) S(x,y,z): -(S Lg + 2 g'/r (x.grad S) + g LS)."""
    r = np.sqrt(x * x + y * y + z * z)
    g = (r - R1) * (r - R2)
    gp = 2 * r - (R1 + R2)
    lap_g = 6 - 2 * (R1 + R2) / r
    sx, sy, sz = np.sin(10 * x), np.sin(4 * y), np.sin(7 * z)
    S = sx * sy * sz
    xgS = x * 10 * np.cos(10 * x) * sy * sz + y * 4 * sx * np.cos(4 * y) * sz + z * 7 * sx * sy * np.cos(7 * z)
    return -(S * lap_g + 2 * gp / r * xgS - 165.0 * g * S)


def study(t, nr, levels, variants, cg_iters=3000, cycles=10):
    mesh = synth.shell_mesh(R1, R2, t, nr)
    rows = {}
    for L in levels:
        num = G.Numbering(mesh, 2 ** L)
        X = num.coords(True)
        unk = num.unknown_mask
        ue = np.where(unk, u_exact(X[:, 0], X[:, 1], X[:, 2]), 0.0)
        mass = fem.rhs_lumped(mesh, num, lambda x, y, z: np.ones_like(x))
        f = fem.rhs_lumped(mesh, num, f_exact)
        ctx = hhg.Ctx.from_mesh(mesh, L)
        df = ctx.zeros(L)
        ctx.scatter_global(L, torch.from_numpy(f).cuda(), df)
        res = {}
        for name, q, method in variants:
            du = ctx.zeros(L)
            try:
                res[name] = solve_error(ctx, L, du, df, name, q, method, cg_iters, cycles, unk, ue, mass)
            except hhg.HHGError as err:
                print(f"  {name}: {err}", flush=True)
                res[name] = float("nan")
        ctx.close()
        rows[L] = res
        print(f"  {mesh.nt} macros L={L}: " + " ".join(f"{k}={v:.2e}" for k, v in res.items()), flush=True)
    return mesh.nt, rows


def solve_error(ctx, L, du, df, name, q, method, cg_iters, cycles, unk, ue, mass):
    if name == "FEM":
        ctx.fit(2, "lsqp", 2)
        # CG on the exact operator: a "V-cycle" whose coarsest level is L itself
        # (level 2: every row is exact, l = 0)
        ctx.vcycle(L, du, df, n_cycles=1, L_coarse=L, cg_iters=cg_iters)
    elif method == "lsqp-faces":  # surrogate face rows too
        ctx.fit(q, "lsqp", 2)
        ctx.vcycle(L, du, df, n_cycles=cycles, op="surrogate_faces")
    elif method == "lsqp-dd":  # double discretisation: exact residual
        ctx.fit(q, "lsqp", 2)
        ctx.vcycle(L, du, df, n_cycles=cycles, residual_op="fem")
    else:
        ctx.fit(q, method, 2)
        ctx.vcycle(L, du, df, n_cycles=cycles)
    torch.cuda.synchronize()
    uh = ctx.gather_global(L, du)
    e = np.where(unk, uh - ue, 0.0)
    return float(np.sqrt(np.sum(mass * e * e)))


# IPOLY: the paper gives interpolation points for q = 2 only
VARIANTS = [("FEM", 0, None), ("LSQP1", 1, "lsqp"), ("LSQP2", 2, "lsqp"), ("LSQP3", 3, "lsqp"),
            ("IPOLY2", 2, "ipoly"), ("LSQP2-DD", 2, "lsqp-dd"), ("LSQP2-F", 2, "lsqp-faces")]


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    t0 = time.time()
    tables = [study(0, 1, [2, 3, 4, 5, 6], VARIANTS), study(1, 2, [2, 3, 4, 5], VARIANTS),
              study(2, 4, [2, 3, 4], VARIANTS)]
    lines = ["# Discretisation error (lumped-mass discrete L2), PAPER.md Table hHstudy setting on the",
             "# synthetic icosahedral shells (parity unpinned: the paper's macro mesh is unknown).",
             "# FEM: CG on the exact element-wise operator; LSQP/IPOLY: 10 V(3,3) cycles (j = 2).",
             "# '*' = relative deviation from e_FEM above 10 % (the paper's italic entries).",
             f"# tests/accuracy_study.py, {time.time() - t0:.0f} s"]
    for nt, rows in tables:
        lines.append(f"\n{nt} macros")
        names = [v[0] for v in VARIANTS]
        lines.append("L  " + "".join(f"{n:>11s}" for n in names) + "   FEM ratio")
        prev = None
        for L, res in rows.items():
            cells = []
            for n in names:
                v = res[n]
                mark = "*" if n != "FEM" and np.isfinite(v) and abs(v - res["FEM"]) > 0.1 * res["FEM"] else " "
                cells.append(f"{v:10.2e}{mark}")
            ratio = f"{prev / res['FEM']:.2f}" if prev else ""
            prev = res["FEM"]
            lines.append(f"{L}  " + "".join(cells) + f"   {ratio}")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write(text + "\n")


if __name__ == "__main__":
    main()
