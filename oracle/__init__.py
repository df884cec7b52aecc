"""CPU oracle for the two-scale surrogate-stencil method (arXiv:1608.06473).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this
package.  The product path (paper_1608_06473_b200/, the C-ABI library) never
imports, links or calls it, and must fail loudly when its CUDA library is
missing instead of falling back here.

Plain, slow, obviously-correct fp64 NumPy/SciPy.  Each function cites the
PAPER.md passage it follows; readings of silent/garbled passages are the
DESIGN.md "readings" table (R1..).  It shares no code with the CUDA path: the
only common module is `synth/` (seeded inputs + macro meshes, no method
arithmetic).

Parity status: every function here is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py, except the one marked "parity unpinned" in its
docstring (absolute values of the paper's Table hHstudy -- not reproduced).
"""
from . import geometry, fem, surrogate, solvers  # noqa: F401
