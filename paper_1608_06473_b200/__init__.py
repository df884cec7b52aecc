"""Python binding of libhhg (include/hhg.h): argument marshalling only.

Every step of the hot path runs in the CUDA library; this module only turns
torch tensors / numpy arrays into pointers and status codes into exceptions.
There is no CPU fallback: if libhhg.so is missing or fails to load, importing
`lib()` raises.  Build with `python -c "import __graft_entry__ as g; g.build()"`.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .partition import partition_rcb  # noqa: F401  (host logic: macro -> rank)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhhg.so")

OPS = {"surrogate": 0, "fem": 1, "fem_elementwise": 1, "const": 2, "const_affine": 2, "surrogate_faces": 3}
FIT = {"lsqp": 0, "ipoly": 1}
STATUS = {0: "HHG_OK", 1: "HHG_ERR_INVALID", 2: "HHG_ERR_MESH", 3: "HHG_ERR_FIT",
          4: "HHG_ERR_NUMERIC", 5: "HHG_ERR_DIVERGED", 6: "HHG_ERR_CUDA", 7: "HHG_ERR_NCCL",
          8: "HHG_ERR_OOM", 9: "HHG_ERR_STATE"}

_lib = None


class HHGError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {msg}")


def lib():
    """Load libhhg.so (fails loudly; no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    L.hhg_setup_macro_mesh.argtypes = [P, P, I64, P, I64, P, I32, P, I32, I32, P, P, ctypes.POINTER(P)]
    L.hhg_fit_surrogates.argtypes = [P, I32, I32, I32]
    L.hhg_gs_prof.argtypes = [P, I32, P]
    L.hhg_sample_nodes.argtypes = [P, I32, I32, I32, P, ctypes.POINTER(I64)]
    L.hhg_fit_from_samples.argtypes = [P, I32, I32, I32, I32, P]
    L.hhg_vector_layout.argtypes = [P, I32, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64)]
    L.hhg_apply.argtypes = [P, I32, I32, P, P]
    L.hhg_residual.argtypes = [P, I32, I32, P, P, P, P]
    L.hhg_gs_sweep.argtypes = [P, I32, I32, P, P, I32]
    L.hhg_vcycle.argtypes = [P, I32, I32, I32, I32, I32, I32, P, P, I32, P]
    L.hhg_vcycle_dd.argtypes = [P, I32, I32, I32, I32, I32, I32, I32, P, P, I32, P]
    L.hhg_vcycle_ex.argtypes = [P, I32, I32, I32, I32, I32, I32, I32, I32, P, P, I32, P]
    L.hhg_gs_sweep_lex.argtypes = [P, I32, I32, P, P, I32]
    L.hhg_gather_global.argtypes = [P, I32, P, P]
    L.hhg_scatter_global.argtypes = [P, I32, P, P]
    L.hhg_sync_copies.argtypes = [P, I32, P]
    L.hhg_eval_stencils.argtypes = [P, I32, I32, I64, P]
    L.hhg_set_host_transport.argtypes = [P, P, I32]
    L.hhg_set_host_transport.restype = ctypes.c_int
    L.hhg_plan_info.argtypes = [P, I32, ctypes.POINTER(I64)]
    L.hhg_plan_info.restype = ctypes.c_int
    L.hhg_plan_check.argtypes = [P, I32, ctypes.POINTER(I64)]
    L.hhg_plan_check.restype = ctypes.c_int
    L.hhg_profile.argtypes = [P, I32]
    L.hhg_profile.restype = ctypes.c_int
    L.hhg_profile_read.argtypes = [P, I32, ctypes.POINTER(D), ctypes.POINTER(I64)]
    L.hhg_profile_read.restype = ctypes.c_int
    L.hhg_kernel_launches.argtypes = [P]
    L.hhg_kernel_launches.restype = I64
    L.hhg_last_error.argtypes = [P]
    L.hhg_last_error.restype = ctypes.c_char_p
    L.hhg_destroy.argtypes = [P]
    L.hhg_nccl_unique_id.argtypes = [P]
    L.hhg_nccl_unique_id.restype = ctypes.c_int
    for name in ("hhg_setup_macro_mesh", "hhg_fit_surrogates", "hhg_vector_layout", "hhg_apply",
                 "hhg_residual", "hhg_gs_sweep", "hhg_gs_sweep_lex", "hhg_vcycle", "hhg_vcycle_dd",
                 "hhg_vcycle_ex", "hhg_gather_global",
                 "hhg_scatter_global", "hhg_sync_copies", "hhg_eval_stencils"):
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _ptr(x, n=None, writable=False):
    """Raw pointer of a float64 torch tensor (cuda or cpu) or numpy array."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if x.dtype != np.float64 or not x.flags["C_CONTIGUOUS"]:
            raise ValueError("numpy vectors must be C-contiguous float64")
        if n is not None and x.size < n:
            raise ValueError(f"vector too short: {x.size} < {n}")
        return x.ctypes.data
    import torch
    if not isinstance(x, torch.Tensor):
        raise TypeError(type(x))
    if x.dtype != torch.float64 or not x.is_contiguous():
        raise ValueError("torch vectors must be contiguous float64")
    if n is not None and x.numel() < n:
        raise ValueError(f"vector too short: {x.numel()} < {n}")
    return x.data_ptr()


HostExchangeFn = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                  ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p)
_keep_alive = []


def nccl_unique_id():
    """128-byte NCCL unique id from the library's own NCCL (rank 0 creates it,
    every rank passes it to Ctx.from_mesh(..., nccl_id=...))."""
    buf = ctypes.create_string_buffer(128)
    st = lib().hhg_nccl_unique_id(buf)
    if st != 0:
        raise HHGError(st, "ncclGetUniqueId")
    return buf.raw


def set_torch_transport(host_only=False, group=None):
    """Route the library's multi-rank exchanges through torch.distributed
    point-to-point (any backend that moves CPU tensors, e.g. gloo) instead of
    NCCL: plumbing for tests and CPU plan checks (hhg_set_host_transport)."""
    import torch
    import torch.distributed as dist

    def cb(user, nranks, sb, send, rb, recv):
        try:
            me = dist.get_rank(group)
            ts = sum(sb[p] for p in range(nranks))
            tr = sum(rb[p] for p in range(nranks))
            sbuf = torch.frombuffer((ctypes.c_char * max(ts, 1)).from_address(send), dtype=torch.uint8) if ts else None
            rbuf = torch.frombuffer((ctypes.c_char * max(tr, 1)).from_address(recv), dtype=torch.uint8) if tr else None
            reqs = []
            so = ro = 0
            for p in range(nranks):
                if p == me:
                    if sb[p]:
                        rbuf[ro:ro + rb[p]].copy_(sbuf[so:so + sb[p]])
                else:
                    if sb[p]:
                        reqs.append(dist.isend(sbuf[so:so + sb[p]].clone(), p, group=group))
                    if rb[p]:
                        reqs.append((dist.irecv(tmp := torch.empty(rb[p], dtype=torch.uint8), p, group=group),
                                     tmp, ro, rb[p]))
                so += sb[p]
                ro += rb[p]
            for r in reqs:
                if isinstance(r, tuple):
                    r[0].wait()
                    rbuf[r[2]:r[2] + r[3]].copy_(r[1])
                else:
                    r.wait()
            return 0
        except Exception as e:  # pragma: no cover
            import sys
            sys.stderr.write(f"hhg host transport failed: {e}\n")
            return 1

    fn = HostExchangeFn(cb)
    _keep_alive.append(fn)
    st = lib().hhg_set_host_transport(ctypes.cast(fn, ctypes.c_void_p), None, 1 if host_only else 0)
    if st != 0:
        raise HHGError(st, "hhg_set_host_transport")


class Ctx:
    """One hhg context (macro mesh + all levels 2..L_max) on the current device."""

    def __init__(self, vertices, radius, tets, dirichlet, L_max, stream=None, owner=None,
                 rank=0, nranks=1, nccl_id=None):
        L = lib()
        self._lib = L
        v = np.ascontiguousarray(vertices, dtype=np.float64)
        r = None if radius is None else np.ascontiguousarray(radius, dtype=np.float64)
        t = np.ascontiguousarray(tets, dtype=np.int64)
        d = np.ascontiguousarray(dirichlet, dtype=np.uint8)
        o = None if owner is None else np.ascontiguousarray(owner, dtype=np.int32)
        if stream is None:
            try:
                import torch
                stream = torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else 0
            except Exception:
                stream = 0
        h = ctypes.c_void_p()
        if nccl_id is not None:
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p)
        st = L.hhg_setup_macro_mesh(v.ctypes.data, None if r is None else r.ctypes.data, v.shape[0],
                                    t.ctypes.data, t.shape[0], d.ctypes.data, int(L_max),
                                    None if o is None else o.ctypes.data, rank, nranks, nccl_id,
                                    ctypes.c_void_p(stream), ctypes.byref(h))
        if st != 0:
            raise HHGError(st, "hhg_setup_macro_mesh failed (see stderr)")
        self.h = h
        self.L_max = int(L_max)
        self.nt = t.shape[0]

    @classmethod
    def from_mesh(cls, mesh, L_max, **kw):
        return cls(mesh.vertices, mesh.radius, mesh.tets, mesh.dirichlet, L_max, **kw)

    def _check(self, st):
        if st != 0:
            raise HHGError(st, self._lib.hhg_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self._lib.hhg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------
    def fit(self, q=2, method="lsqp", j=2):
        self._check(self._lib.hhg_fit_surrogates(self.h, q, FIT[method], j))

    def gs_prof(self, enable=True, read=False):
        """Cycle counters of the single-pass GS kernel (hhg_gs_prof)."""
        out = np.zeros(16, dtype=np.uint64)
        self._check(self._lib.hhg_gs_prof(self.h, 1 if enable else 0, out.ctypes.data if read else None))
        return out

    def sample_nodes(self, L, method="lsqp", j=2):
        """Sampling set of level L used by the fit (test export), [n, 3] int32."""
        n = ctypes.c_int64()
        self._check(self._lib.hhg_sample_nodes(self.h, L, FIT[method], j, None, ctypes.byref(n)))
        out = np.zeros((n.value, 3), dtype=np.int32)
        self._check(self._lib.hhg_sample_nodes(self.h, L, FIT[method], j, out.ctypes.data, ctypes.byref(n)))
        return out

    def fit_from_samples(self, L, samples, q=2, method="lsqp", j=2):
        """Fit level L from planted samples [nt_local, n, 15] (test export)."""
        s = np.ascontiguousarray(samples, dtype=np.float64)
        self._check(self._lib.hhg_fit_from_samples(self.h, L, q, FIT[method], j, s.ctypes.data))

    def layout(self, L):
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        self._check(self._lib.hhg_vector_layout(self.h, L, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    def zeros(self, L, device="cuda"):
        import torch
        return torch.zeros(self.layout(L)[0], dtype=torch.float64, device=device)

    def apply(self, L, u, y, op="surrogate"):
        n = self.layout(L)[0]
        self._check(self._lib.hhg_apply(self.h, L, OPS[op], _ptr(u, n), _ptr(y, n)))
        return y

    def residual(self, L, u, f, r, op="surrogate", norm=False):
        n = self.layout(L)[0]
        nv = ctypes.c_double()
        self._check(self._lib.hhg_residual(self.h, L, OPS[op], _ptr(u, n), _ptr(f, n), _ptr(r, n),
                                           ctypes.byref(nv) if norm else None))
        return nv.value if norm else None

    def gs_sweep(self, L, u, f, n_sweeps=1, op="surrogate", lexicographic=False):
        """Multicolour GS sweeps in place (hhg_gs_sweep), or the paper's
        lexicographic volume ordering (hhg_gs_sweep_lex)."""
        n = self.layout(L)[0]
        fn = self._lib.hhg_gs_sweep_lex if lexicographic else self._lib.hhg_gs_sweep
        self._check(fn(self.h, L, OPS[op], _ptr(u, n), _ptr(f, n), n_sweeps))
        return u

    def vcycle(self, L, u, f, n_cycles=1, nu1=3, nu2=3, L_coarse=2, cg_iters=50, op="surrogate", residual_op=None,
               lexicographic=False):
        """V(nu1,nu2) cycles in place on u; residual_op (e.g. "fem") selects
        double discretisation (hhg_vcycle_dd), lexicographic the paper's
        lexicographic smoother (hhg_vcycle_ex)."""
        n = self.layout(L)[0]
        hist = np.zeros(n_cycles + 1)
        if lexicographic:
            rop = OPS[residual_op if residual_op is not None else op]
            self._check(self._lib.hhg_vcycle_ex(self.h, L, nu1, nu2, L_coarse, cg_iters, OPS[op], rop, 1,
                                                _ptr(u, n), _ptr(f, n), n_cycles, hist.ctypes.data))
        elif residual_op is None:
            self._check(self._lib.hhg_vcycle(self.h, L, nu1, nu2, L_coarse, cg_iters, OPS[op], _ptr(u, n),
                                             _ptr(f, n), n_cycles, hist.ctypes.data))
        else:
            self._check(self._lib.hhg_vcycle_dd(self.h, L, nu1, nu2, L_coarse, cg_iters, OPS[op], OPS[residual_op],
                                                _ptr(u, n), _ptr(f, n), n_cycles, hist.ctypes.data))
        return hist

    def gather_global(self, L, local, out=None):
        n, _, ng = self.layout(L)
        if out is None:
            out = np.zeros(ng)
        self._check(self._lib.hhg_gather_global(self.h, L, _ptr(local, n), _ptr(out, ng)))
        return out

    def scatter_global(self, L, glob, local):
        n, _, ng = self.layout(L)
        self._check(self._lib.hhg_scatter_global(self.h, L, _ptr(glob, ng), _ptr(local, n)))
        return local

    def sync_copies(self, L, local):
        self._check(self._lib.hhg_sync_copies(self.h, L, _ptr(local, self.layout(L)[0])))
        return local

    def eval_stencils(self, L, macro=0, op="surrogate"):
        N = 2 ** L
        n_int = (N - 1) * (N - 2) * (N - 3) // 6
        out = np.zeros((n_int, 15))
        self._check(self._lib.hhg_eval_stencils(self.h, L, OPS[op], macro, out.ctypes.data))
        return out

    def plan_info(self, L):
        info = (ctypes.c_int64 * 5)()
        self._check(self._lib.hhg_plan_info(self.h, L, info))
        return dict(zip(("owned", "send", "recv", "local_macros", "blocks"), list(info)))

    def plan_check(self, L):
        m = ctypes.c_int64()
        self._check(self._lib.hhg_plan_check(self.h, L, ctypes.byref(m)))
        return m.value

    @property
    def kernel_launches(self):
        return int(self._lib.hhg_kernel_launches(self.h))

    def profile(self, enable=True):
        self._check(self._lib.hhg_profile(self.h, 1 if enable else 0))

    def profile_read(self):
        """{class: (total device ms, launches)} since the last read; clears."""
        out = {}
        for k, name in enumerate(("vol_apply", "vol_gs", "lp_rows", "other")):
            ms, n = ctypes.c_double(), ctypes.c_int64()
            self._check(self._lib.hhg_profile_read(self.h, k, ctypes.byref(ms), ctypes.byref(n)))
            out[name] = (ms.value, n.value)
        return out
