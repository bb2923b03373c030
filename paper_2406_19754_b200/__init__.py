"""B200-native AMG-PCG solve phase of PSCToolkit (arXiv 2406.19754).

Thin ctypes binding over ``libpsc.so`` (C ABI declared in ``include/psc.h``).
Argument marshalling only: every numerical step runs in the library's sm_100a
CUDA kernels and NCCL.  There is no CPU fallback: if the shared library is
missing this module raises ImportError, and on a machine without a B200 every
compute call fails with PscError(PSC_ERR_CUDA).

Device vectors are passed as torch CUDA float64 tensors (torch is used only for
device memory, streams and process groups); host vectors as numpy float64.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PSC_LIB: alternative build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("PSC_LIB") or os.path.join(_HERE, "libpsc.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2406_19754_b200.build` "
                      "(or __graft_entry__.build()); there is no fallback path")

_lib = ctypes.CDLL(LIB_PATH)

PSC_OK, PSC_NOT_CONVERGED = 0, 1
PSC_ERR_ARG, PSC_ERR_STATE, PSC_ERR_CUDA, PSC_ERR_NCCL, PSC_ERR_NOMEM, PSC_ERR_BREAKDOWN = -1, -2, -3, -4, -5, -6

_vp, _i64, _i32, _f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double


PSC_COARSE_SWEEPS, PSC_COARSE_PCG = 0, 1
PSC_KRYLOV_PCG, PSC_KRYLOV_FCG = 0, 1
_COARSE = {"sweeps": PSC_COARSE_SWEEPS, "pcg": PSC_COARSE_PCG}
_KRYLOV = {"pcg": PSC_KRYLOV_PCG, "fcg": PSC_KRYLOV_FCG}


class CycleOpts(ctypes.Structure):
    _fields_ = [("pre_sweeps", _i32), ("post_sweeps", _i32), ("coarse_sweeps", _i32), ("coarse_solver", _i32),
                ("coarse_maxit", _i32), ("coarse_tol", _f64), ("variable_v", _i32), ("smoother", _i32),
                ("ainv_drop", _f64)]


class KernelRec(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 64), ("level", _i32), ("calls_per_iter", _i32), ("total_us", _f64),
                ("alg_bytes", _f64), ("layout_bytes", _f64)]


class Stats(ctypes.Structure):
    _fields_ = [("iters", _i32), ("status", _i32), ("rel_res", _f64), ("solve_seconds", _f64),
                ("kernel_launches", _i64), ("collectives", _i64), ("dom_kernel_seconds", _f64),
                ("dom_kernel_launches", _i64), ("dom_kernel_bytes", _f64), ("h2d_bytes", _i64),
                ("d2h_bytes", _i64), ("halo_path", _i32), ("iter_graph_nodes", _i32),
                ("dom_kernel_per_iter", _i32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_P = ctypes.POINTER
_sig("psc_get_unique_id", _i32, [ctypes.c_char_p])
_sig("psc_init", _i32, [_i32, _i32, _i32, ctypes.c_char_p, _vp, _P(_vp)])
_sig("psc_finalize", None, [_vp])
_sig("psc_status_string", ctypes.c_char_p, [_i32])
_sig("psc_last_error", ctypes.c_char_p, [_vp])
_sig("psc_version", ctypes.c_char_p, [])
_sig("psc_ctx_stream", _vp, [_vp])
_sig("psc_halo_plan", _i32, [_i32, _i32, _vp, _i64, _vp, _vp, _P(_i64), _vp])
_sig("psc_send_plan", _i32, [_i32, _i32, _vp, _vp, _vp, _vp])
_sig("psc_desc_create", _i32, [_vp, _i64, _vp, _P(_vp)])
_sig("psc_desc_assemble", _i32, [_vp])
_sig("psc_desc_info", _i32, [_vp, _P(_i64), _P(_i64), _P(_i64)])
_sig("psc_desc_halo", _i32, [_vp, _vp])
_sig("psc_desc_destroy", None, [_vp])
_sig("psc_mat_create_csr", _i32, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _P(_vp)])
_sig("psc_mat_assemble", _i32, [_vp])
_sig("psc_mat_info", _i32, [_vp, _P(_i64), _P(_i64), _P(_i64), _P(_i64), _P(_i32)])
_sig("psc_mat_spmv", _i32, [_vp, _f64, _vp, _f64, _vp])
_sig("psc_mat_destroy", None, [_vp])
_sig("psc_hier_create", _i32, [_vp, _i32, _vp, _vp, _vp, _P(CycleOpts), _P(_vp)])
_sig("psc_hier_info", _i32, [_vp, _P(_i32), _vp, _vp, _vp, _vp])
_sig("psc_hier_vcycle", _i32, [_vp, _vp, _vp])
_sig("psc_hier_dinv", _i32, [_vp, _i32, _vp])
_sig("psc_hier_smooth", _i32, [_vp, _i32, _vp, _vp, _i32])
_sig("psc_pcg_solve", _i32, [_vp, _vp, _vp, _f64, _i32, _vp, _P(Stats)])
_sig("psc_pcg_solve_host", _i32, [_vp, _vp, _vp, _f64, _i32, _vp, _P(Stats)])
_sig("psc_krylov_solve", _i32, [_vp, _i32, _vp, _vp, _f64, _i32, _vp, _P(Stats)])
_sig("psc_krylov_solve_host", _i32, [_vp, _i32, _vp, _vp, _f64, _i32, _vp, _P(Stats)])
_sig("psc_hier_exchange_bench", _i32, [_vp, _i32, _i32, _P(_f64)])
_sig("psc_hier_kernel_profile", _i32, [_vp, _i32, _vp, _i32, _vp, _i32, _P(_i32)])
_sig("psc_hier_destroy", None, [_vp])
_sig("psc_mat_update_values", _i32, [_vp, _vp])
_sig("psc_hier_rebuild_smoothers", _i32, [_vp])


class AmgOpts(ctypes.Structure):
    _fields_ = [("theta", _f64), ("max_levels", _i32), ("coarse_target", _i64), ("stall_ratio", _f64)]


_sig("psc_amg_build", _i32, [_vp, _i64, _vp, _vp, _vp, _P(AmgOpts), _P(_vp)])
_sig("psc_amg_info", _i32, [_vp, _P(_i32), _vp, _vp, _vp, _vp, _vp, _vp])
_sig("psc_amg_level_csr", _i32, [_vp, _i32, _i32, _vp, _vp, _vp])
_sig("psc_amg_aggregates", _i32, [_vp, _i32, _vp, _vp])
_sig("psc_amg_hier_create", _i32, [_vp, _P(CycleOpts), _P(_vp)])
_sig("psc_amg_destroy", None, [_vp])


class PscError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_lib.psc_status_string(code).decode()}: {msg}")
        self.code = code


def version() -> str:
    return _lib.psc_version().decode()


def _check(rc, ctx=None, ok=(PSC_OK,)):
    if rc in ok:
        return rc
    msg = _lib.psc_last_error(ctx.handle if ctx is not None else None).decode()
    raise PscError(rc, msg)


def _dev_ptr(t, n, name):
    """torch CUDA float64 contiguous tensor of n elements -> raw pointer."""
    if t is None:
        if n == 0:
            return None
        raise ValueError(f"{name} is None")
    if not (getattr(t, "is_cuda", False) and str(t.dtype) == "torch.float64" and t.is_contiguous()):
        raise TypeError(f"{name} must be a contiguous CUDA float64 tensor")
    if t.numel() != n:
        raise ValueError(f"{name} has {t.numel()} elements, expected {n}")
    return t.data_ptr()


def _host(a, dtype, name):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a


def halo_plan(nranks: int, rank: int, row_start, refs):
    """Host-only halo plan (psc_halo_plan): sorted unique off-rank columns and per-owner counts."""
    rs = _host(row_start, np.int64, "row_start")
    refs = _host(refs, np.int64, "refs")
    halo = np.zeros(max(len(refs), 1), np.int64)
    nh = _i64()
    rc = np.zeros(nranks, np.int64)
    _check(_lib.psc_halo_plan(nranks, rank, rs.ctypes.data, len(refs), refs.ctypes.data, halo.ctypes.data,
                              ctypes.byref(nh), rc.ctypes.data))
    return halo[: nh.value].copy(), rc


def send_plan(nranks: int, rank: int, row_start, send_count, requests):
    """Host-only send plan (psc_send_plan): local owned indices for the peers' requests."""
    rs = _host(row_start, np.int64, "row_start")
    sc = _host(send_count, np.int64, "send_count")
    rq = _host(requests, np.int64, "requests")
    out = np.zeros(max(int(sc.sum()), 1), np.int32)
    _check(_lib.psc_send_plan(nranks, rank, rs.ctypes.data, sc.ctypes.data, rq.ctypes.data, out.ctypes.data))
    return out[: int(sc.sum())].copy()


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.psc_get_unique_id(buf))
    return buf.raw


class Context:
    """psc_init: rank/nranks/device; unique_id (128 bytes from rank 0) when nranks > 1."""

    def __init__(self, rank=0, nranks=1, device=0, unique_id: bytes | None = None, stream=None):
        if stream is None:
            try:
                import torch
                if torch.cuda.is_available():
                    stream = torch.cuda.current_stream(device).cuda_stream
            except Exception:
                stream = None
        h = _vp()
        _check(_lib.psc_init(rank, nranks, device, unique_id, stream, ctypes.byref(h)))
        self.handle = h.value
        self.rank, self.nranks, self.device = rank, nranks, device
        self._children = []

    @property
    def stream(self) -> int:
        """cudaStream_t (as int) of the library stream; wrap with torch.cuda.ExternalStream."""
        return _lib.psc_ctx_stream(self.handle)

    def close(self):
        if self.handle:
            for c in reversed(self._children):
                c.close()
            self._children = []
            _lib.psc_finalize(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Descriptor:
    def __init__(self, ctx: Context, n_global: int, row_start):
        rs = _host(row_start, np.int64, "row_start")
        if len(rs) != ctx.nranks + 1:
            raise ValueError("row_start must have nranks+1 entries")
        h = _vp()
        _check(_lib.psc_desc_create(ctx.handle, int(n_global), rs.ctypes.data, ctypes.byref(h)), ctx)
        self.ctx, self.handle = ctx, h.value
        self.n_global = int(n_global)
        self.row_start = rs
        ctx._children.append(self)

    def assemble(self):
        _check(_lib.psc_desc_assemble(self.handle), self.ctx)
        return self

    def info(self):
        a, b, c = _i64(), _i64(), _i64()
        _check(_lib.psc_desc_info(self.handle, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), self.ctx)
        return dict(n_owned=a.value, n_halo=b.value, own_begin=c.value)

    def halo(self) -> np.ndarray:
        out = np.zeros(self.info()["n_halo"], dtype=np.int64)
        _check(_lib.psc_desc_halo(self.handle, out.ctypes.data), self.ctx)
        return out

    @property
    def n_owned(self):
        return int(self.row_start[self.ctx.rank + 1] - self.row_start[self.ctx.rank])

    def close(self):
        if self.handle:
            _lib.psc_desc_destroy(self.handle)
            self.handle = None


class Matrix:
    """This rank's rows in CSR with GLOBAL int64 columns (psc_mat_create_csr)."""

    def __init__(self, ctx: Context, rows: Descriptor, cols: Descriptor, row_ptr, col_global, val):
        rp = _host(row_ptr, np.int64, "row_ptr")
        cg = _host(col_global, np.int64, "col_global")
        v = _host(val, np.float64, "val")
        h = _vp()
        _check(_lib.psc_mat_create_csr(ctx.handle, rows.handle, cols.handle, len(rp) - 1, rp.ctypes.data,
                                       cg.ctypes.data, v.ctypes.data, ctypes.byref(h)), ctx)
        self.ctx, self.rows, self.cols, self.handle = ctx, rows, cols, h.value
        ctx._children.append(self)

    def assemble(self):
        _check(_lib.psc_mat_assemble(self.handle), self.ctx)
        return self

    def info(self):
        a, b, c, d, e = _i64(), _i64(), _i64(), _i64(), _i32()
        _check(_lib.psc_mat_info(self.handle, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(d),
                                 ctypes.byref(e)), self.ctx)
        return dict(nnz=a.value, padded=b.value, n_units=c.value, n_rows=d.value, lanes=e.value)

    def update_values(self, val):
        """psc_mat_update_values: new values, same CSR structure as at creation."""
        v = _host(val, np.float64, "val")
        _check(_lib.psc_mat_update_values(self.handle, v.ctypes.data), self.ctx)

    def spmv(self, x, y, alpha=1.0, beta=0.0):
        """y = alpha A x + beta y (device tensors; owned parts)."""
        _check(_lib.psc_mat_spmv(self.handle, float(alpha), _dev_ptr(x, self.cols.n_owned, "x"), float(beta),
                                 _dev_ptr(y, self.rows.n_owned, "y")), self.ctx)
        return y

    def close(self):
        if self.handle:
            _lib.psc_mat_destroy(self.handle)
            self.handle = None


_SMOOTHER = {"l1": 0, "ainv": 1}


def _cycle_opts(pre, post, coarse, coarse_solver, coarse_maxit, coarse_tol, variable_v, smoother, ainv_drop):
    if coarse_solver not in _COARSE:
        raise ValueError(f"coarse_solver must be one of {sorted(_COARSE)}")
    if smoother not in _SMOOTHER:
        raise ValueError(f"smoother must be one of {sorted(_SMOOTHER)}")
    return CycleOpts(pre, post, coarse, _COARSE[coarse_solver], int(coarse_maxit), float(coarse_tol),
                     1 if variable_v else 0, _SMOOTHER[smoother], float(ainv_drop))


class Hierarchy:
    """psc_hier_create over given level matrices A[l], P[l], R[l]; V-cycle + PCG / FCG.

    coarse_solver: "sweeps" (`coarse` l1-Jacobi sweeps) or "pcg" (PCG with
    l1-Jacobi, at most coarse_maxit iterations to coarse_tol).
    variable_v: variable V-cycle, pre/post sweeps doubled per level (P:330 footnote).
    smoother: "l1" (l1-Jacobi) or "ainv" (AINV with drop tolerance ainv_drop,
    P:273-279)."""

    def __init__(self, ctx: Context, A, P, R, pre=4, post=4, coarse=30, coarse_solver="sweeps", coarse_maxit=40,
                 coarse_tol=1e-10, variable_v=False, smoother="l1", ainv_drop=0.1):
        L = len(A)
        Aa = (_vp * L)(*[m.handle for m in A])
        Pa = (_vp * max(L - 1, 1))(*[m.handle for m in P])
        Ra = (_vp * max(L - 1, 1))(*[m.handle for m in R])
        if coarse_solver not in _COARSE:
            raise ValueError(f"coarse_solver must be one of {sorted(_COARSE)}")
        opts = _cycle_opts(pre, post, coarse, coarse_solver, coarse_maxit, coarse_tol, variable_v, smoother, ainv_drop)
        h = _vp()
        _check(_lib.psc_hier_create(ctx.handle, L, Aa, Pa, Ra, ctypes.byref(opts), ctypes.byref(h)), ctx)
        self.ctx, self.handle, self.nlevels = ctx, h.value, L
        self.A, self.P, self.R = list(A), list(P), list(R)
        self.n0 = A[0].rows.n_owned
        ctx._children.append(self)

    def rebuild_smoothers(self):
        """psc_hier_rebuild_smoothers: smoothers from the current A_l values."""
        _check(_lib.psc_hier_rebuild_smoothers(self.handle), self.ctx)

    def info(self):
        L = self.nlevels
        nl = _i32()
        arrs = [np.zeros(L, np.int64) for _ in range(4)]
        _check(_lib.psc_hier_info(self.handle, ctypes.byref(nl), *[a.ctypes.data for a in arrs]), self.ctx)
        return dict(nlevels=nl.value, n_owned=arrs[0].tolist(), nnz_A=arrs[1].tolist(), nnz_P=arrs[2].tolist(),
                    nnz_R=arrs[3].tolist())

    def vcycle(self, r, z):
        _check(_lib.psc_hier_vcycle(self.handle, _dev_ptr(r, self.n0, "r"), _dev_ptr(z, self.n0, "z")), self.ctx)
        return z

    def _n(self, level):
        ln = getattr(self, "_level_n", None)
        return ln[level] if ln else self.A[level].rows.n_owned

    def dinv(self, level, out):
        n = self._n(level)
        _check(_lib.psc_hier_dinv(self.handle, level, _dev_ptr(out, n, "out")), self.ctx)
        return out

    def smooth(self, level, b, x, nsweeps):
        n = self._n(level)
        _check(_lib.psc_hier_smooth(self.handle, level, _dev_ptr(b, n, "b"), _dev_ptr(x, n, "x"), int(nsweeps)),
               self.ctx)
        return x

    def solve(self, b, x, tol=1e-8, maxit=200, method="pcg"):
        """PCG or FCG (method) on device tensors.  Returns (status, stats dict, residual history)."""
        if method not in _KRYLOV:
            raise ValueError(f"method must be one of {sorted(_KRYLOV)}")
        hist = np.full(maxit + 1, np.nan)
        st = Stats()
        rc = _lib.psc_krylov_solve(self.handle, _KRYLOV[method], _dev_ptr(b, self.n0, "b"), _dev_ptr(x, self.n0, "x"),
                                   float(tol), int(maxit), hist.ctypes.data, ctypes.byref(st))
        _check(rc, self.ctx, ok=(PSC_OK, PSC_NOT_CONVERGED))
        return rc, st.as_dict(), hist[: st.iters + 1]

    def solve_host(self, b, x, tol=1e-8, maxit=200, method="pcg"):
        """PCG / FCG on host numpy arrays (end-to-end path: copies inside the call). x updated in place."""
        if method not in _KRYLOV:
            raise ValueError(f"method must be one of {sorted(_KRYLOV)}")
        if not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.c_contiguous):
            raise TypeError("x must be a C-contiguous float64 numpy array")
        b = _host(b, np.float64, "b")
        if len(b) != self.n0 or len(x) != self.n0:
            raise ValueError("b/x size mismatch")
        hist = np.full(maxit + 1, np.nan)
        st = Stats()
        rc = _lib.psc_krylov_solve_host(self.handle, _KRYLOV[method], b.ctypes.data, x.ctypes.data, float(tol),
                                        int(maxit), hist.ctypes.data, ctypes.byref(st))
        _check(rc, self.ctx, ok=(PSC_OK, PSC_NOT_CONVERGED))
        return rc, st.as_dict(), hist[: st.iters + 1]

    def kernel_profile(self, b, iters=5, method="pcg", max_recs=256):
        """psc_hier_kernel_profile: per-(kernel, level) device time per iteration and bytes per call."""
        if method not in _KRYLOV:
            raise ValueError(f"method must be one of {sorted(_KRYLOV)}")
        recs = (KernelRec * max_recs)()
        n = _i32()
        _check(_lib.psc_hier_kernel_profile(self.handle, _KRYLOV[method], _dev_ptr(b, self.n0, "b"), int(iters),
                                            recs, max_recs, ctypes.byref(n)), self.ctx)
        return [dict(name=r.name.decode(), level=r.level, calls_per_iter=r.calls_per_iter, total_us=r.total_us,
                     alg_bytes=r.alg_bytes, layout_bytes=r.layout_bytes) for r in recs[: min(n.value, max_recs)]]

    def exchange_bench(self, level, reps=200):
        """Device microseconds per halo exchange of a level vector (collective)."""
        us = _f64()
        _check(_lib.psc_hier_exchange_bench(self.handle, level, reps, ctypes.byref(us)), self.ctx)
        return us.value

    def close(self):
        if self.handle:
            _lib.psc_hier_destroy(self.handle)
            self.handle = None


class AmgSetup:
    """psc_amg_build: the VMB set-up (aggregation, smoothed P, R = P^T, Galerkin RAP) on
    the device from a host CSR A_0 (one rank).  hierarchy() -> Hierarchy over its levels."""

    _MAXL = 64

    def __init__(self, ctx: Context, A0, theta=0.01, max_levels=20, coarse_target=200, stall_ratio=0.75):
        if hasattr(A0, "indptr"):
            A0 = A0.tocsr()
            A0.sort_indices()
            ptr, col, val = A0.indptr, A0.indices, A0.data
        else:
            ptr, col, val = A0.ptr, A0.col, A0.val
        ptr, col, val = _host(ptr, np.int64, "ptr"), _host(col, np.int64, "col"), _host(val, np.float64, "val")
        o = AmgOpts(float(theta), int(max_levels), int(coarse_target), float(stall_ratio))
        h = _vp()
        _check(_lib.psc_amg_build(ctx.handle, len(ptr) - 1, ptr.ctypes.data, col.ctypes.data, val.ctypes.data,
                                  ctypes.byref(o), ctypes.byref(h)), ctx)
        self.ctx, self.handle = ctx, h.value
        self._hier = None
        ctx._children.append(self)

    def info(self):
        M = self._MAXL
        nl = _i32()
        n, nA, nP = (np.zeros(M, np.int64) for _ in range(3))
        om = np.zeros(M)
        rounds = np.zeros(M, np.int32)
        secs = np.zeros(5)
        _check(_lib.psc_amg_info(self.handle, ctypes.byref(nl), n.ctypes.data, nA.ctypes.data, nP.ctypes.data,
                                 om.ctypes.data, rounds.ctypes.data, secs.ctypes.data), self.ctx)
        L = nl.value
        return dict(nlevels=L, n=n[:L].tolist(), nnz_A=nA[:L].tolist(), nnz_P=nP[:L].tolist(),
                    omega=om[:L].tolist(), mis_rounds=rounds[:L].tolist(),
                    seconds=dict(zip(("aggregate", "prolongator", "transpose", "galerkin", "total"), secs.tolist())))

    def csr(self, level, kind):
        """(ptr, col, val) of A_l (kind "A"), P_l ("P") or R_l ("R") copied to the host."""
        k = {"A": 0, "P": 1, "R": 2}[kind]
        inf = self.info()
        n = inf["n"][level]
        rows = {0: n, 1: n, 2: inf["n"][level + 1] if level + 1 < inf["nlevels"] else 0}[k]
        ptr = np.zeros(rows + 1, np.int64)
        _check(_lib.psc_amg_level_csr(self.handle, level, k, ptr.ctypes.data, None, None), self.ctx)
        col = np.zeros(int(ptr[-1]), np.int64)
        val = np.zeros(int(ptr[-1]))
        _check(_lib.psc_amg_level_csr(self.handle, level, k, None, col.ctypes.data, val.ctypes.data), self.ctx)
        return ptr, col, val

    def aggregates(self, level):
        n = self.info()["n"][level]
        agg = np.zeros(n, np.int64)
        root = np.zeros(n, np.int8)
        _check(_lib.psc_amg_aggregates(self.handle, level, agg.ctypes.data, root.ctypes.data), self.ctx)
        return agg, root.astype(bool)

    def hierarchy(self, pre=4, post=4, coarse=30, coarse_solver="sweeps", coarse_maxit=40, coarse_tol=1e-10,
                  variable_v=False, smoother="l1", ainv_drop=0.1) -> "Hierarchy":
        opts = _cycle_opts(pre, post, coarse, coarse_solver, coarse_maxit, coarse_tol, variable_v, smoother, ainv_drop)
        h = _vp()
        _check(_lib.psc_amg_hier_create(self.handle, ctypes.byref(opts), ctypes.byref(h)), self.ctx)
        H = Hierarchy.__new__(Hierarchy)
        H.ctx, H.handle, H.nlevels = self.ctx, h.value, self.info()["nlevels"]
        H.A, H.P, H.R = [], [], []
        H._level_n = self.info()["n"]
        H.n0 = H._level_n[0]
        self._hier = H
        return H

    def close(self):
        if self.handle:
            if self._hier is not None:
                self._hier.close()
                self._hier = None
            _lib.psc_amg_destroy(self.handle)
            self.handle = None


def build_hierarchy(ctx: Context, levels, pre=4, post=4, coarse=30, **coarse_kw):
    """Create descriptors + matrices for this rank and assemble them, in the
    PSBLAS order.  `levels[l]` is a dict with
      n_global, row_start (nranks+1), A=(row_ptr, col_global, val) for this rank's rows,
      and for l < L-1: P=(...) (rows of space l), R=(...) (rows of space l+1).
    Returns (Hierarchy, descs, A, P, R)."""
    L = len(levels)
    descs = [Descriptor(ctx, lv["n_global"], lv["row_start"]) for lv in levels]
    A = [Matrix(ctx, descs[l], descs[l], *levels[l]["A"]) for l in range(L)]
    P = [Matrix(ctx, descs[l], descs[l + 1], *levels[l]["P"]) for l in range(L - 1)]
    R = [Matrix(ctx, descs[l + 1], descs[l], *levels[l]["R"]) for l in range(L - 1)]
    for d in descs:
        d.assemble()
    for m in A + P + R:
        m.assemble()
    h = Hierarchy(ctx, A, P, R, pre, post, coarse, **coarse_kw)
    return h, descs, A, P, R
