"""CPU oracle for the AMG-PCG solve phase — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product library
(``paper_2406_19754_b200``) never does, and shares no code with it.

Thin ctypes marshalling over ``oracle/psc_oracle.c`` (plain C, fp64,
single-threaded, no fast-math, no FMA contraction).  Each C function cites the
PAPER.md passage it implements.  Pins (tests that tie the oracle to the paper
and to mathematics rather than to itself) live in ``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

STATUS = {0: "converged", 1: "not converged", -6: "breakdown"}


_SO_OMP = os.path.join(_HERE, "liboracle_omp.so")
_threads = 1


def build(force: bool = False) -> str:
    """Serial build (liboracle.so, what the tests use) and the OpenMP build of the same
    source (liboracle_omp.so, bitwise identical results; cpu_baseline on all cores)."""
    src = os.path.join(_HERE, "psc_oracle.c")
    for so, extra in ((_SO, []), (_SO_OMP, ["-fopenmp"])):
        if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            tmp = so + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off", "-fPIC",
                                   "-shared", *extra, "-o", tmp, src, "-lm"])
            os.replace(tmp, so)
    return _SO


def set_threads(n: int) -> int:
    """Use the OpenMP build with n threads (n <= 1: the serial build).  Returns the thread count.
    Must be called before the first oracle call of the process."""
    global _threads, _lib
    if _lib is not None and (n > 1) != (_threads > 1):
        raise RuntimeError("oracle.set_threads must be called before the first oracle call")
    _threads = max(1, int(n))
    if _threads > 1:
        return lib().or_set_threads(_threads)
    return 1


class _CSR(ctypes.Structure):
    _fields_ = [("nrows", ctypes.c_int64), ("ncols", ctypes.c_int64), ("ptr", ctypes.c_void_p),
                ("col", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class _Hier(ctypes.Structure):
    _fields_ = [("nlevels", ctypes.c_int), ("A", ctypes.POINTER(_CSR)), ("P", ctypes.POINTER(_CSR)),
                ("R", ctypes.POINTER(_CSR)), ("pre", ctypes.c_int), ("post", ctypes.c_int),
                ("coarse", ctypes.c_int), ("coarse_pcg", ctypes.c_int), ("coarse_maxit", ctypes.c_int),
                ("coarse_tol", ctypes.c_double), ("variable_v", ctypes.c_int), ("smoother", ctypes.c_int),
                ("ainv_drop", ctypes.c_double), ("ainv_nb", ctypes.c_void_p), ("ainv_rs", ctypes.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO_OMP if _threads > 1 else _SO)
        L.or_set_threads.argtypes = [ctypes.c_int]
        L.or_set_threads.restype = ctypes.c_int
        vp = ctypes.c_void_p
        L.or_spmv.argtypes = [vp, vp, vp]
        L.or_l1_diag.argtypes = [vp, vp]
        L.or_l1_sweep.argtypes = [vp, vp, vp, vp, vp]
        L.or_l1_sweeps_from_zero.argtypes = [vp, vp, vp, ctypes.c_int, vp, vp]
        L.or_vcycle.argtypes = [vp, vp, vp]
        L.or_pcg.argtypes = [vp, vp, vp, ctypes.c_double, ctypes.c_int, vp, ctypes.POINTER(ctypes.c_int)]
        L.or_pcg.restype = ctypes.c_int
        L.or_fcg.argtypes = [vp, vp, vp, ctypes.c_double, ctypes.c_int, vp, ctypes.POINTER(ctypes.c_int)]
        L.or_fcg.restype = ctypes.c_int
        L.or_coarse_pcg.argtypes = [vp, vp, vp, vp, ctypes.c_int, ctypes.c_double]
        L.or_coarse_pcg.restype = ctypes.c_int
        _lib = L
    return _lib


def _arr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class _CsrHolder:
    """Keeps the numpy buffers alive for the lifetime of the C struct."""

    def __init__(self, m):
        if hasattr(m, "indptr"):  # scipy.sparse
            m = m.tocsr()
            m.sort_indices()
            shape, ptr, col, val = m.shape, m.indptr, m.indices, m.data
        else:  # pscgen.CSR duck type
            shape, ptr, col, val = m.shape, m.ptr, m.col, m.val
        self.ptr = _arr(ptr, np.int64)
        self.col = _arr(col, np.int64)
        self.val = _arr(val, np.float64)
        self.c = _CSR(shape[0], shape[1], self.ptr.ctypes.data, self.col.ctypes.data, self.val.ctypes.data)


class _HierHolder:
    def __init__(self, hier, pre=4, post=4, coarse=30, coarse_pcg=False, coarse_maxit=40, coarse_tol=1e-10,
                 variable_v=False, smoother="l1", ainv_drop=0.1, ainv_blocks=None):
        L = hier.nlevels
        self.A = [_CsrHolder(hier.levels[l].A) for l in range(L)]
        self.P = [_CsrHolder(hier.levels[l].P) for l in range(L - 1)]
        self.R = [_CsrHolder(hier.levels[l].R) for l in range(L - 1)]
        self.Aa = (_CSR * L)(*[h.c for h in self.A])
        self.Pa = (_CSR * max(L - 1, 1))(*[h.c for h in self.P])
        self.Ra = (_CSR * max(L - 1, 1))(*[h.c for h in self.R])
        if smoother not in ("l1", "ainv"):
            raise ValueError("smoother must be 'l1' or 'ainv'")
        # AINV block structure per level (None: the whole level matrix)
        nb = np.zeros(L, np.int32)
        self._rs = [None] * L
        rsp = (ctypes.c_void_p * L)()
        for l in range(L):
            blk = ainv_blocks[l] if ainv_blocks is not None and l < len(ainv_blocks) else None
            if blk is not None:
                self._rs[l] = _arr(blk, np.int64)
                nb[l] = len(self._rs[l]) - 1
                rsp[l] = self._rs[l].ctypes.data
        self._nb, self._rsp = nb, rsp
        self.c = _Hier(L, self.Aa, self.Pa, self.Ra, pre, post, coarse, 1 if coarse_pcg else 0, coarse_maxit,
                       coarse_tol, 1 if variable_v else 0, 1 if smoother == "ainv" else 0, float(ainv_drop),
                       nb.ctypes.data, ctypes.cast(rsp, ctypes.c_void_p).value)


def spmv(A, x) -> np.ndarray:
    h = _CsrHolder(A)
    x = _arr(x, np.float64)
    y = np.empty(h.c.nrows, np.float64)
    lib().or_spmv(ctypes.byref(h.c), x.ctypes.data, y.ctypes.data)
    return y


def l1_diag(A) -> np.ndarray:
    h = _CsrHolder(A)
    m = np.empty(h.c.nrows, np.float64)
    lib().or_l1_diag(ctypes.byref(h.c), m.ctypes.data)
    return m


def l1_sweep(A, b, x) -> np.ndarray:
    """One sweep x + M^{-1}(b - A x) (Eq. (2) right factor)."""
    h = _CsrHolder(A)
    m = l1_diag(A)
    b, x = _arr(b, np.float64), _arr(x, np.float64)
    out = np.empty_like(x)
    lib().or_l1_sweep(ctypes.byref(h.c), m.ctypes.data, b.ctypes.data, x.ctypes.data, out.ctypes.data)
    return out


def l1_sweeps_from_zero(A, b, nsweeps: int) -> np.ndarray:
    h = _CsrHolder(A)
    m = l1_diag(A)
    b = _arr(b, np.float64)
    x = np.empty(h.c.nrows, np.float64)
    w = np.empty(h.c.nrows, np.float64)
    lib().or_l1_sweeps_from_zero(ctypes.byref(h.c), m.ctypes.data, b.ctypes.data, int(nsweeps), x.ctypes.data,
                                 w.ctypes.data)
    return x


def vcycle(hier, r, pre=4, post=4, coarse=30, **coarse_kw) -> np.ndarray:
    """z = B_0 r, Eq. (2).  coarse_kw: coarse_pcg, coarse_maxit, coarse_tol,
    variable_v (pre/post sweeps doubled per level, P:330 footnote)."""
    hh = _HierHolder(hier, pre, post, coarse, **coarse_kw)
    r = _arr(r, np.float64)
    z = np.empty_like(r)
    lib().or_vcycle(ctypes.byref(hh.c), r.ctypes.data, z.ctypes.data)
    return z


def coarse_pcg(A, b, maxit=40, tol=1e-10):
    """Coarsest-level PCG with the l1-Jacobi preconditioner.  Returns (x, iterations)."""
    h = _CsrHolder(A)
    m = l1_diag(A)
    b = _arr(b, np.float64)
    x = np.empty(h.c.nrows, np.float64)
    it = lib().or_coarse_pcg(ctypes.byref(h.c), m.ctypes.data, b.ctypes.data, x.ctypes.data, int(maxit), float(tol))
    return x, it


def fcg(hier, b, x0=None, tol=1e-8, maxit=200, pre=4, post=4, coarse=30, **coarse_kw):
    """Flexible CG, FCG(1), one V-cycle per iteration.  Returns (x, iters, status, hist)."""
    hh = _HierHolder(hier, pre, post, coarse, **coarse_kw)
    b = _arr(b, np.float64)
    x = np.zeros_like(b) if x0 is None else _arr(x0, np.float64).copy()
    hist = np.full(maxit + 1, np.nan)
    it = ctypes.c_int(0)
    st = lib().or_fcg(ctypes.byref(hh.c), b.ctypes.data, x.ctypes.data, float(tol), int(maxit), hist.ctypes.data,
                      ctypes.byref(it))
    return x, it.value, st, hist[: it.value + 1]


def pcg(hier, b, x0=None, tol=1e-8, maxit=200, pre=4, post=4, coarse=30, **coarse_kw):
    """PCG preconditioned by one V-cycle per iteration.  Returns (x, iters, status, hist)."""
    hh = _HierHolder(hier, pre, post, coarse, **coarse_kw)
    b = _arr(b, np.float64)
    x = np.zeros_like(b) if x0 is None else _arr(x0, np.float64).copy()
    hist = np.full(maxit + 1, np.nan)
    it = ctypes.c_int(0)
    st = lib().or_pcg(ctypes.byref(hh.c), b.ctypes.data, x.ctypes.data, float(tol), int(maxit), hist.ctypes.data,
                      ctypes.byref(it))
    return x, it.value, st, hist[: it.value + 1]


# ------------------------------------------------------------------ NEXT-1 set-up
def _take_csr(nrows, ncols, pp, pc, pv):
    """Copy a malloc'd CSR (int64 ptr/col, f64 val) into scipy and free it."""
    import scipy.sparse as sp
    L = lib()
    ptr = np.ctypeslib.as_array(ctypes.cast(pp, ctypes.POINTER(ctypes.c_int64)), shape=(nrows + 1,)).copy()
    nnz = int(ptr[-1])
    col = (np.ctypeslib.as_array(ctypes.cast(pc, ctypes.POINTER(ctypes.c_int64)), shape=(nnz,)).copy()
           if nnz else np.zeros(0, np.int64))
    val = (np.ctypeslib.as_array(ctypes.cast(pv, ctypes.POINTER(ctypes.c_double)), shape=(nnz,)).copy()
           if nnz else np.zeros(0))
    for p in (pp, pc, pv):
        L.or_free(p)
    m = sp.csr_matrix((val, col, ptr), shape=(nrows, ncols))
    m.has_sorted_indices = True  # rows are built with increasing columns
    return m


def _setup_sigs():
    L = lib()
    vp = ctypes.c_void_p
    if getattr(L, "_setup_sigs", False):
        return L
    L.or_free.argtypes = [vp]
    L.or_vmb_aggregate.argtypes = [vp, ctypes.c_int, vp, ctypes.c_double, vp, vp]
    L.or_vmb_aggregate.restype = ctypes.c_int64
    L.or_omega.argtypes = [vp]
    L.or_omega.restype = ctypes.c_double
    pp = ctypes.POINTER(vp)
    L.or_smoothed_prolongator.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_double, pp, pp, pp]
    L.or_transpose.argtypes = [vp, pp, pp, pp]
    L.or_galerkin.argtypes = [vp, vp, vp, pp, pp, pp]
    L._setup_sigs = True
    return L


def vmb_aggregate(A, theta=0.01, row_start=None):
    """Decoupled VMB aggregation (readings R17, R18, R20, R26).
    Returns (agg[n], root[n] (bool), n_aggregates)."""
    L = _setup_sigs()
    h = _CsrHolder(A)
    n = h.c.nrows
    rs = np.array([0, n] if row_start is None else row_start, np.int64)
    agg = np.empty(n, np.int64)
    root = np.zeros(n, np.int8)
    nc = L.or_vmb_aggregate(ctypes.byref(h.c), len(rs) - 1, rs.ctypes.data, float(theta), agg.ctypes.data,
                            root.ctypes.data)
    if nc < 0:
        raise RuntimeError("VMB phase 3 reached (a node farther than two strong edges from every root)")
    return agg, root.astype(bool), int(nc)


def omega(A) -> float:
    """omega = 1 / ||D^-1 A||_inf (reading R21)."""
    h = _CsrHolder(A)  # keeps the arrays alive during the call
    return _setup_sigs().or_omega(ctypes.byref(h.c))


def smoothed_prolongator(A, agg, nc, om):
    """P = (I - omega D^-1 A) P^, P^ of Eq. (3) with w = 1."""
    L = _setup_sigs()
    h = _CsrHolder(A)
    agg = _arr(agg, np.int64)
    pp, pc, pv = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    L.or_smoothed_prolongator(ctypes.byref(h.c), agg.ctypes.data, int(nc), float(om), ctypes.byref(pp),
                              ctypes.byref(pc), ctypes.byref(pv))
    return _take_csr(h.c.nrows, int(nc), pp.value, pc.value, pv.value)


def transpose(P):
    """R = P^T, rows by increasing column (BASELINE.json north_star: explicit R)."""
    L = _setup_sigs()
    h = _CsrHolder(P)
    pp, pc, pv = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    L.or_transpose(ctypes.byref(h.c), ctypes.byref(pp), ctypes.byref(pc), ctypes.byref(pv))
    return _take_csr(h.c.ncols, h.c.nrows, pp.value, pc.value, pv.value)


def galerkin(R, A, P):
    """A_c = R A P."""
    L = _setup_sigs()
    hr, ha, hp = _CsrHolder(R), _CsrHolder(A), _CsrHolder(P)
    pp, pc, pv = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    L.or_galerkin(ctypes.byref(hr.c), ctypes.byref(ha.c), ctypes.byref(hp.c), ctypes.byref(pp), ctypes.byref(pc),
                  ctypes.byref(pv))
    return _take_csr(hr.c.nrows, hp.c.ncols, pp.value, pc.value, pv.value)


class SetupLevel:
    def __init__(self, A, row_start):
        self.A, self.P, self.R, self.agg, self.root = A, None, None, None, None
        self.n = A.shape[0]
        self.row_start = np.asarray(row_start, np.int64)
        self.omega = None


class SetupHierarchy:
    """A hierarchy built by the oracle's set-up; usable by oracle.pcg / vcycle / fcg."""

    def __init__(self, levels):
        self.levels = levels

    @property
    def nlevels(self):
        return len(self.levels)

    def operator_complexity(self):
        return sum(L.A.nnz for L in self.levels) / self.levels[0].A.nnz


def amg_setup(A0, theta=0.01, max_levels=20, coarse_target=200, stall_ratio=0.75, row_start=None):
    """The set-up of P:196-240 level by level (readings R17-R21, R26): aggregate, smooth
    the tentative prolongator, R = P^T, A_{l+1} = R A_l P.  Stops when n_l <=
    coarse_target, when an aggregation would leave more than stall_ratio * n_l
    aggregates (R19), or at max_levels."""
    import scipy.sparse as sp
    A = sp.csr_matrix(A0)
    A.sort_indices()
    n = A.shape[0]
    rs = np.array([0, n] if row_start is None else row_start, np.int64)
    levels = [SetupLevel(A, rs)]
    while True:
        L = levels[-1]
        if L.n <= coarse_target or len(levels) >= max_levels:
            break
        agg, root, nc = vmb_aggregate(L.A, theta, L.row_start)
        if nc > stall_ratio * L.n or nc >= L.n:
            break
        om = omega(L.A)
        P = smoothed_prolongator(L.A, agg, nc, om)
        R = transpose(P)
        Ac = galerkin(R, L.A, P)
        # coarse row blocks: the aggregates of each fine block (decoupled, ids block by block)
        crs = np.zeros(len(L.row_start), np.int64)
        for r in range(len(L.row_start) - 1):
            crs[r + 1] = crs[r] + int(root[L.row_start[r]:L.row_start[r + 1]].sum())
        L.P, L.R, L.agg, L.root, L.omega = P, R, agg, root, om
        levels.append(SetupLevel(Ac, crs))
    return SetupHierarchy(levels)


# ------------------------------------------------------------------ NEXT-4 AINV
def ainv(A, drop_tol=0.1, row_start=None):
    """AINV factors (reading R27): A^-1 ~ Z D^-1 Z^T, Z unit upper triangular
    (returned as scipy CSC, columns z_j), D = diag(p).  Block-Jacobi over row_start."""
    import scipy.sparse as sp
    L = _setup_sigs()
    if not getattr(L, "_ainv_sig", False):
        pp = ctypes.POINTER(ctypes.c_void_p)
        L.or_ainv.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_double, pp, pp, pp,
                              ctypes.c_void_p]
        L.or_ainv.restype = ctypes.c_int
        L._ainv_sig = True
    h = _CsrHolder(A)
    n = h.c.nrows
    rs = np.array([0, n] if row_start is None else row_start, np.int64)
    p = np.zeros(n)
    zp, zr, zv = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    st = L.or_ainv(ctypes.byref(h.c), len(rs) - 1, rs.ctypes.data, float(drop_tol), ctypes.byref(zp),
                   ctypes.byref(zr), ctypes.byref(zv), p.ctypes.data)
    Zt = _take_csr(n, n, zp.value, zr.value, zv.value)  # rows of Zt = columns of Z
    if st != 0:
        raise RuntimeError(f"AINV breakdown: pivot {-1 - st} <= 0")
    return sp.csc_matrix((Zt.data, Zt.indices, Zt.indptr), shape=(n, n)), p
