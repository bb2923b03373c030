"""Seeded synthetic inputs shared by the CUDA path and the oracle.

This module is the ONLY code both sides use.  It builds the *given* input of
the solve phase (BASELINE.json north_star: "over a given aggregation
hierarchy (level matrices A_l, prolongators P_l and R_l = P_l^T)") and the
right-hand sides.  It holds none of the solve-phase arithmetic: no l1
diagonal, no smoothing sweep, no V-cycle and no CG (those are in ``oracle/``
and in ``paper_2406_19754_b200/csrc`` separately).

The hierarchy follows PSCToolkit's VBM set-up (Sec.
2.3.1): decoupled Vanek-Mandel-Brezina aggregation, tentative prolongator
Eq. (3) with w = 1, prolongator smoothing P = (I - omega D^-1 A) P^ with
omega = 1/||D^-1 A||_inf, R = P^T, Galerkin A_{l+1} = P^T A P.
The C++ builder is ``pscgen/pscgen.cpp``; input recipe and readings in DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libpscgen.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile pscgen/pscgen.cpp -> pscgen/libpscgen.so (host C++, OpenMP)."""
    src = os.path.join(_HERE, "pscgen.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared",
                               "-std=c++17", "-o", tmp, src])
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        i64, i32, f64, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        L.pscgen_build_grid.restype = vp
        L.pscgen_build_grid.argtypes = [i64, i64, i64, i32, i32, i32, i32, f64, i64, f64, i32, i64, f64, i32, i32,
                                        i32]
        L.pscgen_build_csr.restype = vp
        L.pscgen_build_csr.argtypes = [i64, vp, vp, vp, i32, vp, f64, i32, i64, f64, i32, i32, i32]
        L.pscgen_match.restype = i64
        L.pscgen_match.argtypes = [i64, vp, vp, vp, vp, i32, vp, vp]
        L.pscgen_nlevels.restype = i32
        L.pscgen_nlevels.argtypes = [vp]
        L.pscgen_nranks.restype = i32
        L.pscgen_nranks.argtypes = [vp]
        L.pscgen_level_n.restype = i64
        L.pscgen_level_n.argtypes = [vp, i32]
        L.pscgen_omega.restype = f64
        L.pscgen_omega.argtypes = [vp, i32]
        L.pscgen_row_start.argtypes = [vp, i32, vp]
        L.pscgen_csr.restype = i32
        L.pscgen_csr.argtypes = [vp, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                 ctypes.POINTER(ctypes.POINTER(i64)), ctypes.POINTER(ctypes.POINTER(i64)),
                                 ctypes.POINTER(ctypes.POINTER(f64))]
        L.pscgen_agg.restype = ctypes.POINTER(i64)
        L.pscgen_agg.argtypes = [vp, i32]
        L.pscgen_free.argtypes = [vp]
        L.pscgen_set_threads.argtypes = [i32]
        _lib = L
    return _lib


@dataclass
class CSR:
    """Global CSR: int64 row_ptr, int64 global columns (strictly increasing per row), f64 values."""
    shape: tuple
    ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.ptr[-1]) if len(self.ptr) else 0

    def rows(self, r0: int, r1: int) -> "CSR":
        """Row block [r0, r1) with a re-based row_ptr (columns stay global)."""
        p0, p1 = int(self.ptr[r0]), int(self.ptr[r1])
        return CSR((r1 - r0, self.shape[1]), (self.ptr[r0:r1 + 1] - p0).astype(np.int64),
                   self.col[p0:p1], self.val[p0:p1])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col, self.ptr), shape=self.shape)


@dataclass
class Level:
    n: int
    row_start: np.ndarray  # nranks+1, contiguous row blocks of this level's index space
    A: CSR
    P: CSR | None = None   # n_l x n_{l+1}
    R: CSR | None = None   # n_{l+1} x n_l  (= P^T, stored explicitly)


class _Handle:
    """Owns the C hierarchy; every numpy view of its CSR arrays keeps it alive."""

    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h is not None and _lib is not None:
            _lib.pscgen_free(self.h)
            self.h = None


def _view(ptr, n, ctype, dtype, owner):
    """numpy view of n elements at a C pointer, holding a reference to `owner`."""
    buf = (ctype * n).from_address(ctypes.addressof(ptr.contents))
    buf._owner = owner
    return np.frombuffer(buf, dtype=dtype)


@dataclass
class Hierarchy:
    levels: list
    nranks: int
    meta: dict = field(default_factory=dict)
    _handle: object = None

    @property
    def nlevels(self) -> int:
        return len(self.levels)

    def operator_complexity(self) -> float:
        """sum_l nnz(A_l) / nnz(A_0) (Fig. 3 caption)."""
        return sum(L.A.nnz for L in self.levels) / self.levels[0].A.nnz

    def rank_piece(self, l: int, kind: str, r: int) -> CSR:
        """Rows of A_l / P_l / R_l owned by rank r (rows live in the row space's block)."""
        L = self.levels[l]
        if kind == "A":
            rs = L.row_start
            return L.A.rows(int(rs[r]), int(rs[r + 1]))
        if kind == "P":
            rs = L.row_start
            return L.P.rows(int(rs[r]), int(rs[r + 1]))
        if kind == "R":
            rs = self.levels[l + 1].row_start
            return L.R.rows(int(rs[r]), int(rs[r + 1]))
        raise ValueError(kind)



def _wrap(handle, meta) -> Hierarchy:
    L = lib()
    owner = _Handle(handle)
    nl = L.pscgen_nlevels(handle)
    nr = L.pscgen_nranks(handle)
    levels = []
    for l in range(nl):
        n = L.pscgen_level_n(handle, l)
        rs = np.zeros(nr + 1, dtype=np.int64)
        L.pscgen_row_start(handle, l, rs.ctypes.data)
        mats = []
        for kind in range(3):
            nrows, ncols = ctypes.c_int64(), ctypes.c_int64()
            pp = ctypes.POINTER(ctypes.c_int64)()
            cp = ctypes.POINTER(ctypes.c_int64)()
            vp = ctypes.POINTER(ctypes.c_double)()
            if L.pscgen_csr(handle, l, kind, ctypes.byref(nrows), ctypes.byref(ncols), ctypes.byref(pp),
                            ctypes.byref(cp), ctypes.byref(vp)) != 0:
                mats.append(None)
                continue
            ptr = _view(pp, nrows.value + 1, ctypes.c_int64, np.int64, owner)
            nnz = int(ptr[-1])
            col = _view(cp, nnz, ctypes.c_int64, np.int64, owner) if nnz else np.zeros(0, np.int64)
            val = _view(vp, nnz, ctypes.c_double, np.float64, owner) if nnz else np.zeros(0, np.float64)
            mats.append(CSR((nrows.value, ncols.value), ptr, col, val))
        levels.append(Level(n, rs, mats[0], mats[1], mats[2]))
    meta = dict(meta)
    meta["omega"] = [L.pscgen_omega(handle, l) for l in range(nl - 1)]
    return Hierarchy(levels, nr, meta, owner)


def poisson_hierarchy(nx: int, ny: int | None = None, nz: int | None = None, procs=(1, 1, 1), *,
                      problem: str = "poisson", jump: float = 1e4, cube: int = 32, theta: float = 0.01,
                      max_levels: int = 20, coarse_target: int = 200, stall_ratio: float = 0.75,
                      smooth: bool = True, threads: int = 0, aggregation: str = "vmb",
                      match_sweeps: int = 3) -> Hierarchy:
    """7-point 3D problem on an nx*ny*nz grid split in procs=(px,py,pz) rank boxes.

    problem="poisson": -lap u = 1; "jump": BASELINE.json config 5
    (coefficient `jump` on a checkerboard of `cube`^3 cubes; reading R22).
    aggregation="vmb": decoupled VMB; "matching": compatible weighted matching
    with match_sweeps sweeps, aggregates of at most 2^k nodes (SMATCH/VMATCH,
    P:329-330, reading R29).
    """
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    px, py, pz = procs
    if threads:
        lib().pscgen_set_threads(threads)
    if aggregation not in ("vmb", "matching"):
        raise ValueError("aggregation must be 'vmb' or 'matching'")
    h = lib().pscgen_build_grid(nx, ny, nz, px, py, pz, 0 if problem == "poisson" else 1, jump, cube, theta,
                                max_levels, coarse_target, stall_ratio, 1 if smooth else 0,
                                1 if aggregation == "matching" else 0, match_sweeps)
    if not h:
        raise ValueError("grid not divisible by the process grid")
    meta = dict(problem=problem, grid=(nx, ny, nz), procs=tuple(procs), theta=theta, max_levels=max_levels,
                coarse_target=coarse_target, stall_ratio=stall_ratio, smooth=smooth, aggregation=aggregation,
                jump=jump if problem != "poisson" else None, cube=cube if problem != "poisson" else None)
    return _wrap(h, meta)


def csr_hierarchy(A, row_start=None, *, theta: float = 0.01, max_levels: int = 20, coarse_target: int = 200,
                  stall_ratio: float = 0.75, smooth: bool = True, aggregation: str = "vmb",
                  match_sweeps: int = 3) -> Hierarchy:
    """Hierarchy from a user SPD matrix (scipy.sparse or dense ndarray), row blocks row_start."""
    import scipy.sparse as sp
    A = sp.csr_matrix(A)
    A.sort_indices()
    n = A.shape[0]
    if row_start is None:
        row_start = np.array([0, n], dtype=np.int64)
    row_start = np.ascontiguousarray(row_start, dtype=np.int64)
    ptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
    col = np.ascontiguousarray(A.indices, dtype=np.int64)
    val = np.ascontiguousarray(A.data, dtype=np.float64)
    h = lib().pscgen_build_csr(n, ptr.ctypes.data, col.ctypes.data, val.ctypes.data, len(row_start) - 1,
                               row_start.ctypes.data, theta, max_levels, coarse_target, stall_ratio,
                               1 if smooth else 0, 1 if aggregation == "matching" else 0, match_sweeps)
    return _wrap(h, dict(problem="csr", theta=theta, max_levels=max_levels, coarse_target=coarse_target))


# ----------------------------------------------------------------- right-hand sides
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on uint64 (wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def rhs_random(seed: int, start: int, count: int) -> np.ndarray:
    """u_i = splitmix64(seed XOR global_index) mapped to [-1, 1), for global rows
    [start, start+count).  Keyed by global index, so identical for any partition."""
    g = np.arange(start, start + count, dtype=np.uint64) ^ np.uint64(seed)
    z = splitmix64(g)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -52) - 1.0


def rhs_poisson(grid, start: int, count: int) -> np.ndarray:
    """b = h^2 * f with f = 1 and h = 1/(nx_global + 1) (reading R15)."""
    h = 1.0 / (grid[0] + 1)
    return np.full(count, h * h, dtype=np.float64)


def rank_levels(h: Hierarchy, r: int) -> list:
    """Per-level inputs of rank r for the C ABI (psc_desc_create / psc_mat_create_csr):
    n_global, row_start, and this rank's CSR rows (row_ptr, int64 global cols, values)
    of A_l, P_l (rows in space l) and R_l (rows in space l+1)."""
    out = []
    for l, L in enumerate(h.levels):
        d = dict(n_global=L.n, row_start=L.row_start)
        A = h.rank_piece(l, "A", r)
        d["A"] = (A.ptr, A.col, A.val)
        if l < h.nlevels - 1:
            P = h.rank_piece(l, "P", r)
            R = h.rank_piece(l, "R", r)
            d["P"] = (P.ptr, P.col, P.val)
            d["R"] = (R.ptr, R.col, R.val)
        out.append(d)
    return out


def match(A, w=None, k=1):
    """One matching aggregation (reading R29) of a square matrix with near-kernel
    vector w (default 1): returns (agg, values of P^ per node, number of aggregates)."""
    import scipy.sparse as sp
    A = sp.csr_matrix(A)
    A.sort_indices()
    n = A.shape[0]
    w = np.ones(n) if w is None else np.ascontiguousarray(w, dtype=np.float64)
    ptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
    col = np.ascontiguousarray(A.indices, dtype=np.int64)
    val = np.ascontiguousarray(A.data, dtype=np.float64)
    agg = np.zeros(n, np.int64)
    ph = np.zeros(n)
    nc = lib().pscgen_match(n, ptr.ctypes.data, col.ctypes.data, val.ctypes.data, w.ctypes.data, int(k),
                            agg.ctypes.data, ph.ctypes.data)
    return agg, ph, int(nc)
