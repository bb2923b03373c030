"""Small helpers for tests: grid numbering of pscgen's rank-major ordering and
closed forms of the 7-point operator.  No solve-phase arithmetic here."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, "paper_pins.json")) as f:
        return json.load(f)[name]["value"]


def grid_coords(nx, ny, nz, procs):
    """(gx, gy, gz) of every global row under pscgen's numbering: rank-major
    boxes (rank = rx + px*(ry + py*rz)), x-fastest inside a box."""
    px, py, pz = procs
    bx, by, bz = nx // px, ny // py, nz // pz
    g = np.arange(nx * ny * nz, dtype=np.int64)
    bn = bx * by * bz
    r, li = g // bn, g % bn
    rx, ry, rz = r % px, (r // px) % py, r // (px * py)
    lx, ly, lz = li % bx, (li // bx) % by, li // (bx * by)
    return rx * bx + lx, ry * by + ly, rz * bz + lz


def poisson_eigpair(nx, ny, nz, procs, i, j, k):
    """Eigenpair of the unscaled 7-point Dirichlet Laplacian (6, -1):
    lambda = 6 - 2cos(i pi/(nx+1)) - 2cos(j pi/(ny+1)) - 2cos(k pi/(nz+1)),
    v = sin(i pi (x+1)/(nx+1)) sin(j pi (y+1)/(ny+1)) sin(k pi (z+1)/(nz+1))."""
    gx, gy, gz = grid_coords(nx, ny, nz, procs)
    v = (np.sin(i * np.pi * (gx + 1) / (nx + 1)) * np.sin(j * np.pi * (gy + 1) / (ny + 1))
         * np.sin(k * np.pi * (gz + 1) / (nz + 1)))
    lam = 6 - 2 * np.cos(i * np.pi / (nx + 1)) - 2 * np.cos(j * np.pi / (ny + 1)) - 2 * np.cos(k * np.pi / (nz + 1))
    return lam, v


def poisson_exact_solve(nx, ny, nz, procs, b):
    """x = A^{-1} b for the unscaled 7-point Dirichlet Laplacian by the separable
    sine (DST-I) eigenbasis — a closed form independent of any iteration."""
    from scipy.fft import dstn, idstn
    gx, gy, gz = grid_coords(nx, ny, nz, procs)
    B = np.zeros((nz, ny, nx))
    B[gz, gy, gx] = b
    lx = 2 - 2 * np.cos(np.arange(1, nx + 1) * np.pi / (nx + 1))
    ly = 2 - 2 * np.cos(np.arange(1, ny + 1) * np.pi / (ny + 1))
    lz = 2 - 2 * np.cos(np.arange(1, nz + 1) * np.pi / (nz + 1))
    lam = lz[:, None, None] + ly[None, :, None] + lx[None, None, :]
    X = idstn(dstn(B, type=1) / lam, type=1)
    return X[gz, gy, gx]


def tridiag(n, a=-1.0, d=2.0):
    import scipy.sparse as sp
    return sp.diags([np.full(n - 1, a), np.full(n, d), np.full(n - 1, a)], [-1, 0, 1], format="csr")


def random_spd(n, density, seed):
    """Random sparse SPD matrix: symmetric pattern, diagonally dominant-ish."""
    import scipy.sparse as sp
    rng = np.random.default_rng(seed)
    M = sp.random(n, n, density=density, random_state=rng, data_rvs=lambda m: -rng.random(m))
    M = (M + M.T) * 0.5
    M = M.tolil()
    M.setdiag(0)
    M = M.tocsr()
    d = np.asarray(abs(M).sum(axis=1)).ravel() * rng.uniform(1.0, 1.5, n) + 0.1
    return (M + sp.diags(d)).tocsr()


def random_spd_mixed(n, density, seed):
    """Random sparse SPD with mixed-sign off-diagonals, not diagonally dominant: C^T C + 0.05 I."""
    import scipy.sparse as sp
    rng = np.random.default_rng(seed)
    C = sp.random(n, n, density=density, random_state=rng, data_rvs=lambda m: rng.standard_normal(m))
    C = C + sp.eye(n)
    return (C.T @ C + 0.05 * sp.eye(n)).tocsr()


def ew_err(a, ref):
    """Element-wise error scaled by the reference's magnitude: max_i |a_i - ref_i| / max_i |ref_i|
    (every component is held to the bound, unlike a relative 2-norm)."""
    a, ref = np.asarray(a), np.asarray(ref)
    return float(np.max(np.abs(a - ref)) / np.max(np.abs(ref)))
