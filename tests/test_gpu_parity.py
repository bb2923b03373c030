"""GPU parity: the CUDA path (through the C ABI, libpsc.so) against the CPU
oracle on identical seeded inputs.

Tolerances (BASELINE.json north_star): per-iteration relative residuals within
1e-9 relative over the first 20 iterations; same iteration count +-1 at tol 1e-8;
final-solution relative 2-norm difference <= 1e-7.  Kernel-level checks
(SpMV, l1 diagonal, sweeps, V-cycle) use tolerances derived in DESIGN.md §6
from the arithmetic (FMA vs separate multiply-add, reciprocal vs division).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import pscgen  # noqa: E402
from _util import ew_err  # noqa: E402


@pytest.fixture(scope="module")
def psc():
    import paper_2406_19754_b200 as m
    return m


_CACHE = {}


def setup(psc, grid, procs=(1, 1, 1), **kw):
    key = (grid, procs, tuple(sorted(kw.items())))
    if key not in _CACHE:
        g = grid if isinstance(grid, tuple) else (grid, grid, grid)
        opts = {k: kw[k] for k in ("pre", "post", "coarse") if k in kw}
        gk = {k: v for k, v in kw.items() if k not in opts}
        h = pscgen.poisson_hierarchy(*g, procs=procs, **gk)
        ctx = psc.Context()
        H, descs, A, P, R = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), **opts)
        _CACHE[key] = (h, ctx, H, A, P, R, opts)
    return _CACHE[key]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.cpu().numpy()


def rowscale(M, x):
    """(|M| |x|)_i: the scale of rounding differences in row i of M x."""
    import scipy.sparse as sp
    S = M.to_scipy()
    return abs(S) @ np.abs(x)


# --------------------------------------------------------------------- SpMV
@pytest.mark.parametrize("grid", [16, (13, 11, 7), 32])
def test_spmv_all_level_matrices(psc, grid):
    h, ctx, H, A, P, R, _ = setup(psc, grid, coarse_target=20)
    rng = np.random.default_rng(1)
    for l in range(h.nlevels):
        mats = [("A", h.levels[l].A, A[l])]
        if l < h.nlevels - 1:
            mats += [("P", h.levels[l].P, P[l]), ("R", h.levels[l].R, R[l])]
        for name, M, Mg in mats:
            x = rng.standard_normal(M.shape[1])
            y0 = rng.standard_normal(M.shape[0])
            ref = 1.5 * oracle.spmv(M, x) - 0.5 * y0
            y = dev(y0)
            Mg.spmv(dev(x), y, alpha=1.5, beta=-0.5)
            err = np.abs(host(y) - ref)
            tol = 1e-14 * (1.5 * rowscale(M, x) + 0.5 * np.abs(y0)) + 1e-300
            assert np.all(err <= tol), (name, l, float((err / tol).max()))


@pytest.mark.parametrize("env", [{}, {"PSC_NO_DIA": "1"}, {"PSC_NO_DIA": "1", "PSC_NO_TMA": "1"},
                                 {"PSC_COL16": "0", "PSC_NO_DIA": "1"}], ids=["default", "ell", "ell-notma", "col32"])
def test_spmv_mixed_column_spans(psc, env, monkeypatch):
    """Slices of at most 8 columns whose columns span less than 2^16 store 16-bit column
    offsets (kEll16), the others 32-bit columns: a tridiagonal matrix plus far couplings
    every 97th row (span ~10^5) mixes both kinds; SpMV against the oracle."""
    import scipy.sparse as sp
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    n = 200_003
    i = np.arange(0, n, 97)
    j = (i + 100_003) % n
    far = sp.coo_matrix((np.full(len(i), -0.25), (i, j)), shape=(n, n))
    A = (sp.diags([-np.ones(n - 1), 4 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1]) + far + far.T).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    ctx = psc.Context()
    d = psc.Descriptor(ctx, n, [0, n])
    M = psc.Matrix(ctx, d, d, A.indptr, A.indices, A.data)
    d.assemble()
    M.assemble()
    rng = np.random.default_rng(5)
    x = rng.standard_normal(n)
    y = dev(np.zeros(n))
    M.spmv(dev(x), y)
    h = pscgen.csr_hierarchy(A, max_levels=1)
    ref = oracle.spmv(h.levels[0].A, x)
    err = np.abs(host(y) - ref)
    assert np.all(err <= 1e-14 * (abs(A) @ np.abs(x)) + 1e-300)
    ctx.close()


def _check_layout(M, info):
    lens = np.diff(M.ptr)
    n = len(lens)
    G = info["lanes"]
    assert info["nnz"] == M.nnz and info["n_rows"] == n
    if G == 1:  # sliced ELL, 32-row slices padded to the slice's longest row (ELL slices) or
        # to the slice's number of distinct diagonals (DIA slices): padded >= 32 * sum of widths
        nsl = (n + 31) // 32
        pad = np.zeros(nsl * 32, np.int64)
        pad[:n] = lens
        assert info["n_units"] == nsl
        widths = int(pad.reshape(nsl, 32).max(axis=1).sum()) * 32
        assert widths <= info["padded"] <= 1.5 * widths
    else:  # row groups: rows padded to multiples of G, 32/G rows per warp
        assert G in (4, 8, 16, 32)
        assert info["n_units"] == (n + 32 // G - 1) // (32 // G)
        assert info["padded"] == int((((lens + G - 1) // G) * G).sum())
    mean = M.nnz / max(n, 1)
    assert (G == 1) == (mean < 100)


def test_device_layout_info(psc):
    h, ctx, H, A, P, R, _ = setup(psc, 32)
    for l in range(h.nlevels):
        _check_layout(h.levels[l].A, A[l].info())
        if l < h.nlevels - 1:
            _check_layout(h.levels[l].P, P[l].info())
            _check_layout(h.levels[l].R, R[l].info())


# ---------------------------------------------------------- l1 diag / sweeps
@pytest.mark.parametrize("grid", [16, (13, 11, 7)])
def test_l1_dinv_bit_exact(psc, grid):
    h, ctx, H, *_ = setup(psc, grid, coarse_target=20)
    for l in range(h.nlevels):
        n = h.levels[l].n
        out = torch.zeros(n, dtype=torch.float64, device="cuda")
        H.dinv(l, out)
        ref = 1.0 / oracle.l1_diag(h.levels[l].A)
        assert np.array_equal(host(out), ref)


@pytest.mark.parametrize("nsweeps", [1, 2, 4, 30])
def test_smoother_sweeps_every_level(psc, nsweeps):
    h, ctx, H, *_ = setup(psc, (13, 11, 7), coarse_target=20)
    rng = np.random.default_rng(nsweeps)
    for l in range(h.nlevels):
        n = h.levels[l].n
        b = rng.standard_normal(n)
        x = torch.zeros(n, dtype=torch.float64, device="cuda")
        H.smooth(l, dev(b), x, nsweeps)
        ref = oracle.l1_sweeps_from_zero(h.levels[l].A, b, nsweeps)
        err = ew_err(host(x), ref)
        assert err <= 1e-13 * nsweeps, (l, err)


# ------------------------------------------------------------------ V-cycle
@pytest.mark.parametrize("grid,kw", [(16, dict(max_levels=2)), (16, {}), ((13, 11, 7), dict(coarse_target=20)),
                                     (32, dict(pre=2, post=3, coarse=7))])
def test_vcycle(psc, grid, kw):
    h, ctx, H, A, P, R, opts = setup(psc, grid, **kw)
    n = h.levels[0].n
    for seed in (1, 2):
        r = pscgen.rhs_random(seed, 0, n)
        z = torch.zeros(n, dtype=torch.float64, device="cuda")
        H.vcycle(dev(r), z)
        ref = oracle.vcycle(h, r, opts.get("pre", 4), opts.get("post", 4), opts.get("coarse", 30))
        err = ew_err(host(z), ref)
        assert err <= 1e-12, err


# ---------------------------------------------------------------------- PCG
def _pcg_parity(psc, grid, b, x0=None, tol=1e-8, maxit=200, **kw):
    h, ctx, H, A, P, R, opts = setup(psc, grid, **kw)
    xo, ito, sto, histo = oracle.pcg(h, b, x0=x0, tol=tol, maxit=maxit, pre=opts.get("pre", 4),
                                     post=opts.get("post", 4), coarse=opts.get("coarse", 30))
    x = dev(np.zeros(len(b)) if x0 is None else x0)
    rc, st, hist = H.solve(dev(b), x, tol=tol, maxit=maxit)
    xg = host(x)
    assert sto == 0 and rc == 0
    assert abs(st["iters"] - ito) <= 1
    k = min(20, ito, st["iters"]) + 1
    np.testing.assert_allclose(hist[:k], histo[:k], rtol=1e-9, atol=0)
    assert np.linalg.norm(xg - xo) / np.linalg.norm(xo) <= 1e-7
    return st, hist, xg


@pytest.mark.parametrize("rhs", ["poisson", 1, 2, 3])
def test_pcg_c1_16cube_two_level(psc, rhs):
    """BASELINE.json configs[0]: 16^3, 2-level aggregation AMG, PCG tol 1e-8, 1 GPU."""
    n = 16 ** 3
    b = pscgen.rhs_poisson((16, 16, 16), 0, n) if rhs == "poisson" else pscgen.rhs_random(rhs, 0, n)
    st, hist, x = _pcg_parity(psc, 16, b, max_levels=2)
    assert st["status"] == 0 and hist[-1] <= 1e-8


@pytest.mark.parametrize("grid", [(13, 11, 7), (40, 24, 16)])
def test_pcg_ragged_multilevel(psc, grid):
    n = int(np.prod(grid))
    _pcg_parity(psc, grid, pscgen.rhs_random(9, 0, n), coarse_target=20)


def test_pcg_nonzero_initial_guess_and_jump(psc):
    n = 24 ** 3
    x0 = pscgen.rhs_random(5, 0, n)
    _pcg_parity(psc, 24, pscgen.rhs_random(4, 0, n), x0=x0, problem="jump", cube=4)


def test_pcg_edge_cases(psc):
    h, ctx, H, *_ = setup(psc, 16, max_levels=2)
    n = h.levels[0].n
    # b = 0 -> x = 0, 0 iterations
    x = dev(np.ones(n))
    rc, st, hist = H.solve(dev(np.zeros(n)), x)
    assert rc == 0 and st["iters"] == 0 and not host(x).any()
    # maxit = 0 -> not converged, history has the initial residual only
    b = pscgen.rhs_random(1, 0, n)
    x = dev(np.zeros(n))
    rc, st, hist = H.solve(dev(b), x, maxit=0)
    assert rc == psc.PSC_NOT_CONVERGED and st["iters"] == 0 and hist[0] == pytest.approx(1.0, rel=1e-15)
    # tol met by x0 -> 0 iterations
    rc, st, hist = H.solve(dev(b), x, tol=2.0)
    assert rc == 0 and st["iters"] == 0


def test_pcg_deterministic_and_host_path(psc):
    h, ctx, H, *_ = setup(psc, 32)
    n = h.levels[0].n
    b = pscgen.rhs_random(2, 0, n)
    x1, x2 = dev(np.zeros(n)), dev(np.zeros(n))
    _, s1, h1 = H.solve(dev(b), x1)
    _, s2, h2 = H.solve(dev(b), x2)
    assert torch.equal(x1, x2) and np.array_equal(h1, h2)
    xh = np.zeros(n)
    _, s3, h3 = H.solve_host(b, xh)
    assert np.array_equal(xh, host(x1)) and np.array_equal(h3, h1)
    assert s3["h2d_bytes"] == 16 * n and s3["d2h_bytes"] == 8 * n


@pytest.mark.parametrize("rhs", ["poisson", 1])
def test_pcg_c2_128cube(psc, rhs):
    """BASELINE.json configs[1]: 128^3 Poisson, full V-cycle hierarchy, 1 B200."""
    n = 128 ** 3
    b = pscgen.rhs_poisson((128,) * 3, 0, n) if rhs == "poisson" else pscgen.rhs_random(rhs, 0, n)
    st, hist, x = _pcg_parity(psc, 128, b)
    assert st["status"] == 0


def test_breakdown_is_reported(psc):
    """Indefinite A: p^T A p <= 0 must come back as PSC_ERR_BREAKDOWN."""
    import scipy.sparse as sp
    A = sp.csr_matrix(np.diag([1.0, -1.0]))
    h = pscgen.csr_hierarchy(A, max_levels=1)
    ctx = psc.Context()
    H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), pre=1, post=1, coarse=1)
    x = dev(np.zeros(2))
    with pytest.raises(psc.PscError) as e:
        H.solve(dev(np.ones(2)), x)
    assert e.value.code == psc.PSC_ERR_BREAKDOWN


# ------------------------------------------------ kernel / layout variants
# Every code path of the library (TMA-staged vs plain row kernels, DIA vs ELL
# slices, row-group lane counts, dense vs sparse one-CTA coarsest solver) must
# give the oracle's answer.  The switches are read at assembly (layout), at
# hierarchy creation (coarsest solver) and at launch (kernel family).
VARIANTS = [
    {},
    {"PSC_NO_TMA": "1"},
    {"PSC_NO_FUSED_SCALE": "1"},
    {"PSC_NO_DIA": "1"},
    {"PSC_NO_RG_TMA": "1", "PSC_NO_DENSE_COARSE": "1"},
    {"PSC_LANES": "1", "PSC_NO_DENSE_COARSE": "1"},
    {"PSC_LANES": "8"},
    {"PSC_LANES": "32", "PSC_NO_TMA": "1"},
    {"PSC_RG_MIN": "4", "PSC_RG_DIV": "1"},
    {"PSC_SORT": "1"},
    {"PSC_SORT": "1", "PSC_NO_TMA": "1", "PSC_NO_DENSE_COARSE": "1", "PSC_NO_DIA": "1"},
    {"PSC_RG_SMALL_MB": "200"},
    {"PSC_DIA_MAX": "64"},
    {"PSC_NO_FUSED_SCALE": "1", "PSC_NO_DIA": "1", "PSC_NO_TMA": "1"},
    {"PSC_COL16": "0"},
    {"PSC_COL16": "0", "PSC_NO_DIA": "1", "PSC_NO_TMA": "1"},
    {"PSC_NO_TMA4": "1"},
    {"PSC_TMA_RING": "1", "PSC_TMA_RING_E16": "2"},
    {"PSC_TMA_RING": "3", "PSC_TMA_RING_ANY": "2"},
    {"PSC_TMA_RING": "4", "PSC_NO_XPRE": "1"},
]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
@pytest.mark.parametrize("grid", [(21, 19, 17), 40])
def test_variants_pcg_parity(psc, env, grid, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = grid if isinstance(grid, tuple) else (grid,) * 3
    h = pscgen.poisson_hierarchy(*g, coarse_target=60)
    ctx = psc.Context()
    H, descs, A, P, R = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0))
    n = h.levels[0].n
    b = pscgen.rhs_random(17, 0, n)
    for l in range(h.nlevels):
        r = pscgen.rhs_random(l + 3, 0, h.levels[l].n)
        z = torch.zeros(h.levels[l].n, dtype=torch.float64, device="cuda")
        H.smooth(l, dev(r), z, 5)
        ref = oracle.l1_sweeps_from_zero(h.levels[l].A, r, 5)
        assert ew_err(host(z), ref) <= 1e-12
    z = torch.zeros(n, dtype=torch.float64, device="cuda")
    H.vcycle(dev(b), z)
    zo = oracle.vcycle(h, b)
    assert ew_err(host(z), zo) <= 1e-12
    xo, ito, sto, histo = oracle.pcg(h, b, tol=1e-8, maxit=100)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    rc, st, hist = H.solve(dev(b), x, tol=1e-8, maxit=100)
    assert rc == 0 and abs(st["iters"] - ito) <= 1
    k = min(20, ito, st["iters"]) + 1
    np.testing.assert_allclose(hist[:k], histo[:k], rtol=1e-9, atol=0)
    assert np.linalg.norm(host(x) - xo) / np.linalg.norm(xo) <= 1e-7
    ctx.close()


@pytest.mark.slow
def test_pcg_full_size_256cube_bench_config(psc):
    """BASELINE.json configs[2] at full size, in bench.py's launch configuration
    (256^3, one rank, default layouts/kernels, b = h^2 1, x0 = 0, tol 1e-8): the
    whole oracle solve (~2-3 min single-threaded) against the GPU solve."""
    g = 256
    h = pscgen.poisson_hierarchy(g)
    n = h.levels[0].n
    b = pscgen.rhs_poisson((g, g, g), 0, n)
    ctx = psc.Context()
    H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0))
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    rc, st, hist = H.solve(dev(b), x, tol=1e-8, maxit=200)
    xg = host(x)
    # one V-cycle compared in full
    r = pscgen.rhs_random(23, 0, n)
    z = torch.zeros(n, dtype=torch.float64, device="cuda")
    H.vcycle(dev(r), z)
    zo = oracle.vcycle(h, r)
    assert ew_err(host(z), zo) <= 1e-12
    xo, ito, sto, histo = oracle.pcg(h, b, tol=1e-8, maxit=200)
    assert rc == 0 and sto == 0 and abs(st["iters"] - ito) <= 1
    k = min(20, ito, st["iters"]) + 1
    np.testing.assert_allclose(hist[:k], histo[:k], rtol=1e-9, atol=0)
    assert np.linalg.norm(xg - xo) / np.linalg.norm(xo) <= 1e-7
    ctx.close()


@pytest.mark.parametrize("name", ["tridiag40", "poisson6"])
def test_one_level_hierarchy_pcg_parity(psc, name):
    """A one-level hierarchy: the coarsest solver (l1-Jacobi sweeps from zero) is the
    whole preconditioner, and the Krylov iteration's (r, z) is reduced after it."""
    if name == "tridiag40":
        import scipy.sparse as sp
        A = sp.diags([-np.ones(39), 2 * np.ones(40), -np.ones(39)], [-1, 0, 1], format="csr")
        h = pscgen.csr_hierarchy(A, max_levels=1)
    else:
        h = pscgen.poisson_hierarchy(6, max_levels=1)
    n = h.levels[0].n
    b = pscgen.rhs_random(3, 0, n)
    for coarse in (1, 3, 30):
        ctx = psc.Context()
        H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), pre=1, post=1, coarse=coarse)
        # tol 1e-6: with a one-sweep l1-Jacobi preconditioner the 1-D operator is ill
        # conditioned enough that residuals below ~1e-10 differ in the 9th digit by the
        # dot-product order alone
        xo, ito, sto, histo = oracle.pcg(h, b, tol=1e-6, maxit=100, pre=1, post=1, coarse=coarse)
        x = dev(np.zeros(n))
        rc, st, hist = H.solve(dev(b), x, tol=1e-6, maxit=100)
        assert rc == 0 and sto == 0 and abs(st["iters"] - ito) <= 1, (coarse, st["iters"], ito)
        k = min(20, ito, st["iters"]) + 1
        np.testing.assert_allclose(hist[:k], histo[:k], rtol=1e-9, atol=0)
        assert np.linalg.norm(host(x) - xo) / np.linalg.norm(xo) <= 1e-7
        ctx.close()
