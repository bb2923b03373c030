"""GPU parity of NEXT-4: the AINV smoother (reading R27;
factors built on the host by the library, applied on the device as SpMVs with Z^T and
Z) and the structure-preserving coefficient update + smoother rebuild,
against the oracle (oracle.vcycle / oracle.pcg with smoother="ainv"; pinned in
tests/test_oracle_ainv.py).

Bars: V-cycle element-wise within 1e-12 of max|z| (the library's AINV factors come
from the same biconjugation in the same operation order as the oracle's; the sweeps
differ by FMA contraction and 1/p vs division); PCG at the north-star bar.
"""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import pscgen  # noqa: E402
from _util import ew_err  # noqa: E402


@pytest.fixture(scope="module")
def psc():
    import paper_2406_19754_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("grid,kw,drop,sw", [(12, dict(coarse_target=30), 0.1, (1, 1)),
                                             ((13, 11, 7), dict(coarse_target=20), 0.05, (2, 2)),
                                             (16, dict(max_levels=2), 0.2, (1, 2)),
                                             (12, dict(problem="jump", cube=3, coarse_target=30), 0.1, (1, 1))],
                         ids=["poisson12", "ragged", "2level", "jump"])
def test_ainv_vcycle_and_pcg_parity(psc, grid, kw, drop, sw):
    g = grid if isinstance(grid, tuple) else (grid,) * 3
    h = pscgen.poisson_hierarchy(*g, **kw)
    n = h.levels[0].n
    pre, post = sw
    ctx = psc.Context()
    H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), pre=pre, post=post, smoother="ainv", ainv_drop=drop)
    okw = dict(pre=pre, post=post, smoother="ainv", ainv_drop=drop)
    # smoothing sweeps alone at every non-coarsest level
    for l in range(h.nlevels - 1):
        r = pscgen.rhs_random(l + 3, 0, h.levels[l].n)
        z = torch.zeros(h.levels[l].n, dtype=torch.float64, device="cuda")
        H.smooth(l, dev(r), z, 3)
        Z, p = oracle.ainv(h.levels[l].A, drop)
        A = h.levels[l].A.to_scipy()
        x = np.zeros(len(r))
        for _ in range(3):
            x = x + Z @ ((Z.T @ (r - A @ x)) / p)
        assert ew_err(host(z), x) <= 1e-12, l
    r = pscgen.rhs_random(9, 0, n)
    z = torch.zeros(n, dtype=torch.float64, device="cuda")
    H.vcycle(dev(r), z)
    assert ew_err(host(z), oracle.vcycle(h, r, **okw)) <= 1e-12
    b = pscgen.rhs_random(10, 0, n)
    xo, ito, sto, histo = oracle.pcg(h, b, tol=1e-8, maxit=200, **okw)
    x = dev(np.zeros(n))
    rc, st, hist = H.solve(dev(b), x, tol=1e-8, maxit=200)
    assert rc == 0 and sto == 0 and abs(st["iters"] - ito) <= 1
    k = min(20, ito, st["iters"]) + 1
    np.testing.assert_allclose(hist[:k], histo[:k], rtol=1e-9, atol=0)
    assert np.linalg.norm(host(x) - xo) / np.linalg.norm(xo) <= 1e-7
    # FCG on the same hierarchy (B fixed and SPD: FCG(1) = PCG)
    xo2, ito2, sto2, histo2 = oracle.fcg(h, b, tol=1e-8, maxit=200, **okw)
    x2 = dev(np.zeros(n))
    rc2, st2, hist2 = H.solve(dev(b), x2, tol=1e-8, maxit=200, method="fcg")
    assert rc2 == 0 and abs(st2["iters"] - ito2) <= 1
    ctx.close()


def _scaled_levels(h, f):
    """The hierarchy's per-rank pieces with A_0's values replaced by f(values) (same pattern)."""
    lv = pscgen.rank_levels(h, 0)
    ptr, col, val = lv[0]["A"]
    lv[0] = dict(lv[0])
    lv[0]["A"] = (ptr, col, f(np.asarray(val)))
    return lv


@pytest.mark.parametrize("smoother", ["l1", "ainv"])
def test_update_values_and_rebuild_smoothers(psc, smoother):
    """new A_0 coefficients on the same structure (psc_mat_update_values),
    then the smoothers rebuilt on the reused hierarchy (psc_hier_rebuild_smoothers):
    the V-cycle and PCG equal the oracle on {A_0', A_1.., P, R} (coarse levels kept)."""
    h = pscgen.poisson_hierarchy(12, coarse_target=30)
    n = h.levels[0].n
    ctx = psc.Context()
    H, descs, A, P, R = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), smoother=smoother, ainv_drop=0.1,
                                            pre=1 if smoother == "ainv" else 4, post=1 if smoother == "ainv" else 4)
    b = pscgen.rhs_random(2, 0, n)
    # new coefficients on the same pattern, still SPD (diagonally dominant): a variable
    # diagonal and scaled couplings
    A0 = h.levels[0].A.to_scipy().tocsr()
    rows = np.repeat(np.arange(n), np.diff(A0.indptr))
    newval = np.where(A0.indices == rows, A0.data * (1.1 + 0.2 * np.sin(rows)), 0.9 * A0.data)
    A[0].update_values(newval)
    # the matrix itself changed at once
    xr = pscgen.rhs_random(5, 0, n)
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    A[0].spmv(dev(xr), y)
    A0n = sp.csr_matrix((newval, A0.indices, A0.indptr), shape=A0.shape)
    np.testing.assert_allclose(host(y), A0n @ xr, rtol=1e-14, atol=1e-14 * np.abs(A0n @ xr).max())
    H.rebuild_smoothers()
    # oracle hierarchy: new A_0, the old P, R and coarse matrices
    class L:
        pass
    lv = []
    for l in range(h.nlevels):
        o = L()
        o.A = A0n if l == 0 else h.levels[l].A
        o.P, o.R = h.levels[l].P, h.levels[l].R
        o.n = h.levels[l].n
        lv.append(o)

    class Hh:
        levels = lv
        nlevels = h.nlevels
    okw = dict(smoother=smoother, ainv_drop=0.1, pre=1 if smoother == "ainv" else 4, post=1 if smoother == "ainv" else 4)
    z = torch.zeros(n, dtype=torch.float64, device="cuda")
    H.vcycle(dev(b), z)
    assert ew_err(host(z), oracle.vcycle(Hh, b, **okw)) <= 1e-12
    xo, ito, sto, histo = oracle.pcg(Hh, b, tol=1e-8, maxit=200, **okw)
    x = dev(np.zeros(n))
    rc, st, hist = H.solve(dev(b), x, tol=1e-8, maxit=200)
    assert rc == 0 and sto == 0 and abs(st["iters"] - ito) <= 1
    k = min(20, ito, st["iters"]) + 1
    np.testing.assert_allclose(hist[:k], histo[:k], rtol=1e-9, atol=0)
    assert np.linalg.norm(host(x) - xo) / np.linalg.norm(xo) <= 1e-7
    ctx.close()


def test_ainv_argument_errors(psc):
    h = pscgen.poisson_hierarchy(8, max_levels=2)
    ctx = psc.Context()
    with pytest.raises(psc.PscError) as e:
        psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), smoother="ainv", ainv_drop=-1.0)
    assert e.value.code == psc.PSC_ERR_ARG
    with pytest.raises(ValueError):
        psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), smoother="gauss-seidel")
    ctx.close()
