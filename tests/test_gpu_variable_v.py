"""GPU parity of the variable V-cycle (its solve-path part):
"2 smoother iteration at the first level, and doubled at each following level"
(P:330 footnote, VMATCH), i.e. pre/post sweeps pre*2^l / post*2^l at level l
(reading R25), against oracle.vcycle(variable_v=True) / oracle.pcg (pinned in
tests/test_oracle_pins.py against the dense Eq. (2) composition).

Tolerances: V-cycle 1e-12 relative (summation order only, as the plain V-cycle
tests); PCG the BASELINE north_star bar (relative residuals within 1e-9 over the
first 20 iterations, iterations +-1 at tol 1e-8, final x within 1e-7).
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.cpu().numpy()


CASES = [(16, dict(max_levels=2)), (16, {}), ((13, 11, 7), dict(coarse_target=20)), (48, {}),
         (24, dict(problem="jump", cube=4, coarse_target=200))]


@pytest.mark.parametrize("dense_suffix", ["default", "off"])
@pytest.mark.parametrize("pre,post", [(2, 2), (1, 3)])
@pytest.mark.parametrize("grid,kw", CASES)
def test_variable_vcycle_parity(psc, grid, kw, pre, post, dense_suffix, monkeypatch):
    if dense_suffix == "off":
        monkeypatch.setenv("PSC_DENSE_SUFFIX_ROWS", "0")
    g = grid if isinstance(grid, tuple) else (grid,) * 3
    h = pscgen.poisson_hierarchy(*g, **kw)
    n = h.levels[0].n
    ctx = psc.Context()
    H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), pre=pre, post=post, variable_v=True)
    r = pscgen.rhs_random(11, 0, n)
    z = torch.zeros(n, dtype=torch.float64, device="cuda")
    H.vcycle(dev(r), z)
    zo = oracle.vcycle(h, r, pre, post, 30, variable_v=True)
    err = ew_err(host(z), zo)
    assert err <= 1e-12, err
    if h.nlevels > 2:  # really the variable cycle, not the plain one
        zp = oracle.vcycle(h, r, pre, post, 30)
        assert np.linalg.norm(zp - zo) / np.linalg.norm(zo) > 1e-6
    ctx.close()


@pytest.mark.parametrize("grid,kw", CASES + [(64, {})])
def test_variable_vcycle_pcg_parity(psc, grid, kw):
    g = grid if isinstance(grid, tuple) else (grid,) * 3
    h = pscgen.poisson_hierarchy(*g, **kw)
    n = h.levels[0].n
    b = pscgen.rhs_random(2, 0, n)
    ctx = psc.Context()
    H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), pre=2, post=2, variable_v=True)
    xo, ito, sto, histo = oracle.pcg(h, b, tol=1e-8, maxit=200, pre=2, post=2, variable_v=True)
    x = dev(np.zeros(n))
    rc, st, hist = H.solve(dev(b), x, tol=1e-8, maxit=200)
    assert sto == 0 and rc == 0
    assert abs(st["iters"] - ito) <= 1, (st["iters"], ito)
    k = min(20, ito, st["iters"]) + 1
    np.testing.assert_allclose(hist[:k], histo[:k], rtol=1e-9, atol=0)
    assert np.linalg.norm(host(x) - xo) / np.linalg.norm(xo) <= 1e-7
    ctx.close()


def test_variable_vcycle_rejects_overflowing_sweep_counts(psc):
    h = pscgen.poisson_hierarchy(16)
    assert h.nlevels >= 3
    ctx = psc.Context()
    with pytest.raises(psc.PscError):
        psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), pre=1 << 20, post=1, variable_v=True)
    ctx.close()


@pytest.mark.parametrize("grid,kw", [(16, {}), ((40, 24, 16), {}), (24, dict(problem="jump", cube=4, coarse_target=300))])
def test_variable_vcycle_vbm_choices_fcg_parity(psc, grid, kw):
    """VMATCH's "further algorithmic choices as in VBM": FCG(1) outer
    iterations and the coarsest PCG(<= 40) with l1-Jacobi, with the variable cycle."""
    g = grid if isinstance(grid, tuple) else (grid,) * 3
    h = pscgen.poisson_hierarchy(*g, **kw)
    n = h.levels[0].n
    b = pscgen.rhs_random(6, 0, n)
    ctx = psc.Context()
    H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), pre=2, post=2, variable_v=True,
                                coarse_solver="pcg")
    xo, ito, sto, histo = oracle.fcg(h, b, tol=1e-8, maxit=200, pre=2, post=2, variable_v=True, coarse_pcg=True)
    x = dev(np.zeros(n))
    rc, st, hist = H.solve(dev(b), x, tol=1e-8, maxit=200, method="fcg")
    assert sto == 0 and rc == 0
    assert abs(st["iters"] - ito) <= 1, (st["iters"], ito)
    k = min(20, ito, st["iters"]) + 1
    np.testing.assert_allclose(hist[:k], histo[:k], rtol=1e-9, atol=0)
    assert np.linalg.norm(host(x) - xo) / np.linalg.norm(xo) <= 1e-7
    ctx.close()


@pytest.mark.parametrize("grid", [16, (40, 24, 16), 48])
def test_variable_vcycle_unsmoothed_p_pcg_parity(psc, grid):
    """VMATCH's other solve-relevant choice: un-smoothed (tentative)
    prolongators, here on the decoupled aggregates, with the variable cycle."""
    g = grid if isinstance(grid, tuple) else (grid,) * 3
    h = pscgen.poisson_hierarchy(*g, smooth=False)
    n = h.levels[0].n
    b = pscgen.rhs_random(8, 0, n)
    ctx = psc.Context()
    H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), pre=2, post=2, variable_v=True)
    r = pscgen.rhs_random(9, 0, n)
    z = torch.zeros(n, dtype=torch.float64, device="cuda")
    H.vcycle(dev(r), z)
    zo = oracle.vcycle(h, r, 2, 2, 30, variable_v=True)
    assert ew_err(host(z), zo) <= 1e-12
    xo, ito, sto, histo = oracle.pcg(h, b, tol=1e-8, maxit=300, pre=2, post=2, variable_v=True)
    x = dev(np.zeros(n))
    rc, st, hist = H.solve(dev(b), x, tol=1e-8, maxit=300)
    assert sto == 0 and rc == 0
    assert abs(st["iters"] - ito) <= 1, (st["iters"], ito)
    k = min(20, ito, st["iters"]) + 1
    np.testing.assert_allclose(hist[:k], histo[:k], rtol=1e-9, atol=0)
    assert np.linalg.norm(host(x) - xo) / np.linalg.norm(xo) <= 1e-7
    ctx.close()
