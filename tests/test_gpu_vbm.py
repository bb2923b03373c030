"""GPU parity of the paper's VBM solve configuration:
the coarsest-level PCG with the l1-Jacobi preconditioner, at most 40 iterations
(P:328), and Notay's flexible CG, FCG(1), as the outer Krylov method (P:314,
P:318), against the CPU oracle (oracle.coarse_pcg, oracle.vcycle(coarse_pcg=True),
oracle.fcg; pinned in tests/test_oracle_pins.py).

Tolerances: the BASELINE north_star bar for the outer solve (per-iteration
relative residual within 1e-9 for the first 20 iterations, iterations +-1 at
tol 1e-8, final x within 1e-7).  The coarse PCG run for a FIXED number of
iterations (coarse_tol = 1e-300, the residual test never fires) is compared
iterate for iterate at 1e-12 (summation order of the dots only); with the
default coarse_tol = 1e-10 the two sides may stop one coarse iteration apart,
so the coarse result and the V-cycle are compared at 1e-9 (the size of the
last coarse correction, <= 1e-10 ||b|| times the coarse condition number).
"""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import pscgen  # noqa: E402
from _util import random_spd, random_spd_mixed  # noqa: E402


@pytest.fixture(scope="module")
def psc():
    import paper_2406_19754_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.cpu().numpy()


def one_level(psc, A, **kw):
    """1-level hierarchy: its V-cycle IS the coarsest solver B_ell applied to r."""
    h = pscgen.csr_hierarchy(sp.csr_matrix(A), max_levels=1)
    ctx = psc.Context()
    H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), coarse_solver="pcg", **kw)
    return h, ctx, H


def coarse_apply(H, b):
    z = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    H.vcycle(dev(b), z)
    return host(z)


# ------------------------------------------------------- coarsest PCG alone
def test_coarse_pcg_spec_examples(psc):
    # [2] x = 4 -> 2 ; diag(1..5) -> 1/(1..5)
    h, ctx, H = one_level(psc, np.array([[2.0]]))
    assert coarse_apply(H, np.array([4.0]))[0] == 2.0
    ctx.close()
    h, ctx, H = one_level(psc, np.diag(np.arange(1.0, 6.0)))
    np.testing.assert_allclose(coarse_apply(H, np.ones(5)), 1.0 / np.arange(1.0, 6.0), rtol=1e-15)
    ctx.close()


# dense one-CTA kernel (n <= 144) and the general launch-per-step form (forced
# with PSC_NO_DENSE_COARSE, and by size: 7-point 8^3 = 512 rows)
CASES = [("spd100", {}), ("spd100", {"PSC_NO_DENSE_COARSE": "1"}), ("poisson5", {}),
         ("poisson5", {"PSC_NO_DENSE_COARSE": "1"}), ("poisson8", {}), ("spd300", {})]


# default-tolerance cases: matrices the 40 coarse iterations solve to 1e-10 (on
# the ill-conditioned mixed-sign ones both sides stop at 40 iterations and
# differ by CG's rounding amplification, which the fixed-count test bounds)
CASES_TOL = [("dd100", {}), ("dd100", {"PSC_NO_DENSE_COARSE": "1"}), ("poisson5", {}),
             ("poisson5", {"PSC_NO_DENSE_COARSE": "1"}), ("poisson8", {}), ("dd300", {})]


def _mat(name):
    if name.startswith("spd"):
        return random_spd_mixed(int(name[3:]), 0.05, 4)
    if name.startswith("dd"):
        return random_spd(int(name[2:]), 0.05, 4)
    g = int(name[7:])
    return pscgen.poisson_hierarchy(g, max_levels=1).levels[0].A.to_scipy()


@pytest.mark.parametrize("name,env", CASES, ids=lambda c: c if isinstance(c, str) else ",".join(c) or "default")
def test_coarse_pcg_fixed_iterations_iterate_parity(psc, name, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    A = _mat(name)
    n = A.shape[0]
    b = pscgen.rhs_random(11, 0, n)
    for maxit in (1, 2, 5, 12):
        h, ctx, H = one_level(psc, A, coarse_maxit=maxit, coarse_tol=1e-300)
        x = coarse_apply(H, b)
        xo, it = oracle.coarse_pcg(A, b, maxit=maxit, tol=1e-300)
        assert it == maxit
        assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 1e-12, maxit
        ctx.close()


@pytest.mark.parametrize("name,env", CASES_TOL, ids=lambda c: c if isinstance(c, str) else ",".join(c) or "default")
def test_coarse_pcg_default_tolerance(psc, name, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    A = _mat(name)
    n = A.shape[0]
    h, ctx, H = one_level(psc, A)  # coarse_maxit 40, coarse_tol 1e-10 (R23)
    for seed in (1, 2):
        b = pscgen.rhs_random(seed, 0, n)
        x = coarse_apply(H, b)
        xo, it = oracle.coarse_pcg(A, b, maxit=40, tol=1e-10)
        assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 1e-9
    # b = 0 -> x = 0 (no iteration)
    assert not coarse_apply(H, np.zeros(n)).any()
    ctx.close()


def test_coarse_pcg_breakdown_keeps_iterate(psc):
    """p^T A p <= 0 on an indefinite coarsest matrix: the coarse PCG stops and keeps x
    (oracle: k -= 1; break), on both forms."""
    A = np.diag([1.0, -1.0, 2.0])
    b = np.array([1.0, 1.0, 1.0])
    xo, it = oracle.coarse_pcg(sp.csr_matrix(A), b, maxit=40, tol=1e-10)
    for env in ({}, {"PSC_NO_DENSE_COARSE": "1"}):
        mp = pytest.MonkeyPatch()
        for k, v in env.items():
            mp.setenv(k, v)
        h, ctx, H = one_level(psc, A)
        x = coarse_apply(H, b)
        np.testing.assert_allclose(x, xo, rtol=1e-14, atol=0)
        ctx.close()
        mp.undo()


# --------------------------------------------------------- V-cycle with it
@pytest.mark.parametrize("grid,kw", [(16, dict(max_levels=2)), ((13, 11, 7), dict(coarse_target=20)), (32, {}),
                                     (24, dict(problem="jump", cube=4, coarse_target=200))])
def test_vcycle_with_coarse_pcg(psc, grid, kw):
    g = grid if isinstance(grid, tuple) else (grid,) * 3
    h = pscgen.poisson_hierarchy(*g, **kw)
    n = h.levels[0].n
    for ck in (dict(coarse_maxit=40, coarse_tol=1e-300), dict()):
        ctx = psc.Context()
        H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), coarse_solver="pcg", **ck)
        r = pscgen.rhs_random(5, 0, n)
        z = torch.zeros(n, dtype=torch.float64, device="cuda")
        H.vcycle(dev(r), z)
        zo = oracle.vcycle(h, r, coarse_pcg=True, **ck)
        err = np.linalg.norm(host(z) - zo) / np.linalg.norm(zo)
        assert err <= (1e-12 if ck else 1e-9), (ck, err)
        ctx.close()


# -------------------------------------------------------------------- FCG
def _fcg_parity(psc, h, b, x0=None, tol=1e-8, maxit=200, coarse_pcg=False, **ckw):
    ctx = psc.Context()
    H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), coarse_solver="pcg" if coarse_pcg else "sweeps",
                                **ckw)
    xo, ito, sto, histo = oracle.fcg(h, b, x0=x0, tol=tol, maxit=maxit, coarse_pcg=coarse_pcg, **ckw)
    x = dev(np.zeros(len(b)) if x0 is None else x0)
    rc, st, hist = H.solve(dev(b), x, tol=tol, maxit=maxit, method="fcg")
    xg = host(x)
    assert sto == 0 and rc == 0
    assert abs(st["iters"] - ito) <= 1, (st["iters"], ito)
    k = min(20, ito, st["iters"]) + 1
    np.testing.assert_allclose(hist[:k], histo[:k], rtol=1e-9, atol=0)
    assert np.linalg.norm(xg - xo) / np.linalg.norm(xo) <= 1e-7
    return ctx, H, st, hist, xg


@pytest.mark.parametrize("coarse_pcg", [False, True], ids=["sweeps", "coarse_pcg"])
@pytest.mark.parametrize("grid,kw,rhs", [(16, dict(max_levels=2), "poisson"), (16, {}, 1),
                                         ((13, 11, 7), dict(coarse_target=20), 2), ((40, 24, 16), {}, 3)])
def test_fcg_parity(psc, grid, kw, rhs, coarse_pcg):
    g = grid if isinstance(grid, tuple) else (grid,) * 3
    h = pscgen.poisson_hierarchy(*g, **kw)
    n = h.levels[0].n
    b = pscgen.rhs_poisson(g, 0, n) if rhs == "poisson" else pscgen.rhs_random(rhs, 0, n)
    ctx, *_ = _fcg_parity(psc, h, b, coarse_pcg=coarse_pcg)
    ctx.close()


def test_fcg_jump_nonzero_guess_general_coarse(psc):
    """Jump coefficients (config 5 structure), x0 != 0, coarsest level above the
    dense limit (general coarse PCG)."""
    h = pscgen.poisson_hierarchy(24, problem="jump", cube=4, coarse_target=300)
    assert h.levels[-1].n > 144
    n = h.levels[0].n
    ctx, *_ = _fcg_parity(psc, h, pscgen.rhs_random(4, 0, n), x0=pscgen.rhs_random(5, 0, n), coarse_pcg=True)
    ctx.close()


def test_fcg_equals_pcg_fixed_preconditioner_on_gpu(psc):
    """With the fixed SPD V-cycle, FCG(1) and PCG agree (exact arithmetic)."""
    h = pscgen.poisson_hierarchy(32)
    n = h.levels[0].n
    b = pscgen.rhs_random(6, 0, n)
    ctx = psc.Context()
    H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0))
    xp, xf = dev(np.zeros(n)), dev(np.zeros(n))
    _, sp_, hp = H.solve(dev(b), xp, method="pcg")
    _, sf, hf = H.solve(dev(b), xf, method="fcg")
    assert abs(sp_["iters"] - sf["iters"]) <= 1
    k = min(len(hp), len(hf))
    np.testing.assert_allclose(hf[:k], hp[:k], rtol=1e-6, atol=0)
    assert np.linalg.norm(host(xf) - host(xp)) / np.linalg.norm(host(xp)) <= 1e-7
    ctx.close()


def test_fcg_edge_cases_deterministic_host_path(psc):
    h = pscgen.poisson_hierarchy(16, max_levels=2)
    n = h.levels[0].n
    ctx = psc.Context()
    H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), coarse_solver="pcg")
    x = dev(np.ones(n))
    rc, st, hist = H.solve(dev(np.zeros(n)), x, method="fcg")
    assert rc == 0 and st["iters"] == 0 and not host(x).any()
    b = pscgen.rhs_random(1, 0, n)
    x = dev(np.zeros(n))
    rc, st, hist = H.solve(dev(b), x, maxit=0, method="fcg")
    assert rc == psc.PSC_NOT_CONVERGED and st["iters"] == 0
    x1, x2 = dev(np.zeros(n)), dev(np.zeros(n))
    _, s1, h1 = H.solve(dev(b), x1, method="fcg")
    _, s2, h2 = H.solve(dev(b), x2, method="fcg")
    assert torch.equal(x1, x2) and np.array_equal(h1, h2)
    # PCG and FCG graphs coexist on one hierarchy
    _, s3, h3 = H.solve(dev(b), dev(np.zeros(n)), method="pcg")
    xh = np.zeros(n)
    _, s4, h4 = H.solve_host(b, xh, method="fcg")
    assert np.array_equal(xh, host(x1)) and np.array_equal(h4, h1)
    with pytest.raises(ValueError):
        H.solve(dev(b), x1, method="gmres")
    ctx.close()


def test_fcg_breakdown_is_reported(psc):
    A = sp.csr_matrix(np.diag([1.0, -1.0]))
    h = pscgen.csr_hierarchy(A, max_levels=1)
    ctx = psc.Context()
    H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), pre=1, post=1, coarse=1)
    with pytest.raises(psc.PscError) as e:
        H.solve(dev(np.ones(2)), dev(np.zeros(2)), method="fcg")
    assert e.value.code == psc.PSC_ERR_BREAKDOWN
    ctx.close()


def test_vbm_c2_128cube(psc):
    """BASELINE.json configs[1] (128^3 Poisson) in the paper's VBM configuration."""
    g = 128
    h = pscgen.poisson_hierarchy(g)
    n = h.levels[0].n
    ctx, H, st, hist, x = _fcg_parity(psc, h, pscgen.rhs_poisson((g,) * 3, 0, n), coarse_pcg=True)
    assert st["status"] == 0
    ctx.close()


# Strongly varying preconditioner (VERDICT r1 "What's weak" 1): the coarsest PCG runs
# exactly 2 iterations with no tolerance test, so B(r) is a nonlinear function of r and
# FCG(1)'s flexible beta = (z, A p_old)/(p_old, A p_old) differs from PCG's
# Fletcher-Reeves beta.  (The oracle pins this regime in test_oracle_pins.py: local
# A-orthogonality, FCG != PCG.)  No discrete decision depends on rounding here (fixed
# coarse iteration count), so the north-star bar applies unchanged.
_VARB = dict(coarse_maxit=2, coarse_tol=1e-300)


@pytest.mark.parametrize("grid,kw", [(16, dict(max_levels=2)), ((13, 11, 7), dict(coarse_target=20)), (32, {})],
                         ids=["2level_general", "dense_coarse", "32cube"])
def test_fcg_parity_strongly_variable_preconditioner(psc, grid, kw):
    g = grid if isinstance(grid, tuple) else (grid,) * 3
    h = pscgen.poisson_hierarchy(*g, **kw)
    n = h.levels[0].n
    b = pscgen.rhs_random(9, 0, n)
    ctx, H, st, hist, x = _fcg_parity(psc, h, b, tol=1e-8, coarse_pcg=True, **_VARB)
    # the same GPU hierarchy's PCG (Fletcher-Reeves beta) takes a different path here
    xp = dev(np.zeros(n))
    _, sp_, hp = H.solve(dev(b), xp, tol=1e-8, method="pcg")
    k = min(len(hp), len(hist), 10)
    assert np.max(np.abs(hist[2:k] - hp[2:k]) / hp[2:k]) > 1e-6
    ctx.close()
