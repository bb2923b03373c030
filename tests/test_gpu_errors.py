"""Error contract of the C ABI (include/psc.h; SURVEY.md §8(b) "Conventions"):
malformed CSR, bad partitions and wrong call order return PSC_ERR_ARG /
PSC_ERR_STATE with a message, and the context stays usable afterwards.

CSR rules: row_ptr[0] = 0 and non-decreasing; columns strictly
increasing within a row; indices in [0, n_global).  Partition:
row_start[0] = 0, non-decreasing, row_start[nranks] = n_global.  Order:
descriptor -> matrices -> desc_assemble -> mat_assemble -> hier_create -> solve.
"""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import pscgen  # noqa: E402


@pytest.fixture(scope="module")
def psc():
    import paper_2406_19754_b200 as m
    return m


def _tridiag(n):
    A = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")
    A.sort_indices()
    return A


def _expect(psc, code, fn):
    with pytest.raises(psc.PscError) as e:
        fn()
    assert e.value.code == code, (e.value.code, str(e.value))
    assert str(e.value)  # a message, not an empty string
    return e.value


@pytest.mark.parametrize("case", ["rowptr0", "rowptr_decreasing", "unsorted", "duplicate", "col_negative",
                                  "col_too_big", "n_rows"])
def test_malformed_csr_is_psc_err_arg(psc, case):
    n = 8
    A = _tridiag(n)
    ptr, col, val = A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data.copy()
    if case == "rowptr0":
        ptr = ptr + 1
    elif case == "rowptr_decreasing":
        ptr = ptr.copy()
        ptr[3] = ptr[4] + 1
    elif case == "unsorted":
        col = col.copy()
        col[ptr[2]], col[ptr[2] + 1] = col[ptr[2] + 1], col[ptr[2]]
    elif case == "duplicate":
        col = col.copy()
        col[ptr[2] + 1] = col[ptr[2]]
    elif case == "col_negative":
        col = col.copy()
        col[0] = -1
    elif case == "col_too_big":
        col = col.copy()
        col[-1] = n
    ctx = psc.Context()
    d = psc.Descriptor(ctx, n, [0, n])
    if case == "n_rows":
        ptr = ptr[:-1]
    _expect(psc, psc.PSC_ERR_ARG, lambda: psc.Matrix(ctx, d, d, ptr, col, val))
    # the context survives a rejected call: a correct matrix still goes through
    m = psc.Matrix(ctx, d, d, A.indptr, A.indices, A.data)
    d.assemble()
    m.assemble()
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    m.spmv(x, y)
    assert np.array_equal(y.cpu().numpy(), A @ np.ones(n))
    ctx.close()


@pytest.mark.parametrize("row_start", [[1, 8], [0, 7], [0, 9]], ids=["start_not_0", "short", "long"])
def test_non_covering_partition_is_psc_err_arg(psc, row_start):
    ctx = psc.Context()
    _expect(psc, psc.PSC_ERR_ARG, lambda: psc.Descriptor(ctx, 8, row_start))
    ctx.close()


def test_wrong_call_order_is_psc_err_state(psc):
    n = 8
    A = _tridiag(n)
    ctx = psc.Context()
    d = psc.Descriptor(ctx, n, [0, n])
    m = psc.Matrix(ctx, d, d, A.indptr, A.indices, A.data)
    # matrix assembly before the descriptors are assembled
    _expect(psc, psc.PSC_ERR_STATE, m.assemble)
    d.assemble()
    # a matrix registered after its column descriptor was assembled
    _expect(psc, psc.PSC_ERR_STATE, lambda: psc.Matrix(ctx, d, d, A.indptr, A.indices, A.data))
    # descriptor assembled twice
    _expect(psc, psc.PSC_ERR_STATE, d.assemble)
    # SpMV on an unassembled matrix
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    _expect(psc, psc.PSC_ERR_STATE, lambda: m.spmv(x, y))
    # hierarchy over an unassembled level matrix
    _expect(psc, psc.PSC_ERR_STATE, lambda: psc.Hierarchy(ctx, [m], [], []))
    m.assemble()
    _expect(psc, psc.PSC_ERR_STATE, m.assemble)  # assembled twice
    H = psc.Hierarchy(ctx, [m], [], [], pre=1, post=1, coarse=3)
    b = torch.ones(n, dtype=torch.float64, device="cuda")
    xs = torch.zeros(n, dtype=torch.float64, device="cuda")
    rc, st, hist = H.solve(b, xs, tol=1e-30, maxit=2)
    assert rc == psc.PSC_NOT_CONVERGED and st["iters"] == 2
    ctx.close()


def test_bad_hierarchy_arguments_are_psc_err_arg(psc):
    h = pscgen.poisson_hierarchy(8, max_levels=2)
    ctx = psc.Context()
    levels = pscgen.rank_levels(h, 0)
    for kw in (dict(pre=-1), dict(coarse_solver_code=7), dict(coarse_maxit=-1), dict(coarse_tol=float("nan"))):
        code = kw.pop("coarse_solver_code", None)
        with pytest.raises((psc.PscError, KeyError, ValueError)) as e:
            if code is not None:
                psc.build_hierarchy(ctx, levels, coarse_solver=code)
            else:
                psc.build_hierarchy(ctx, levels, **kw)
        if isinstance(e.value, psc.PscError):
            assert e.value.code == psc.PSC_ERR_ARG
    # P_l given with its spaces swapped (R in P's place)
    H, descs, A, P, R = psc.build_hierarchy(ctx, levels)
    _expect(psc, psc.PSC_ERR_ARG, lambda: psc.Hierarchy(ctx, A, R, P))
    # solve arguments
    n = h.levels[0].n
    b = torch.ones(n, dtype=torch.float64, device="cuda")
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    _expect(psc, psc.PSC_ERR_ARG, lambda: H.solve(b, x, tol=-1.0))
    _expect(psc, psc.PSC_ERR_ARG, lambda: H.solve(b, x, maxit=-1))
    with pytest.raises(ValueError):
        H.solve(b, torch.zeros(n - 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(TypeError):
        H.solve(b, torch.zeros(n, dtype=torch.float32, device="cuda"))
    ctx.close()
