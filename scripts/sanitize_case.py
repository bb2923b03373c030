"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):
the TMA ring kernels (DIA level 0), plain sliced-ELL and row-group kernels, the
ticketed reductions, one-CTA and dense coarsest solvers, the coarsest PCG, FCG, the
device set-up (psc_amg_build) and the AINV smoother.  Exit 0 when every solve matches
the oracle at the north-star bar."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2406_19754_b200 as psc  # noqa: E402
import pscgen  # noqa: E402


def check(H, h, b, **kw):
    method = kw.pop("method", "pcg")
    x = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    rc, st, hist = H.solve(torch.from_numpy(b).cuda(), x, tol=1e-8, maxit=100, method=method)
    xo, ito, sto, histo = (oracle.fcg if method == "fcg" else oracle.pcg)(h, b, tol=1e-8, maxit=100, **kw)
    k = min(20, ito, st["iters"]) + 1
    ok = rc == 0 and abs(st["iters"] - ito) <= 1 and np.allclose(hist[:k], histo[:k], rtol=1e-9, atol=0)
    print(("ok" if ok else "FAIL"), method, kw, st["iters"], ito, flush=True)
    return ok


ok = True
ctx = psc.Context()
h = pscgen.poisson_hierarchy(24, coarse_target=60)
b = pscgen.rhs_random(1, 0, h.levels[0].n)
H, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0))
ok &= check(H, h, b)
H2, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h, 0), coarse_solver="pcg")
ok &= check(H2, h, b, method="fcg", coarse_pcg=True)
h3 = pscgen.poisson_hierarchy(12, coarse_target=30)
b3 = pscgen.rhs_random(2, 0, h3.levels[0].n)
H3, *_ = psc.build_hierarchy(ctx, pscgen.rank_levels(h3, 0), pre=1, post=1, smoother="ainv", ainv_drop=0.1)
ok &= check(H3, h3, b3, pre=1, post=1, smoother="ainv", ainv_drop=0.1)
A0 = pscgen.poisson_hierarchy(16, max_levels=1).levels[0].A.to_scipy()
S = psc.AmgSetup(ctx, A0)
Ho = oracle.amg_setup(A0)
agg, root = S.aggregates(0)
ok &= bool(np.array_equal(agg, Ho.levels[0].agg))
Hd = S.hierarchy()
ok &= check(Hd, Ho, pscgen.rhs_random(3, 0, A0.shape[0]))
ctx.close()
print("ALL OK" if ok else "FAILED")
sys.exit(0 if ok else 1)
