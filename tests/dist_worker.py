"""Worker for tests/test_gpu_dist.py (launched by torchrun, one process per GPU).

Rank 0 generates the global hierarchy for the rank-box grid, every rank maps its
rows, the distributed CUDA path (NCCL halo exchange, replicated coarsest level)
runs SpMV / V-cycle / PCG, and rank 0 compares with the CPU oracle on the global
hierarchy.  Prints one JSON line on rank 0; exit code 0 on success.
"""
import json
import os
import sys
import tempfile

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _util import ew_err  # noqa: E402


def main():
    grid = tuple(int(v) for v in os.environ.get("PSC_TEST_GRID", "32,32,64").split(","))
    procs = tuple(int(v) for v in os.environ.get("PSC_TEST_PROCS", "1,1,2").split(","))
    problem = os.environ.get("PSC_TEST_PROBLEM", "poisson")
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    shm = os.environ.get("PSC_TEST_SHM") or tempfile.gettempdir()
    ok, out = check(grid, procs, problem, shm, rank, world, local, full=True)
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


def check(grid, procs, problem, shm, rank, world, local, full=True):
    """The distributed CUDA path against the oracle on the global hierarchy (rank 0
    compares).  Needs an initialised torch.distributed process group; returns
    (ok on every rank, result dict on rank 0).  full=False: SpMV, V-cycle and PCG
    only (no VBM / variable-cycle legs)."""
    import bench
    import paper_2406_19754_b200 as psc
    import pscgen

    d = os.path.join(shm, f"psc_dist_{grid[0]}x{grid[1]}x{grid[2]}_{procs}_{problem}".replace(" ", ""))
    h = None
    if rank == 0:
        h = pscgen.poisson_hierarchy(*grid, procs=procs, problem=problem, cube=8, coarse_target=60)
        bench.save_rank_levels(d, h, world)
    dist.barrier()
    levels, meta = bench.load_rank_levels(d, rank)
    obj = [psc.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = psc.Context(rank=rank, nranks=world, device=local, unique_id=obj[0])
    H, descs, A, P, R = psc.build_hierarchy(ctx, levels)
    rs = levels[0]["row_start"]
    r0, r1 = int(rs[rank]), int(rs[rank + 1])
    N = int(levels[0]["n_global"])
    out = {}
    # SpMV of every level matrix
    spmv = []
    for l in range(meta["nlevels"]):
        mats = [("A", A[l], l, l)] + ([("P", P[l], l, l + 1), ("R", R[l], l + 1, l)] if l < meta["nlevels"] - 1 else [])
        for name, M, rsp, csp in mats:
            crs = levels[csp]["row_start"]
            rrs = levels[rsp]["row_start"]
            xg = pscgen.rhs_random(31 + l, 0, int(levels[csp]["n_global"]))
            x = torch.from_numpy(xg[int(crs[rank]):int(crs[rank + 1])].copy()).cuda()
            y = torch.zeros(int(rrs[rank + 1] - rrs[rank]), dtype=torch.float64, device="cuda")
            M.spmv(x, y)
            spmv.append((name, l, y.cpu().numpy()))
    allspmv = [None] * world
    dist.all_gather_object(allspmv, spmv)
    # V-cycle and PCG on the global RHS
    b = pscgen.rhs_random(7, 0, N)
    z = torch.zeros(r1 - r0, dtype=torch.float64, device="cuda")
    H.vcycle(torch.from_numpy(b[r0:r1].copy()).cuda(), z)
    x = torch.zeros(r1 - r0, dtype=torch.float64, device="cuda")
    rc, st, hist = H.solve(torch.from_numpy(b[r0:r1].copy()).cuda(), x, tol=1e-8, maxit=200)
    parts = [None] * world
    dist.all_gather_object(parts, (z.cpu().numpy(), x.cpu().numpy(), rc, st["iters"], hist))
    parts2 = parts3 = None
    if full:
        # the paper's VBM solve (NEXT-2): coarsest PCG(<= 40) with l1-Jacobi + FCG, on
        # the same matrices (a general-form coarse PCG with all-gathers when the
        # coarsest level is distributed, PSC_REPL_ROWS=0)
        H2 = psc.Hierarchy(ctx, A, P, R, coarse_solver="pcg")
        z2 = torch.zeros(r1 - r0, dtype=torch.float64, device="cuda")
        H2.vcycle(torch.from_numpy(b[r0:r1].copy()).cuda(), z2)
        x2 = torch.zeros(r1 - r0, dtype=torch.float64, device="cuda")
        rc2, st2, hist2 = H2.solve(torch.from_numpy(b[r0:r1].copy()).cuda(), x2, tol=1e-8, maxit=200, method="fcg")
        parts2 = [None] * world
        dist.all_gather_object(parts2, (z2.cpu().numpy(), x2.cpu().numpy(), rc2, st2["iters"], hist2))
        H2.close()
        # the variable V-cycle (P:330 footnote): 2 sweeps at level 0, doubled per level,
        # through the distributed levels and the replicated suffix alike
        H3 = psc.Hierarchy(ctx, A, P, R, pre=2, post=2, variable_v=True)
        z3 = torch.zeros(r1 - r0, dtype=torch.float64, device="cuda")
        H3.vcycle(torch.from_numpy(b[r0:r1].copy()).cuda(), z3)
        parts3 = [None] * world
        dist.all_gather_object(parts3, z3.cpu().numpy())
        H3.close()
        # NEXT-4: the AINV smoother, block-Jacobi across ranks on the distributed levels
        # (each rank factors its diagonal block), whole-matrix factors on the
        # replicated suffix
        H4 = psc.Hierarchy(ctx, A, P, R, pre=1, post=1, smoother="ainv", ainv_drop=0.1)
        z4 = torch.zeros(r1 - r0, dtype=torch.float64, device="cuda")
        H4.vcycle(torch.from_numpy(b[r0:r1].copy()).cuda(), z4)
        x4 = torch.zeros(r1 - r0, dtype=torch.float64, device="cuda")
        rc4, st4, hist4 = H4.solve(torch.from_numpy(b[r0:r1].copy()).cuda(), x4, tol=1e-8, maxit=200)
        parts4 = [None] * world
        dist.all_gather_object(parts4, (z4.cpu().numpy(), x4.cpu().numpy(), rc4, st4["iters"], hist4))
        H4.close()
    ok = True
    if rank == 0:
        import oracle
        for k, (name, l, _) in enumerate(spmv):
            M = getattr(h.levels[l], name)
            rsp = l if name != "R" else l + 1
            csp = l if name != "P" else l + 1
            xg = pscgen.rhs_random(31 + l, 0, M.shape[1])
            ref = oracle.spmv(M, xg)
            got = np.concatenate([allspmv[p][k][2] for p in range(world)])
            scale = abs(M.to_scipy()) @ np.abs(xg)
            e = float((np.abs(got - ref) / (scale + 1e-300)).max())
            out[f"spmv_{name}{l}"] = e
            ok &= e <= 1e-14
        zg = np.concatenate([p[0] for p in parts])
        zo = oracle.vcycle(h, b)
        out["vcycle_rel"] = float(ew_err(zg, zo))
        ok &= out["vcycle_rel"] <= 1e-12
        xg = np.concatenate([p[1] for p in parts])
        xo, ito, sto, histo = oracle.pcg(h, b, tol=1e-8, maxit=200)
        its = {p[3] for p in parts}
        out.update(iters_gpu=sorted(its), iters_oracle=ito, rc=[p[2] for p in parts])
        k = min(20, ito, parts[0][3]) + 1
        out["hist_rel"] = float(np.max(np.abs(parts[0][4][:k] - histo[:k]) / histo[:k]))
        out["x_rel"] = float(np.linalg.norm(xg - xo) / np.linalg.norm(xo))
        same_hist = all(np.array_equal(parts[0][4], p[4]) for p in parts)
        out["hist_identical_across_ranks"] = same_hist
        ok &= (len(its) == 1 and abs(parts[0][3] - ito) <= 1 and all(p[2] == 0 for p in parts)
               and out["hist_rel"] <= 1e-9 and out["x_rel"] <= 1e-7 and same_hist)
        if full:
            zg2 = np.concatenate([p[0] for p in parts2])
            zo2 = oracle.vcycle(h, b, coarse_pcg=True)
            out["vbm_vcycle_rel"] = float(ew_err(zg2, zo2))
            xg2 = np.concatenate([p[1] for p in parts2])
            xo2, ito2, sto2, histo2 = oracle.fcg(h, b, tol=1e-8, maxit=200, coarse_pcg=True)
            its2 = {p[3] for p in parts2}
            k2 = min(20, ito2, parts2[0][3]) + 1
            out.update(vbm_iters_gpu=sorted(its2), vbm_iters_oracle=ito2,
                       vbm_hist_rel=float(np.max(np.abs(parts2[0][4][:k2] - histo2[:k2]) / histo2[:k2])),
                       vbm_x_rel=float(np.linalg.norm(xg2 - xo2) / np.linalg.norm(xo2)))
            ok &= (out["vbm_vcycle_rel"] <= 1e-9 and len(its2) == 1 and abs(parts2[0][3] - ito2) <= 1
                   and all(p[2] == 0 for p in parts2) and out["vbm_hist_rel"] <= 1e-9 and out["vbm_x_rel"] <= 1e-7
                   and all(np.array_equal(parts2[0][4], p[4]) for p in parts2))
            # AINV blocks as the library forms them: the rank row blocks on distributed
            # levels, the whole matrix from the first replicated level (hier.cu
            # replica_first: first level >= 1 with at most PSC_REPL_ROWS global rows)
            lim = int(os.environ.get("PSC_REPL_ROWS", "50000"))
            L = meta["nlevels"]
            first = next((l for l in range(1, L) if lim and int(levels[l]["n_global"]) <= lim), L)
            blocks = [np.asarray(levels[l]["row_start"], np.int64) if l < first and world > 1 else None
                      for l in range(L)]
            akw = dict(pre=1, post=1, smoother="ainv", ainv_drop=0.1, ainv_blocks=blocks)
            zg4 = np.concatenate([p[0] for p in parts4])
            out["ainv_vcycle_rel"] = float(ew_err(zg4, oracle.vcycle(h, b, **akw)))
            xo4, ito4, sto4, histo4 = oracle.pcg(h, b, tol=1e-8, maxit=200, **akw)
            xg4 = np.concatenate([p[1] for p in parts4])
            k4 = min(20, ito4, parts4[0][3]) + 1
            out.update(ainv_first_replicated=first, ainv_iters_gpu=sorted({p[3] for p in parts4}),
                       ainv_iters_oracle=ito4,
                       ainv_hist_rel=float(np.max(np.abs(parts4[0][4][:k4] - histo4[:k4]) / histo4[:k4])),
                       ainv_x_rel=float(np.linalg.norm(xg4 - xo4) / np.linalg.norm(xo4)))
            ok &= (out["ainv_vcycle_rel"] <= 1e-12 and len({p[3] for p in parts4}) == 1
                   and abs(parts4[0][3] - ito4) <= 1 and all(p[2] == 0 for p in parts4)
                   and out["ainv_hist_rel"] <= 1e-9 and out["ainv_x_rel"] <= 1e-7)
            zg3 = np.concatenate(parts3)
            zo3 = oracle.vcycle(h, b, 2, 2, 30, variable_v=True)
            out["varv_vcycle_rel"] = float(ew_err(zg3, zo3))
            ok &= out["varv_vcycle_rel"] <= 1e-12
        out["ok"] = bool(ok)
    flag = [ok]
    dist.broadcast_object_list(flag, src=0)
    H.close()
    ctx.close()
    return bool(flag[0]), out


if __name__ == "__main__":
    main()
