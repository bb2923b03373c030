"""Halo-exchange microbenchmark (torchrun, one process per GPU): the weak-scaling
256^3-per-GPU hierarchy, psc_hier_exchange_bench at every distributed level (eager
back-to-back exchanges, device time per exchange), max over ranks.  The exchange
kernel's knobs come from the environment (PSC_P2P_FENCE, PSC_P2P_BX, PSC_P2P_PER_CTA)."""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2406_19754_b200 as psc  # noqa: E402
import pscgen  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    g = int(os.environ.get("XB_GRID", "256"))
    px, py, pz = bench.procs_for(world)
    grid = (g * px, g * py, g * pz)
    shm = f"/dev/shm/psc_xb_{grid[0]}x{grid[1]}x{grid[2]}_{px}{py}{pz}"
    if rank == 0 and not os.path.exists(os.path.join(shm, "meta.json")):
        bench.save_rank_levels(shm, pscgen.poisson_hierarchy(*grid, procs=(px, py, pz)), world)
    dist.barrier()
    levels, meta = bench.load_rank_levels(shm, rank)
    obj = [psc.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = psc.Context(rank=rank, nranks=world, device=local, unique_id=obj[0])
    H, *_ = psc.build_hierarchy(ctx, levels)
    out = {}
    for l in range(meta["nlevels"]):
        try:
            us = H.exchange_bench(l, 500)
        except psc.PscError as e:
            us = None
        t = [None] * world
        dist.all_gather_object(t, us)
        out[l] = None if any(v is None for v in t) else round(max(t), 2)
    if rank == 0:
        print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("PSC_P2P")}, "us": out}))
    H.close()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
