"""torchrun worker: per-level halo exchange latency (psc_hier_exchange_bench)."""
import json, os, sys, tempfile
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_2406_19754_b200 as psc, pscgen
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
g = int(os.environ.get("EXB_GRID", "128"))
procs = bench.procs_for(world)
d = f"/dev/shm/exb_{g}_{world}"
if rank == 0 and not os.path.exists(os.path.join(d, "meta.json")):
    bench.save_rank_levels(d, pscgen.poisson_hierarchy(g * procs[0], g * procs[1], g * procs[2], procs=procs), world)
dist.barrier()
levels, meta = bench.load_rank_levels(d, rank)
obj = [psc.get_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
ctx = psc.Context(rank=rank, nranks=world, device=rank, unique_id=obj[0])
H, *_ = psc.build_hierarchy(ctx, levels)
res = [round(H.exchange_bench(l, 200), 2) for l in range(meta["nlevels"] - 1)]
if rank == 0:
    print(json.dumps({"env": os.environ.get("PSC_DEBUG_EX", "") + "|" + os.environ.get("PSC_NO_P2P", ""), "us_per_level": res}), flush=True)
ctx.close()
dist.destroy_process_group()
