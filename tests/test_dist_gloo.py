"""N > 1 host logic on CPU: two processes (torch.distributed, gloo, 127.0.0.1).

* bench.py's multi-rank input plumbing: rank 0 writes the per-rank hierarchy pieces,
  every rank maps its own rows; they must equal the rows of the global hierarchy.
* the descriptor-assembly arithmetic of libpsc (host-only psc_halo_plan /
  psc_send_plan, the same code psc_desc_assemble runs before its NCCL exchange):
  after exchanging requests with gloo, what each owner would send must be exactly
  what each requester's halo slots expect, for every level index space.
* SPEC S:160 example: 1D Laplacian N=10 split 5/5 -> halos {5} and {4}.
"""
import os
import socket
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _level_refs(levels, l):
    """Global columns referenced in index space l by this rank: A_l, R_l rows, and P_{l-1} rows."""
    refs = [levels[l]["A"][1]]
    if "R" in levels[l]:
        refs.append(levels[l]["R"][1])
    if l > 0:
        refs.append(levels[l - 1]["P"][1])
    return np.concatenate([np.asarray(r) for r in refs])


def _worker(rank, world, port, shm, grid, procs, out_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import paper_2406_19754_b200 as psc
        import pscgen
        h = pscgen.poisson_hierarchy(*grid, procs=procs, coarse_target=10)
        if rank == 0:
            bench.save_rank_levels(shm, h, world)
        dist.barrier()
        levels, meta = bench.load_rank_levels(shm, rank)
        ref = pscgen.rank_levels(h, rank)
        assert meta["nlevels"] == h.nlevels
        for l in range(h.nlevels):
            for k in ("A", "P", "R"):
                if k in ref[l]:
                    for a, b in zip(levels[l][k], ref[l][k]):
                        assert np.array_equal(np.asarray(a), np.asarray(b)), (l, k)
        # halo plan + exchange per level index space
        for l in range(h.nlevels):
            rs = np.asarray(levels[l]["row_start"], np.int64)
            halo, rcount = psc.halo_plan(world, rank, rs, _level_refs(levels, l))
            own = (rs[rank], rs[rank + 1])
            assert np.all((halo < own[0]) | (halo >= own[1])) and np.all(np.diff(halo) > 0)
            allh = [None] * world
            dist.all_gather_object(allh, (halo, rcount))
            # requests addressed to me, in peer order
            req = [allh[p][0][(allh[p][0] >= own[0]) & (allh[p][0] < own[1])] for p in range(world)]
            send_count = np.array([len(q) for q in req], np.int64)
            assert np.array_equal(send_count, np.array([allh[p][1][rank] for p in range(world)]))
            idx = psc.send_plan(world, rank, rs, send_count, np.concatenate(req) if req else np.zeros(0))
            # "send" x = global index of my owned entries; peers check their halo slots
            x_own = np.arange(own[0], own[1], dtype=np.int64)
            sent = np.split(x_own[idx], np.cumsum(send_count)[:-1]) if len(send_count) > 1 else [x_own[idx]]
            recv = [None] * world
            dist.all_gather_object(recv, sent)
            got = np.concatenate([recv[p][rank] for p in range(world)]) if world > 1 else np.zeros(0)
            assert np.array_equal(got, halo), (l, rank)
        out_q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        out_q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("grid,procs", [((8, 8, 8), (1, 1, 2)), ((12, 8, 8), (2, 1, 1)), ((8, 8, 8), (1, 2, 2)),
                                        ((8, 8, 8), (2, 2, 2))],
                         ids=["2ranks_z", "2ranks_x", "4ranks", "8ranks_2x2x2"])
def test_multi_rank_gloo_halo_plan_and_bench_inputs(grid, procs):
    """2, 4 and 8 processes (the 8-GPU layout 2 x 2 x 2 of bench.py, where every level-0
    rank box has 3 neighbours and an x split)."""
    world = procs[0] * procs[1] * procs[2]
    import bench
    assert bench.procs_for(world) == procs or world == 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as shm:
        port = _free_port()
        ps = [ctx.Process(target=_worker, args=(r, world, port, shm, grid, procs, q)) for r in range(world)]
        for p in ps:
            p.start()
        for p in ps:
            p.join(timeout=240)
        res = dict(q.get(timeout=5) for _ in range(world))
    assert res == {r: "ok" for r in range(world)}, res


def test_spec_descriptor_example_1d_laplacian():
    """1D Laplacian N=10, 2 shards 5/5 -> shard 0 halo {5}, shard 1 halo {4}."""
    import paper_2406_19754_b200 as psc
    rs = [0, 5, 10]
    cols0 = [c for i in range(5) for c in (i - 1, i, i + 1) if 0 <= c < 10]
    cols1 = [c for i in range(5, 10) for c in (i - 1, i, i + 1) if 0 <= c < 10]
    h0, rc0 = psc.halo_plan(2, 0, rs, cols0)
    h1, rc1 = psc.halo_plan(2, 1, rs, cols1)
    assert h0.tolist() == [5] and h1.tolist() == [4]
    assert rc0.tolist() == [0, 1] and rc1.tolist() == [1, 0]
    # one shard: empty halo
    h, rc = psc.halo_plan(1, 0, [0, 10], cols0 + cols1)
    assert len(h) == 0 and rc.tolist() == [0]
    # interface node: local index >= |owned| -> halo is ordered after the owned block
    idx = psc.send_plan(2, 1, rs, np.array([1, 0]), np.array([5]))
    assert idx.tolist() == [0]
    with pytest.raises(psc.PscError):
        psc.send_plan(2, 1, rs, np.array([1, 0]), np.array([3]))  # not owned by rank 1
