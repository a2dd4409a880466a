"""Multi-rank host logic on CPU: world_size 2 over gloo.

The GPU path per rank is `mayura_comine` on `shard_range(...)`; here (no GPU) each
rank counts its range with the oracle (test infrastructure) and the counts are summed
by the package's `reduce_counts` all-reduce.  Checks: the split is identical on every
rank and covers [0, E) exactly; range counts reduced over ranks equal the whole-graph
counts (R16 additivity); the reduction of int64 counts is exact."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import __graft_entry__
        __graft_entry__._builder().build()
        import oracle
        import paper_2507_14813_b200 as M
        from paper_2507_14813_b200 import parallel
        cfg = synth.CONFIGS[cfg_name]
        src, dst, t, V = cfg.graph()
        g = M.Graph(src, dst, t, V, device=-1)                   # host-only: partitioning works
        rb, re_ = parallel.shard_range(g, cfg.delta, rank, world)
        bounds = torch.tensor([rb, re_], dtype=torch.int64)
        allb = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allb, bounds)
        part = oracle.backtrack(src, dst, t, V, cfg.group(), cfg.delta, root_range=(rb, re_), threads=2)
        counts = torch.tensor(part, dtype=torch.int64)
        parallel.reduce_counts(counts)
        big = torch.tensor([(1 << 61) + rank], dtype=torch.int64)   # exact int64 reduction
        parallel.reduce_counts(big)
        if rank == 0:
            full = oracle.backtrack(src, dst, t, V, cfg.group(), cfg.delta, threads=2)
            q.put(dict(bounds=[b.tolist() for b in allb], counts=counts.tolist(), full=full,
                       E=len(src), big=int(big.item()), part0=part))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_shard_and_reduce(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, "C1", q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    b = res["bounds"]
    assert b[0][0] == 0 and b[-1][1] == res["E"]
    assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))     # contiguous, disjoint
    assert all(x[1] - x[0] > 0.2 * res["E"] / world for x in b)      # balanced (not degenerate)
    assert res["counts"] == res["full"]                                # additivity + all_reduce
    assert res["part0"] != res["full"]                                 # the split did split work
    assert res["big"] == 2 * (1 << 61) + sum(range(world))
