"""Step a8 on the GPU: two ranks co-mine their root shards with the CUDA kernels and sum the
per-motif int64 counts with one all-reduce ("parallelises
over first-edge candidates"; north_star (5)).

This box has one GPU, so both ranks run on cuda:0 over gloo (the all-reduce of a CUDA tensor);
the code path per rank is the product's `parallel.comine_distributed` (shard_range ->
mayura_comine with device output -> reduce_counts), identical to the NCCL run, and the counts
are compared with the oracle element by element.  A second rank-0 call passes a side stream
(the event join before the collective).  The bench's multi-rank mode is exercised the same way
(torchrun, MAYURA_BENCH_SHARED_GPU=1)."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_name, kernel, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if kernel:
        os.environ["MAYURA_KERNEL"] = kernel
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2507_14813_b200 as M
        from paper_2507_14813_b200 import parallel
        cfg = synth.CONFIGS[cfg_name]
        src, dst, t, V = cfg.graph()
        g = M.Graph(src, dst, t, V, device=0)
        tree = M.MGTree(cfg.group(), cfg.delta)
        counts = torch.zeros(tree.n_motifs, dtype=torch.int64, device="cuda:0")
        parallel.comine_distributed(g, tree, counts)                   # current stream
        torch.cuda.synchronize()
        side = torch.cuda.Stream()
        counts2 = torch.zeros_like(counts)
        parallel.comine_distributed(g, tree, counts2, stream=side.cuda_stream)  # joined by an event
        torch.cuda.synchronize()
        rb, re_ = parallel.shard_range(g, cfg.delta, rank, world)
        mine = M.comine(g, tree, (rb, re_))
        out = dict(rank=rank, counts=counts.cpu().tolist(), counts2=counts2.cpu().tolist(), range=(rb, re_),
                   part=mine, form=M.mayura_kernel_form(g.handle))
        q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg_name,kernel", [("C2", None), ("C2", "warp"), ("C5s", None)])
def test_two_ranks_cuda_counts_all_reduced(oracle_mod, cfg_name, kernel):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg_name, kernel, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=900) for _ in range(world)], key=lambda r: r["rank"])
    for p in procs:
        p.join(900)
        assert p.exitcode == 0
    cfg = synth.CONFIGS[cfg_name]
    src, dst, t, V = cfg.graph()
    full = oracle_mod.backtrack(src, dst, t, V, cfg.group(), cfg.delta)
    for r in res:
        assert r["counts"] == full and r["counts2"] == full           # one all-reduce: whole-graph counts
    assert res[0]["range"][0] == 0 and res[0]["range"][1] == res[1]["range"][0] and res[1]["range"][1] == len(src)
    assert [a + b for a, b in zip(res[0]["part"], res[1]["part"])] == full   # shards are disjoint (R16)
    assert res[0]["part"] != full                                      # the split did split work
    if kernel:
        assert res[0]["form"] == kernel


def test_bench_two_ranks_shared_gpu(oracle_mod):
    """bench.py under torchrun with 2 ranks on cuda:0 (gloo): one JSON line from rank 0, n_gpus 2,
    counts equal the oracle's whole-graph counts."""
    env = dict(os.environ, MAYURA_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--config", "C2", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-enum",
           "--no-indep", "--no-cpu-baseline"]
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    cfg = synth.CONFIGS["C2"]
    src, dst, t, V = cfg.graph()
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "root-partition2"
    assert list(d["counts"].values()) == oracle_mod.backtrack(src, dst, t, V, cfg.group(), cfg.delta)
