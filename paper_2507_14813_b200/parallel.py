"""Multi-GPU co-mining: root-edge sharding + one all-reduce.

Every match has exactly one root (its first edge), so counts are additive over any
partition of the root ids (reading R16; the paper parallelises over
first-edge candidates).  Each rank holds the full graph, co-mines a
contiguous, work-balanced range of roots (``mayura_partition_roots``), and the
k-entry int64 count vector is summed by ONE ``all_reduce`` (``north_star`` (5)).
Integer sums are exact in any reduction order.

One process per GPU; ``torch.distributed`` (NCCL on GPUs) is plumbing only -- the
search runs in libmayura.so's kernels.  The host-side pieces (``shard_range``,
``reduce_counts``) are backend-agnostic so the gloo tests can exercise them on CPU.
"""
from __future__ import annotations

from typing import List, Optional, Tuple

from .mayura import Graph, MGTree, mayura_comine


def shard_range(graph: Graph, delta: int, rank: int, world: int) -> Tuple[int, int]:
    """This rank's root range [begin, end): the rank-th part of the work-balanced split
    (identical on every rank: host-deterministic from the graph and delta)."""
    if not 0 <= rank < world:
        raise ValueError("rank %d outside world %d" % (rank, world))
    bounds = graph.partition(delta, world)
    return bounds[rank], bounds[rank + 1]


def reduce_counts(counts, group=None):
    """Sum a per-rank int64 count tensor over all ranks in place (one all_reduce)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def comine_distributed(graph: Graph, tree: MGTree, counts_out, stream: Optional[int] = None,
                       group=None, rank: Optional[int] = None, world: Optional[int] = None):
    """Co-mine this rank's share of the roots into the device tensor ``counts_out``
    (k int64 on the graph's GPU), then all-reduce it.  ``stream`` (a cudaStream_t as int)
    defaults to torch's current stream on the tensor's device; a different stream is joined
    to the current one with an event before the collective.  Returns ``counts_out``, which
    holds the whole-graph counts on every rank once the stream completes."""
    import torch.distributed as dist
    if rank is None or world is None:
        if dist.is_available() and dist.is_initialized():
            rank, world = dist.get_rank(group), dist.get_world_size(group)
        else:
            rank, world = 0, 1
    rb, re_ = shard_range(graph, tree.delta, rank, world)
    import torch
    dev = counts_out.device if getattr(counts_out, "is_cuda", False) else None
    cur = torch.cuda.current_stream(dev) if dev is not None else None
    if stream is None and cur is not None:
        stream = cur.cuda_stream          # not the legacy default stream: all_reduce follows `cur`
    mayura_comine(graph.handle, tree.handle, rb, re_, stream, counts_out)
    if cur is not None and stream != cur.cuda_stream:
        # the collective is ordered after torch's current stream only: make it wait for the
        # mining kernels enqueued on the caller's stream
        ev = torch.cuda.Event()
        ev.record(torch.cuda.ExternalStream(stream, device=dev))
        cur.wait_event(ev)
    return reduce_counts(counts_out, group)


def split_points(graph: Graph, delta: int, world: int) -> List[int]:
    return graph.partition(delta, world)
