"""Multi-GPU driver logic for the PixelBox path.

One process per GPU (torchrun).  The pair list shards naturally: each rank owns
whole images (config 4, a study of many slide pairs) or whole tiles (the
paper's tile-granularity tasks) and runs the single-GPU path on them;
per-pair results stay on their rank.  The only exchange is one all_reduce of
the int64 ``sccg_sums`` vector (SUM).  Every field is an integer -- the J'
ratio sum is carried as exact fixed-point limbs (R12) -- so the
reduced totals, and J', are bit-identical for any number of ranks and any
sharding.  Host logic only: nothing here touches polygon data.
"""
from __future__ import annotations

import heapq


def lpt_shards(costs, world: int) -> list[list[int]]:
    """Longest-processing-time-first assignment of items (costs[i] >= 0) to
    ``world`` ranks; returns each rank's item list (sorted).  Deterministic:
    ties broken by item index, then rank index."""
    if world < 1:
        raise ValueError("world must be >= 1")
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    out: list[list[int]] = [[] for _ in range(world)]
    for i in sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i)):
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + float(costs[i]), r))
    return [sorted(s) for s in out]


def shard_for_rank(n_items: int, world: int, rank: int, costs=None) -> list[int]:
    """The items rank ``rank`` owns: LPT on ``costs`` (default: equal costs,
    i.e. round robin in index order)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    c = costs if costs is not None else [1.0] * n_items
    if len(c) != n_items:
        raise ValueError("len(costs) != n_items")
    return lpt_shards(c, world)[rank]


def allreduce_sums(sums, group=None):
    """In-place SUM of an int64 sums vector over the process group (NCCL for
    CUDA tensors, gloo for CPU tensors).  Returns the tensor."""
    import torch
    import torch.distributed as dist

    if sums.dtype != torch.int64:
        raise TypeError("sums must be int64 (exact integer reduction)")
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    return sums


def run_images(images, make_sets, device, threshold: int = 0, sums=None):
    """Run the whole path over this rank's images, accumulating into one
    device sums vector (sccg_pixelbox adds into it, P:302 batching).
    ``make_sets(image) -> (A, B)`` host PolygonSets.  Returns (sums, n_pairs)."""
    import paper_1208_0277_b200 as sccg

    sums = sums if sums is not None else sccg.new_sums(device)
    n_pairs = 0
    for img in images:
        A, B = make_sets(img)
        P = sccg.DeviceSet(*sccg.to_device(A.xy, A.offsets, device))
        Q = sccg.DeviceSet(*sccg.to_device(B.xy, B.offsets, device))
        pairs = sccg.filter_pairs(P, Q)
        sccg.pixelbox(P, Q, pairs, threshold=threshold, sums=sums, want_inter=False, want_union=False)
        n_pairs += int(pairs.shape[0])
    return sums, n_pairs
