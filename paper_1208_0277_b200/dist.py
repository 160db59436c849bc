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


def ring_bounds(xy, offsets):
    """Per-ring y extent [ylo, yhi) of packed rings (numpy; for the sharding
    plan only -- the device computes its own MBRs in prep)."""
    import numpy as np

    xy = np.asarray(xy).reshape(-1, 2)
    off = np.asarray(offsets, dtype=np.int64)
    n = off.shape[0] - 1
    ylo = np.full(n, np.iinfo(np.int64).max, np.int64)
    yhi = np.full(n, np.iinfo(np.int64).min, np.int64)
    nz = off[1:] > off[:-1]
    if nz.any():
        starts = off[:-1][nz]
        ylo[nz] = np.minimum.reduceat(xy[:, 1].astype(np.int64), starts)
        yhi[nz] = np.maximum.reduceat(xy[:, 1].astype(np.int64), starts)
    return ylo, yhi


def band_shards(p_ylo, p_yhi, q_ylo, q_yhi, world: int):
    """One slide over ``world`` ranks (SURVEY §8(e) "C2 at 8"; the paper's
    tile-granularity tasks): P is cut into ``world`` horizontal bands of
    equal polygon count by its MBRs' ylo (each p owned by exactly one rank);
    rank r gets every q whose y extent meets [min ylo, max yhi) of its P band.
    Any q that overlaps a p of band r meets that range, so the join of
    (P_r, Q_r) yields exactly the pairs whose p is in band r: the ranks' pair
    lists partition the slide's, and their integer sums add up to the slide's
    bit for bit.  Returns [(p_idx, q_idx)] per rank (sorted index arrays;
    empty rings -- ylo > yhi -- go with band 0 and pair with nothing)."""
    import numpy as np

    if world < 1:
        raise ValueError("world must be >= 1")
    p_ylo, p_yhi = np.asarray(p_ylo, np.int64), np.asarray(p_yhi, np.int64)
    q_ylo, q_yhi = np.asarray(q_ylo, np.int64), np.asarray(q_yhi, np.int64)
    order = np.lexsort((np.arange(p_ylo.shape[0]), p_ylo))  # by ylo, ties by index
    cuts = [(len(order) * r) // world for r in range(world + 1)]
    out = []
    for r in range(world):
        pi = np.sort(order[cuts[r] : cuts[r + 1]])
        live = pi[p_ylo[pi] < p_yhi[pi]]
        if live.size == 0:
            out.append((pi, np.zeros(0, np.int64)))
            continue
        lo, hi = int(p_ylo[live].min()), int(p_yhi[live].max())
        qi = np.nonzero((q_ylo < hi) & (q_yhi > lo))[0].astype(np.int64)
        out.append((pi, qi))
    return out


def subset_rings(xy, offsets, idx):
    """The packed rings ``idx`` of (xy, offsets), vectorised: (xy, offsets)."""
    import numpy as np

    xy = np.asarray(xy).reshape(-1, 2)
    off = np.asarray(offsets, dtype=np.int64)
    idx = np.asarray(idx, dtype=np.int64)
    lens = off[idx + 1] - off[idx]
    new_off = np.zeros(idx.shape[0] + 1, np.int64)
    np.cumsum(lens, out=new_off[1:])
    total = int(new_off[-1])
    src = np.repeat(off[idx] - new_off[:-1], lens) + np.arange(total, dtype=np.int64)
    return np.ascontiguousarray(xy[src], dtype=np.int32), new_off


REDUCE_WORDS = 26  # SCCG_REDUCE_WORDS: 10 additive fields + 16 status bits as 0/1


def pack_sums(sums):
    """Host mirror of sccg_sums_pack for CPU tensors (gloo): the int64 vector
    whose element-wise SUM over ranks unpacks to the reduced sums."""
    import torch

    st = int(sums[10])
    bits = torch.tensor([(st >> b) & 1 for b in range(REDUCE_WORDS - 10)], dtype=torch.int64)
    return torch.cat([sums[:10].to(torch.int64), bits])


def unpack_sums(vec, sums):
    """Host mirror of sccg_sums_unpack: status = OR of the ranks' status words
    (bit b set iff some rank set it), the other fields summed."""
    sums[:10] = vec[:10]
    sums[10] = sum(1 << b for b in range(REDUCE_WORDS - 10) if int(vec[10 + b]) != 0)
    return sums


def allreduce_sums(sums, group=None, force: bool = False):
    """In-place reduction of an int64 sums vector over the process group: the
    ten additive fields are summed, the status words OR-ed (NCCL has no
    bitwise-or: the status bits travel as 0/1 counts in the one SUM
    all-reduce, sccg_sums_pack / sccg_sums_unpack on the GPU).  Bit-exact for
    any rank count.  force: run the collective even at world size 1 (tests).
    Returns the tensor."""
    import torch
    import torch.distributed as dist

    if sums.dtype != torch.int64:
        raise TypeError("sums must be int64 (exact integer reduction)")
    if dist.is_available() and dist.is_initialized() and (dist.get_world_size(group) > 1 or force):
        if sums.is_cuda:
            import paper_1208_0277_b200 as sccg

            vec = sccg.sums_pack(sums)
            dist.all_reduce(vec, op=dist.ReduceOp.SUM, group=group)
            sccg.sums_unpack(vec, sums)
        else:
            vec = pack_sums(sums)
            dist.all_reduce(vec, op=dist.ReduceOp.SUM, group=group)
            unpack_sums(vec, sums)
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
