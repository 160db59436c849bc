"""Multi-process host logic of the sharded path (``-m "not gpu"``): gloo,
world size 2, on CPU.  Each rank computes its images' integer sums (the
``sccg_sums`` layout; here from the oracle, since there is no GPU), the sums are
all-reduced, and J' from the reduced integers (through the library's
``sccg_jaccard``) must equal the single-process value over all images,
bit for bit, for any sharding."""
import os
import socket
from fractions import Fraction

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1208_0277_b200 import dist as sdist


def test_lpt_shards_cover_each_item_once():
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 8):
        costs = rng.integers(1, 100, 100).tolist()
        shards = sdist.lpt_shards(costs, world)
        flat = sorted(i for s in shards for i in s)
        assert flat == list(range(100))
        loads = [sum(costs[i] for i in s) for s in shards]
        assert max(loads) - min(loads) <= max(costs)  # LPT bound
        assert shards == sdist.lpt_shards(costs, world)  # deterministic
    assert sdist.shard_for_rank(5, 2, 0) + sdist.shard_for_rank(5, 2, 1) != []
    with pytest.raises(ValueError):
        sdist.shard_for_rank(5, 2, 2)


def image_sums(image):
    """Integer sums of one synthetic image (C1 tile, seed per image) from the oracle."""
    import oracle
    import synth

    A, B = synth.generate("tile", image=image)
    A, B = A.subset(range(0, A.n, 5)), B.subset(range(0, B.n, 5))
    pairs = oracle.join(A, B)
    inter, uni = oracle.pair_areas(A, B, pairs, threads=1)
    s = oracle.sums(A, B, pairs, inter, uni)
    units = sum(int(Fraction(int(i) / int(u)) * (1 << 116)) for i, u in zip(inter, uni) if i)
    limbs = [(units >> (30 * k)) & ((1 << 30) - 1) for k in range(3)] + [units >> 90]
    vec = [s["n_pairs"], s["n_nonzero"], s["sum_inter"], s["sum_union"], s["sum_area_p"], s["sum_area_q"]] + limbs + [0]
    return vec, list(zip(inter.tolist(), uni.tolist()))


def _worker(rank, world, port, images, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = sdist.shard_for_rank(len(images), world, rank, costs=[1 + (i % 3) for i in range(len(images))])
    total = torch.zeros(11, dtype=torch.int64)
    for i in mine:
        v, _ = image_sums(images[i])
        total += torch.tensor(v, dtype=torch.int64)
    sdist.allreduce_sums(total)
    out[rank] = total.tolist()
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ranks_allreduce_is_exact(world):
    import oracle
    import paper_1208_0277_b200 as sccg

    images = [0, 1, 2, 3, 4]
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, images, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    assert all(out[r] == out[0] for r in range(world))
    # single-process reference over all images
    ref = [0] * 11
    allpairs = []
    for img in images:
        v, iu = image_sums(img)
        ref = [a + b for a, b in zip(ref, v)]
        allpairs += iu
    assert out[0] == ref
    j, _ = sccg.jaccard(out[0])
    ex = oracle.jaccard_exact([i for i, _ in allpairs], [u for _, u in allpairs])
    assert abs(j - float(ex)) <= 1e-12 * float(ex)


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_band_shards_partition_the_slide_pairs(world):
    """One slide over `world` ranks: P cut into y bands, Q_r =
    the q that meet band r's y range.  The ranks' joins, mapped back to global
    indices, partition the single-process join (each pair on exactly one rank)
    and the ranks' integer sums add up to the slide's (oracle, CPU)."""
    import oracle
    import synth

    A, B = synth.generate("tile", image=3)
    pylo, pyhi = sdist.ring_bounds(A.xy, A.offsets)
    qylo, qyhi = sdist.ring_bounds(B.xy, B.offsets)
    want = oracle.join(A, B)
    shards = sdist.band_shards(pylo, pyhi, qylo, qyhi, world)
    assert sorted(np.concatenate([pi for pi, _ in shards]).tolist()) == list(range(A.n))
    got, tot = [], None
    for pi, qi in shards:
        xa, oa = sdist.subset_rings(A.xy, A.offsets, pi)
        xb, ob = sdist.subset_rings(B.xy, B.offsets, qi)
        Ar, Br = synth.PolygonSet(xa, oa), synth.PolygonSet(xb, ob)
        pr = oracle.join(Ar, Br)
        if len(pr):
            got.append(np.stack([pi[pr[:, 0]], qi[pr[:, 1]]], 1))
            inter, uni = oracle.pair_areas(Ar, Br, pr, threads=1)
            s = oracle.sums(Ar, Br, pr, inter, uni)
            tot = s if tot is None else {k: tot[k] + s[k] for k in s}
    got = np.concatenate(got) if got else np.zeros((0, 2), np.int64)
    got = got[np.lexsort((got[:, 1], got[:, 0]))]
    assert got.shape == want.shape and (got == want).all()  # each pair exactly once
    inter, uni = oracle.pair_areas(A, B, want, threads=1)
    full = oracle.sums(A, B, want, inter, uni)
    assert {k: int(v) for k, v in tot.items()} == {k: int(v) for k, v in full.items()}


def test_band_shards_degenerate():
    # empty / zero-height rings belong to a band but pair with nothing; more ranks than polygons
    s = sdist.band_shards([5, 9, 0], [5, 12, 4], [0, 10], [3, 11], 5)
    assert sorted(np.concatenate([p for p, _ in s]).tolist()) == [0, 1, 2]
    for pi, qi in s:
        assert set(pi.tolist()) <= {0, 1, 2}
    with pytest.raises(ValueError):
        sdist.band_shards([0], [1], [0], [1], 0)


def _status_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r: additive fields r + 1, status bits: every rank sets ARG (bit 0); rank 0 STACK (bit 3), rank 1
    # CAPACITY (bit 4) -- a plain SUM would carry 1 + 1 into bit 1 and lose bit 0
    st = 1 | (8 if rank == 0 else 0) | (16 if rank == 1 else 0)
    v = torch.tensor([rank + 1] * 10 + [st], dtype=torch.int64)
    sdist.allreduce_sums(v)
    out[rank] = v.tolist()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(120)
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_allreduce_ors_status_bits(world):
    """the status word is an OR of SCCG_STATUS_* bits, never summed
    across ranks (pack: bits as 0/1 counts, one SUM, unpack: count > 0)."""
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_status_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(100)
        assert p.exitcode == 0
    want = [sum(range(1, world + 1))] * 10 + [1 | 8 | 16]
    for r in range(world):
        assert out[r] == want


def test_pack_unpack_host_mirror():
    v = torch.tensor(list(range(10)) + [0b10110], dtype=torch.int64)
    vec = sdist.pack_sums(v)
    assert vec.shape[0] == sdist.REDUCE_WORDS and vec[:10].tolist() == list(range(10))
    assert vec[10:].tolist() == [0, 1, 1, 0, 1] + [0] * 11
    back = sdist.unpack_sums(vec * 3, torch.zeros(11, dtype=torch.int64))  # three ranks with the same bits
    assert back[:10].tolist() == [3 * i for i in range(10)] and int(back[10]) == 0b10110


def test_study_instancing_preserves_every_pair():
    """configs[3] instancing (bench.study_images / instance_xy): each image is
    its base under one of the 8 lattice symmetries plus a translation; the
    oracle's MBR pair list and every pair's (I, U) must be the base's, so the
    study's expected sums are sums of the bases' (the bench self-check)."""
    import sys

    import oracle
    import synth

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    plan = bench.study_images(16, 2)
    assert sorted({p["sym"] for p in plan}) == list(range(8))
    assert len({(p["dx"], p["dy"]) for p in plan}) == 16
    A, B = synth.generate("tile", image=3)
    A, B = A.subset(range(0, A.n, 3)), B.subset(range(0, B.n, 3))
    base_pairs = oracle.join(A, B)
    bi, bu = oracle.pair_areas(A, B, base_pairs)
    for im in plan[:8]:
        xa = bench.instance_xy(torch.from_numpy(A.xy), im["sym"], im["dx"], im["dy"]).numpy()
        xb = bench.instance_xy(torch.from_numpy(B.xy), im["sym"], im["dx"], im["dy"]).numpy()
        A2, B2 = synth.PolygonSet(xa, A.offsets), synth.PolygonSet(xb, B.offsets)
        pairs = oracle.join(A2, B2)
        assert np.array_equal(pairs, base_pairs)
        i2, u2 = oracle.pair_areas(A2, B2, pairs)
        assert np.array_equal(i2, bi) and np.array_equal(u2, bu)
        assert (xa.min() > 0) and (xa.max() < 2**30)
