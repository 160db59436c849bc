"""CPU pre-screen of the kernel's bit-parallel formulas (tests/kernel_model.py)
against the oracle: pixel-row masks, edge-parallel Lemma-1 classification and
the sampling-box loop must reproduce the oracle's |p n q| exactly for every
threshold (SPEC S:189 oracle equivalence for all T)."""
import numpy as np

import kernel_model as km
import oracle
import synth
from synth import combs


def test_model_pixelization_matches_oracle(tile_sets):
    a, b = tile_sets
    pairs = oracle.join(a, b)[:200]
    inter, _ = oracle.pair_areas(a, b, pairs)
    for k, (p, q) in enumerate(pairs):
        assert km.pair_intersection(a.ring(int(p)), b.ring(int(q)), T=1 << 40) == inter[k]


def test_model_sampling_boxes_match_oracle_all_T(tile_sets):
    a, b = tile_sets
    pairs = oracle.join(a, b)[:60]
    inter, _ = oracle.pair_areas(a, b, pairs)
    for T in (2, 7, 33, 100, 512):
        for k, (p, q) in enumerate(pairs):
            assert km.pair_intersection(a.ring(int(p)), b.ring(int(q)), T=T) == inter[k], (T, k)


def test_model_large_shapes():
    A, B = synth.generate("skewed", width=4096, height=4096)
    pairs = oracle.join(A, B)
    ma, mb = np.diff(A.offsets), np.diff(B.offsets)
    big = [k for k, (p, q) in enumerate(pairs) if ma[p] > 200 and mb[q] > 200][:4]
    big += [k for k, (p, q) in enumerate(pairs) if ma[p] > 200 and mb[q] < 100][:4]
    pairs = pairs[big]
    inter, _ = oracle.pair_areas(A, B, pairs)
    for T in (64, 2048):
        stats = {}
        for k, (p, q) in enumerate(pairs):
            assert km.pair_intersection(A.ring(int(p)), B.ring(int(q)), T=T, stats=stats) == inter[k]
        assert stats.get("splits", 0) > 0
    C, D, (RA, RB) = combs.generate(n_pairs=3, want_rects=True, max_vertices=600)
    for k in range(3):
        want = combs.rect_decomp_intersection(RA[k], RB[k])
        assert km.pair_intersection(C.ring(k), D.ring(k), T=256) == want


def test_model_region_items_local_culling():
    """Large-pair path: region items + local lists + left-column/bottom-row
    parity paths reproduce the oracle for every T and region size."""
    A, B = synth.generate("skewed", width=4096, height=4096)
    pairs = oracle.join(A, B)
    ma, mb = np.diff(A.offsets), np.diff(B.offsets)
    sel = [k for k, (p, q) in enumerate(pairs) if ma[p] > 200 and mb[q] > 200][:3]
    sel += [k for k, (p, q) in enumerate(pairs) if ma[p] > 200 and mb[q] < 100][:3]
    sel += list(range(0, len(pairs), max(1, len(pairs) // 20)))[:20]
    pairs = pairs[sel]
    inter, _ = oracle.pair_areas(A, B, pairs)
    for T, region in ((64, 37), (2048, 128), (300, 1000)):
        stats = {}
        for k, (p, q) in enumerate(pairs):
            got = km.pair_intersection_regions(A.ring(int(p)), B.ring(int(q)), T=T, region=region, stats=stats)
            assert got == inter[k], (T, region, k)
        assert stats.get("splits", 0) > 0
    C, D, (RA, RB) = combs.generate(n_pairs=3, want_rects=True, max_vertices=600)
    for k in range(3):
        want = combs.rect_decomp_intersection(RA[k], RB[k])
        assert km.pair_intersection_regions(C.ring(k), D.ring(k), T=256, region=96) == want
        assert km.pair_intersection_regions(C.ring(k), D.ring(k), T=256, region=96, mode=1) == want
