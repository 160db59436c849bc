"""GPU parity: the CUDA path, called through the C ABI, against the CPU oracle.

Bar (BASELINE.json north_star): per-pair areas and the integer sums bit-exact;
J' within 1e-12 relative of the exact rational mean.  Inputs are seeded and
synthetic (synth/), at sizes the oracle finishes in seconds that still span many
warps, ragged tails and every code path (pixelization, sampling boxes, the
shared-memory overflow path), plus the full-size bench configuration on
sampled pairs and on size-independent properties.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from synth import combs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def sccg():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests (no CPU fallback exists)")
    import paper_1208_0277_b200 as m

    m.load()
    return m


def dev(pset, sccg):
    xy, off = sccg.to_device(pset.xy, pset.offsets)
    return sccg.DeviceSet(xy, off)


def exact_ratio_units(inter, uni):
    """sum over I != 0 of RN64(I/U) * 2^116, exactly (Python floats are IEEE RN)."""
    tot = 0
    for i, u in zip(inter, uni):
        if i:
            tot += int(Fraction(int(i) / int(u)) * (1 << 116))
    return tot


def check_batch(sccg, A, B, pairs_np, inter, uni, sums, exact=True):
    """Compare a whole batch against the oracle, element by element."""
    ei, eu = oracle.pair_areas(A, B, pairs_np)
    gi, gu = inter.cpu().numpy(), uni.cpu().numpy()
    bad = np.nonzero((gi != ei) | (gu != eu))[0]
    assert len(bad) == 0, f"{len(bad)} mismatches, first {bad[:5]}: gpu {gi[bad[:5]]} {gu[bad[:5]]} oracle {ei[bad[:5]]} {eu[bad[:5]]}"
    s = sums.cpu().tolist()
    os_ = oracle.sums(A, B, pairs_np, ei, eu)
    for k, f in enumerate(["n_pairs", "n_nonzero", "sum_inter", "sum_union", "sum_area_p", "sum_area_q"]):
        assert s[k] == os_[f], f
    assert s[10] == 0, f"status {s[10]}"
    limbs = s[6:10]
    assert sum(l << (30 * i) for i, l in enumerate(limbs)) == exact_ratio_units(ei, eu)
    j, pooled = sccg.jaccard(sums)
    ex = oracle.jaccard_exact(ei, eu)
    if ex is None:
        assert math.isnan(j)
    else:
        assert abs(j - float(ex)) <= 1e-12 * float(ex)
        assert abs(j - oracle.jaccard(ei, eu)) <= 1e-12 * float(ex)
    return ei, eu


# ------------------------------------------------------------------ prep
def test_prep_matches_oracle(sccg, tile_sets):
    for s in tile_sets:
        D = dev(s, sccg)
        area, mbr = oracle.set_props(s)
        assert (D.area.cpu().numpy() == area).all()
        assert (D.mbr.cpu().numpy() == mbr).all()
        assert D.status.cpu().tolist()[0] == 0


def test_prep_sets_one_launch_equals_separate(sccg):
    """sccg_prep_sets over several sets in one launch (shared dynamic tile
    space) gives exactly the per-set results of sccg_prep."""
    sets = [synth.generate("tile", image=i)[i % 2] for i in range(3)]
    sets.append(synth.generate("skewed")[0])
    one = [dev(s, sccg) for s in sets]  # prepped one by one
    many = []
    for s in sets:
        xy, off = sccg.to_device(s.xy, s.offsets)
        many.append(sccg.DeviceSet(xy, off, prep=False))
    arr = (sccg.PolySet * len(many))(*[m.c for m in many])
    assert sccg.load().sccg_prep_sets(arr, len(many), 1, None) == 0
    torch.cuda.synchronize()
    for a, b in zip(one, many):
        for f in ("mbr", "area", "ecount", "status"):
            assert torch.equal(getattr(a, f), getattr(b, f)), f
        sa, sb = a.stats_bytes(), b.stats_bytes()
        assert torch.equal(sa[:24], sb[:24]) and torch.equal(sa[32:64], sb[32:64])  # bounds, extents, moments
        assert torch.equal(a.used_edge_words(), b.used_edge_words())  # records + raster rows
    shared = (sccg.PolySet * 2)(many[0].c, many[0].c)
    assert sccg.load().sccg_prep_sets(shared, 2, 1, None) == sccg.E_ARG


def test_prep_tiles_at_odd_offsets(sccg):
    """Prep's 128-ring tiles start at odd vertex offsets (an odd-V ring opens
    every tile) and every tile ends with a 4-vertex rect whose records + raster
    fill its whole slot: a tile's write-back must not touch the previous tile's
    last slot.  The rects' pairs are checked against the oracle."""
    penta = lambda x, y: [[x, y], [x + 4, y], [x + 4, y + 2], [x + 2, y + 4], [x, y + 4]]
    rect = lambda x, y, w, h: [[x, y], [x + w, y], [x + w, y + h], [x, y + h]]
    rings_p, rings_q = [], []
    rng = np.random.default_rng(17)
    for t in range(300):
        y0 = 40 * t
        rings_p.append(penta(0, y0))
        rings_p += [rect(10 + 3 * i, y0, 2, 2) for i in range(126)]
        h = int(rng.integers(3, 5))
        rings_p.append(rect(500, y0, 5, h))  # raster: 2 records + ceil(h/2) row slots = V
        rings_q.append(rect(502, y0 + 1, 6, 5))
    A, B = synth.pack(rings_p), synth.pack(rings_q)
    xy, off = sccg.to_device(A.xy, A.offsets)
    P = sccg.DeviceSet(xy, off, validate=False)
    Q = dev(B, sccg)
    pairs = sccg.filter_pairs(P, Q)
    assert pairs.shape[0] == 300
    inter, uni, sums = sccg.pixelbox(P, Q, pairs, threshold=2048)
    check_batch(sccg, A, B, pairs.cpu().numpy(), inter, uni, sums)


# ---------------------------------------------------------------- filter
@pytest.mark.parametrize("config", ["tile", "skewed"])
def test_filter_pairs_matches_oracle(sccg, config):
    A, B = synth.generate(config)
    P, Q = dev(A, sccg), dev(B, sccg)
    got = sccg.filter_pairs(P, Q).cpu().numpy()
    want = oracle.join(A, B)
    assert got.shape == want.shape and (got == want).all()


def test_filter_random_boxes_and_touching(sccg):
    rng = np.random.default_rng(11)
    for trial in range(20):
        rings = []
        for n in rng.integers(1, 300, 2):
            rs = []
            for _ in range(n):
                x, y = (int(v) for v in rng.integers(-500, 500, 2))
                w, h = (int(v) for v in rng.integers(1, 60, 2))
                rs.append([[x, y], [x + w, y], [x + w, y + h], [x, y + h]])
            rings.append(synth.pack(rs))
        A, B = rings
        got = sccg.filter_pairs(dev(A, sccg), dev(B, sccg)).cpu().numpy()
        assert got.tolist() == oracle.join(A, B, "nested").tolist()
    # touching MBRs share no pixel -> no pair (reading R4)
    A = synth.pack([[[0, 0], [2, 0], [2, 2], [0, 2]]])
    B = synth.pack([[[2, 0], [4, 0], [4, 2], [2, 2]], [[0, 2], [2, 2], [2, 4], [0, 4]]])
    assert sccg.filter_pairs(dev(A, sccg), dev(B, sccg)).shape[0] == 0


def test_filter_long_segments(sccg):
    """Polygons of P that pair with many Q (a gland over nuclei, C3): segments
    of 5..32 (thread sort), 33..4096 (warp bitonic sort) and > 4096 (fallback)
    pairs, from MBRs covering few or many grid cells, all sorted by (p, q)."""
    rng = np.random.default_rng(23)
    rings_q = []
    for i in range(9000):  # small boxes on a jittered lattice
        x, y = 3 * (i % 100) + int(rng.integers(0, 2)), 3 * (i // 100) + int(rng.integers(0, 2))
        rings_q.append([[x, y], [x + 2, y], [x + 2, y + 2], [x, y + 2]])
    far = lambda i: [[5000 + 3 * i, 5000], [5001 + 3 * i, 5000], [5001 + 3 * i, 5001], [5000 + 3 * i, 5001]]
    rings_p = [[[0, 0], [300, 0], [300, 300], [0, 300]]]  # > 4096 pairs: its 128-polygon tile overflows its bucket
    rings_p += [far(i) for i in range(127)]
    rings_p += [[[10, 10], [70, 10], [70, 70], [10, 70]],  # ~400 pairs: sorted by the compaction pass
                [[100, 100], [112, 100], [112, 106], [100, 106]],  # ~10-30 pairs: sorted by its thread
                [[150, 150], [152, 150], [152, 152], [150, 152]],  # a few: sorted in registers
                [[20, 200], [80, 200], [80, 240], [20, 240]]]  # ~270 pairs, same tile as the ~400
    A, B = synth.pack(rings_p), synth.pack(rings_q)
    got = sccg.filter_pairs(dev(A, sccg), dev(B, sccg)).cpu().numpy()
    want = oracle.join(A, B)
    assert got.tolist() == want.tolist()
    counts = np.bincount(want[:, 0], minlength=132)
    assert counts[0] > 4096 and 32 < counts[128] <= 1024 and 4 < counts[129] <= 32 and counts[131] > 32, counts


def test_filter_crowded_buckets_overflow_chains(sccg):
    """Many Q MBRs in one grid cell: a bucket's count runs past its 32 slots
    into the overflow chain (walked by thread-per-p visits and by big-MBR
    visits), and stacked identical boxes; also the closed join and every pair
    list against the nested-loop oracle."""
    rng = np.random.default_rng(5)
    rings_q = [[[0, 0], [4, 0], [4, 4], [0, 4]] for _ in range(150)]  # 150 identical boxes
    for _ in range(400):  # a crowd of small boxes in a 40 x 40 patch
        x, y = (int(v) for v in rng.integers(0, 40, 2))
        rings_q.append([[x, y], [x + 3, y], [x + 3, y + 3], [x, y + 3]])
    rings_q += [[[5000 + 10 * i, 0], [5004 + 10 * i, 0], [5004 + 10 * i, 4], [5000 + 10 * i, 4]] for i in range(50)]
    rings_p = [[[1, 1], [3, 1], [3, 3], [1, 3]], [[0, 0], [45, 0], [45, 45], [0, 45]],  # small, crowd-wide
               [[-2000, -2000], [3000, -2000], [3000, 3000], [-2000, 3000]]]  # a big MBR over many cells
    for _ in range(200):
        x, y = (int(v) for v in rng.integers(-10, 50, 2))
        rings_p.append([[x, y], [x + 2, y], [x + 2, y + 5], [x, y + 5]])
    A, B = synth.pack(rings_p), synth.pack(rings_q)
    P, Q = dev(A, sccg), dev(B, sccg)
    got = sccg.filter_pairs(P, Q).cpu().numpy()
    assert got.tolist() == oracle.join(A, B, "nested").tolist()
    assert np.bincount(got[:, 0]).max() > 500
    gotc = sccg.filter_pairs(P, Q, closed=True).cpu().numpy()
    assert gotc.tolist() == oracle.join(A, B, "closed").tolist()


def test_filter_closed_matches_oracle(sccg, tile_sets):
    """Closed-box join (touching MBRs pair too): the ST_Touches candidates."""
    A, B = tile_sets
    got = sccg.filter_pairs(dev(A, sccg), dev(B, sccg), closed=True).cpu().numpy()
    _, mp = oracle.set_props(A)
    _, mq = oracle.set_props(B)
    assert got.tolist() == oracle.join_mbrs(mp, mq, "closed").tolist()
    rng = np.random.default_rng(13)
    for trial in range(10):
        sets = []
        for n in rng.integers(1, 200, 2):
            rs = []
            for _ in range(n):
                x, y = (int(v) for v in rng.integers(0, 60, 2))
                w, h = (int(v) for v in rng.integers(1, 8, 2))
                rs.append([[x, y], [x + w, y], [x + w, y + h], [x, y + h]])
            sets.append(synth.pack(rs))
        S, T = sets
        got = sccg.filter_pairs(dev(S, sccg), dev(T, sccg), closed=True).cpu().numpy()
        want = oracle.join_mbrs(oracle.set_props(S)[1], oracle.set_props(T)[1], "closed")
        assert got.tolist() == want.tolist()


def _touch_sets():
    """Hand-made contact cases (one pair each, far apart) and the expected
    answers: shared side, partial side, corner, gap, overlap, identical,
    contained with a shared side, L-shape notch contact, containing."""
    sq = lambda x, y, w, h: [[x, y], [x + w, y], [x + w, y + h], [x, y + h]]
    L = lambda x, y: [[x, y], [x + 4, y], [x + 4, y + 2], [x + 2, y + 2], [x + 2, y + 4], [x, y + 4]]
    cases = [
        (sq(0, 0, 2, 2), sq(2, 0, 2, 2), True),
        (sq(0, 0, 4, 4), sq(4, 1, 2, 2), True),
        (sq(0, 0, 2, 2), sq(2, 2, 2, 2), True),
        (sq(0, 0, 2, 2), sq(3, 0, 2, 2), False),
        (sq(0, 0, 3, 3), sq(2, 2, 3, 3), False),
        (sq(0, 0, 2, 2), sq(0, 0, 2, 2), False),
        (sq(0, 0, 4, 4), sq(0, 0, 2, 4), False),
        (L(0, 0), sq(2, 2, 2, 2), True),
        (L(0, 0), sq(3, 3, 1, 1), False),
        (sq(0, 0, 6, 6), sq(2, 2, 2, 2), False),
    ]
    P, Q, want = [], [], []
    for i, (a, b, t) in enumerate(cases):
        off = np.array([20 * i, 0], np.int32)
        P.append(np.asarray(a, np.int32) + off)
        Q.append(np.asarray(b, np.int32) + off)
        want.append(t)
    return synth.pack(P), synth.pack(Q), want


def test_touches_matches_oracle(sccg, tile_sets):
    """ST_Touches (R21) through the C ABI: closed-join candidates,
    PixelBox intersections, then the vertex-on-edge test -- against the
    oracle's pixel-adjacency definition, on hand-made cases, on the tile
    sets and on rectilinear blobs packed edge to edge."""
    A, B, want = _touch_sets()
    P, Q = dev(A, sccg), dev(B, sccg)
    pairs = sccg.filter_pairs(P, Q, closed=True)
    pl = pairs.cpu().numpy()
    assert pl.tolist() == oracle.join(A, B, "closed").tolist()  # the gap case's MBRs do not even meet
    inter, _, _ = sccg.pixelbox(P, Q, pairs)
    t = dict(zip(map(tuple, pl.tolist()), sccg.touches(P, Q, pairs, inter).cpu().numpy().astype(bool).tolist()))
    assert [t.get((k, k), False) for k in range(len(want))] == want
    assert [oracle.touches(A.ring(k), B.ring(k)) for k in range(len(want))] == want
    # tile sets (nuclei hardly ever touch), partitions of a square against
    # themselves (neighbouring pieces touch along sides / at corners) and
    # against another partition of the same square (mostly overlapping)
    parts = [synth.partition(s) for s in (3, 4, 5)]
    total = 0
    for S, T in (tile_sets, (parts[0], parts[0]), (parts[1], parts[1]), (parts[1], parts[2])):
        P, Q = dev(S, sccg), dev(T, sccg)
        pairs = sccg.filter_pairs(P, Q, closed=True)
        inter, _, _ = sccg.pixelbox(P, Q, pairs)
        got = sccg.touches(P, Q, pairs, inter).cpu().numpy()
        exp = oracle.touches_pairs(S, T, pairs.cpu().numpy())
        assert (got == exp).all(), np.nonzero(got != exp)[0][:10]
        total += int(exp.sum())
    assert total > 300


def test_filter_capacity_retry(sccg, tile_sets):
    A, B = tile_sets
    got = sccg.filter_pairs(dev(A, sccg), dev(B, sccg), cap=3).cpu().numpy()
    assert got.tolist() == oracle.join(A, B).tolist()


# -------------------------------------------------------------- pixelbox
@pytest.mark.parametrize("raster", [True, False])
@pytest.mark.parametrize("T", [2, 37, 512, 2048, 1 << 30])
def test_pixelbox_tile_all_T(sccg, tile_sets, T, raster):
    """Every path and threshold; raster=False forces the per-pair edge
    pixelization (the paper's schedule) where prep stored a ring's raster."""
    A, B = tile_sets
    P, Q = dev(A, sccg), dev(B, sccg)
    pairs = sccg.filter_pairs(P, Q)
    inter, uni, sums = sccg.pixelbox(P, Q, pairs, threshold=T, raster=raster)
    check_batch(sccg, A, B, pairs.cpu().numpy(), inter, uni, sums)


@pytest.mark.parametrize("mode", [1, 2])
def test_pixelbox_baseline_modes(sccg, tile_sets, mode):
    """The §5.2 baselines: PixelOnly (1) and PixelBox-NoSep (2) count
    the union directly -- it must equal the oracle's directly counted union,
    which also checks |p u q| = |p| + |q| - |p n q| on the GPU side."""
    A, B = tile_sets
    P, Q = dev(A, sccg), dev(B, sccg)
    pairs = sccg.filter_pairs(P, Q)
    for T in (64, 2048):
        inter, uni, sums = sccg.pixelbox(P, Q, pairs, mode=mode, threshold=T)
        check_batch(sccg, A, B, pairs.cpu().numpy(), inter, uni, sums)
    S, R = synth.generate("skewed", width=4096, height=4096)
    P, Q = dev(S, sccg), dev(R, sccg)
    pairs = sccg.filter_pairs(P, Q)
    inter, uni, sums = sccg.pixelbox(P, Q, pairs, mode=mode, threshold=256)
    check_batch(sccg, S, R, pairs.cpu().numpy(), inter, uni, sums)
    C, D = combs.generate(n_pairs=8)
    P, Q = dev(C, sccg), dev(D, sccg)
    pairs = sccg.filter_pairs(P, Q)
    inter, uni, sums = sccg.pixelbox(P, Q, pairs, mode=mode, threshold=512)
    check_batch(sccg, C, D, pairs.cpu().numpy(), inter, uni, sums)


@pytest.mark.parametrize("T", [64, 2048])
def test_pixelbox_skewed_glands(sccg, T):
    """Config 3 analog: nuclei + glands (MBR side up to 512, ~1000 vertices):
    deep sampling-box subdivision and the shared-memory overflow path."""
    A, B = synth.generate("skewed", width=8192, height=8192)
    P, Q = dev(A, sccg), dev(B, sccg)
    pairs = sccg.filter_pairs(P, Q)
    counters = torch.zeros(8, dtype=torch.int64, device="cuda")
    inter, uni, sums = sccg.pixelbox(P, Q, pairs, threshold=T, counters=counters)
    check_batch(sccg, A, B, pairs.cpu().numpy(), inter, uni, sums)
    c = counters.cpu().tolist()
    assert c[sccg.CNT_SPLITS] > 0 and c[sccg.CNT_PIXBOXES] > 0
    # Alg. 1's split order as written (no dense-split shortcut): the same areas
    i2, u2, s2 = sccg.pixelbox(P, Q, pairs, threshold=T, paper_split=True)
    assert torch.equal(i2, inter) and torch.equal(u2, uni) and torch.equal(s2, sums)


def _staircase(x0, y0, n, step=1):
    """Rectilinear staircase ring with n unit steps: n + 1 vertical edges."""
    ring = [[x0, y0], [x0 + n * step, y0]]
    for i in range(n, 0, -1):
        ring += [[x0 + i * step, y0 + (n - i + 1) * step], [x0 + (i - 1) * step, y0 + (n - i + 1) * step]]
    return ring[:-1] + [[x0, y0 + n * step]]


def test_pixelbox_windows_and_wide_pairs(sccg):
    """Pair boxes of 33..64 px (pixelized in <= 32 x 32 windows) and polygons
    with 65..128 vertical edges (the non-pipelined loop), against the oracle."""
    rng = np.random.default_rng(31)
    rp, rq = [], []
    for t in range(400):
        x0, y0 = 400 * (t % 20), 400 * (t // 20)
        kind = t % 4
        if kind == 0:  # windows: random rects, boxes up to 64
            w1, h1, w2, h2 = (int(v) for v in rng.integers(20, 65, 4))
            dx, dy = (int(v) for v in rng.integers(-10, 10, 2))
            rp.append([[x0, y0], [x0 + w1, y0], [x0 + w1, y0 + h1], [x0, y0 + h1]])
            rq.append([[x0 + dx, y0 + dy], [x0 + dx + w2, y0 + dy], [x0 + dx + w2, y0 + dy + h2], [x0 + dx, y0 + dy + h2]])
        elif kind == 1:  # wide: a staircase of 65..127 steps over a box <= 64
            n = int(rng.integers(65, 128))
            rp.append(_staircase(x0, y0, n))
            a, b = int(rng.integers(0, n - 64)), int(rng.integers(0, n - 64))
            rq.append([[x0 + a, y0 + b], [x0 + a + 60, y0 + b], [x0 + a + 60, y0 + b + 50], [x0 + a, y0 + b + 50]])
        elif kind == 2:  # wide on both sides
            n, m = (int(v) for v in rng.integers(65, 128, 2))
            rp.append(_staircase(x0, y0, n))
            ox, oy = x0 + n - 60, y0 + n - 60  # MBR overlap 60 x 60
            rq.append([[ox + x, oy + m - y] for x, y in _staircase(0, 0, m)][::-1])
        else:  # a 1-px-step staircase against a staircase: many edges, box 33..64
            n = int(rng.integers(33, 64))
            rp.append(_staircase(x0, y0, n))
            rq.append(_staircase(x0 + 2, y0 + 1, n))
    A, B = synth.pack(rp), synth.pack(rq)
    P, Q = dev(A, sccg), dev(B, sccg)
    pairs = sccg.filter_pairs(P, Q)
    assert pairs.shape[0] >= 400
    # by construction every pair is on the small kernel (box <= 64 x 64, <= 128
    # vertical edges per polygon), and both new routes occur
    pr = pairs.long()
    mp, mq = P.mbr.long()[pr[:, 0]], Q.mbr.long()[pr[:, 1]]
    W = torch.minimum(mp[:, 2], mq[:, 2]) - torch.maximum(mp[:, 0], mq[:, 0])
    H = torch.minimum(mp[:, 3], mq[:, 3]) - torch.maximum(mp[:, 1], mq[:, 1])
    nvm = sccg.RASTER_FLAG - 1  # ecount[:, 0] = count | raster flag
    nv = torch.maximum(P.ecount.long()[pr[:, 0], 0] & nvm, Q.ecount.long()[pr[:, 1], 0] & nvm)
    assert int(W.max()) <= 64 and int(H.max()) <= 64 and int(nv.max()) <= 128
    assert int(((W > 32) | (H > 32)).sum()) > 50 and int((nv > 64).sum()) > 50
    for raster in (True, False):
        inter, uni, sums = sccg.pixelbox(P, Q, pairs, threshold=1 << 30, raster=raster)
        check_batch(sccg, A, B, pairs.cpu().numpy(), inter, uni, sums)
    counters = torch.zeros(8, dtype=torch.int64, device="cuda")
    sccg.pixelbox(P, Q, pairs, threshold=1 << 30, counters=counters)
    assert int(counters[sccg.CNT_BOXES]) == 0  # every pair took the small kernel's pixelization


def test_pixelbox_combs_closed_form(sccg):
    """Config 5 analog: highly concave combs, pinned by rectangle decomposition."""
    A, B, (RA, RB) = combs.generate(n_pairs=96, want_rects=True)
    P, Q = dev(A, sccg), dev(B, sccg)
    pairs = sccg.filter_pairs(P, Q)
    assert pairs.cpu().numpy().tolist() == [[k, k] for k in range(96)]
    # small T: many small leaf boxes (per-row crossings); 2^30: whole regions
    # pixelized in bands (difference trick); modes 1/2 count the union directly
    # paper_split: every continuing sub-box pushed (Alg. 1 as written) instead of dense splits pixelized whole
    for T, mode, ps in ((256, 0, False), (256, 0, True), (2048, 0, False), (2048, 0, True), (4096, 0, False),
                        (1 << 30, 0, False), (1 << 30, 1, False), (4096, 2, False)):
        inter, uni, sums = sccg.pixelbox(P, Q, pairs, threshold=T, mode=mode, paper_split=ps)
        gi, gu = inter.cpu().numpy(), uni.cpu().numpy()
        for k in range(96):
            want = combs.rect_decomp_intersection(RA[k], RB[k])
            assert gi[k] == want, (T, mode, ps, k)
            assert gu[k] == combs.rect_decomp_area(RA[k]) + combs.rect_decomp_area(RB[k]) - want, (T, mode, ps, k)
    check_batch(sccg, A, B, pairs.cpu().numpy()[:24], *sccg.pixelbox(P, Q, pairs[:24]))


def test_pixelbox_exhaustive_tiny(sccg):
    """Every clean 3x3 polyomino against every other at offsets in [-2, 2]^2."""
    import itertools

    polys = []
    for bits in range(1, 512):
        m = np.array([(bits >> i) & 1 for i in range(9)], np.uint8).reshape(3, 3)
        ring, cleaned = synth.trace_mask(m)
        if ring is not None and (cleaned == m).all():
            polys.append(ring)
    offs = list(itertools.product(range(-2, 3), repeat=2))
    A = synth.pack(polys)
    B = synth.pack([r + np.array(o, np.int32) for r in polys for o in offs])
    P, Q = dev(A, sccg), dev(B, sccg)
    pairs_np = np.array([(i, j) for i in range(len(polys)) for j in range(len(polys) * len(offs))], np.int32)
    pairs = torch.from_numpy(pairs_np).cuda()
    for T in (2, 4, 2048):
        inter, uni, sums = sccg.pixelbox(P, Q, pairs, threshold=T)
        ei, eu = oracle.pair_areas(A, B, pairs_np)
        assert (inter.cpu().numpy() == ei).all() and (uni.cpu().numpy() == eu).all()


def test_pixelbox_edge_cases(sccg, tile_sets):
    A, B = tile_sets
    P, Q = dev(A, sccg), dev(B, sccg)
    # empty batch
    inter, uni, sums = sccg.pixelbox(P, Q, torch.zeros((0, 2), dtype=torch.int32, device="cuda"))
    assert inter.numel() == 0 and sums.cpu().tolist() == [0] * 11
    assert math.isnan(sccg.jaccard(sums)[0])
    # pairs with disjoint MBRs are allowed: I = 0, U = |p| + |q|
    pairs_np = np.array([[0, B.n - 1], [A.n - 1, 0], [3, 3]], np.int32)
    inter, uni, sums = sccg.pixelbox(P, Q, torch.from_numpy(pairs_np).cuda())
    check_batch(sccg, A, B, pairs_np, inter, uni, sums)
    # a single ragged pair, identical polygons -> r = 1 exactly
    pairs_np = np.array([[5, 5]], np.int32)
    inter, uni, sums = sccg.pixelbox(P, P, torch.from_numpy(pairs_np).cuda())
    assert inter.item() == uni.item() == oracle.area_shoelace(A.ring(5))
    assert sccg.jaccard(sums)[0] == 1.0
    # out-of-range pair index: skipped and flagged, never read out of bounds
    bad = torch.tensor([[0, 10**6]], dtype=torch.int32, device="cuda")
    _, _, sums = sccg.pixelbox(P, Q, bad, check=False)
    assert sums.cpu().tolist()[10] == sccg.STATUS_ARG


def test_sums_accumulate_and_launch_shape_invariance(sccg, tile_sets):
    A, B = tile_sets
    P, Q = dev(A, sccg), dev(B, sccg)
    pairs = sccg.filter_pairs(P, Q)
    ref = sccg.pixelbox(P, Q, pairs)
    for grid in (1, 3, 37):
        got = sccg.pixelbox(P, Q, pairs, grid=grid)
        assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1]) and torch.equal(got[2], ref[2])
    # batching: two halves accumulated into one sums == one call
    sums = sccg.new_sums()
    h = pairs.shape[0] // 2
    sccg.pixelbox(P, Q, pairs[:h], sums=sums)
    sccg.pixelbox(P, Q, pairs[h:], sums=sums)
    assert torch.equal(sums, ref[2])


def test_async_pipeline_matches_sync(sccg, tile_sets):
    """sccg_filter_pairs_async + sccg_pixelbox_async (device-side pair count),
    eager and captured as CUDA graphs, equal the synchronous path bit for bit."""
    A, B = tile_sets
    P, Q = dev(A, sccg), dev(B, sccg)
    pairs = sccg.filter_pairs(P, Q)
    ref = sccg.pixelbox(P, Q, pairs)[2]
    for graph in (False, True):
        pipe = sccg.Pipeline(P, Q, graph=graph)
        for _ in range(3):
            s = pipe.run()
        assert torch.equal(s, ref)
        assert pipe.check() == pairs.shape[0]
        assert torch.equal(pipe.pairs[: pairs.shape[0]], pairs)
    # the bench's step: the PixelBox graph ends with the read-back kernel into pinned slot k
    rb = [torch.zeros(ref.shape, dtype=torch.int64).pin_memory() for _ in range(2)]
    pipe = sccg.Pipeline(P, Q, graph=True, readback=rb)
    for i in range(4):
        s = pipe.run(slot=i % 2)
        torch.cuda.synchronize()
        assert rb[i % 2].tolist() == ref.tolist() and torch.equal(s, ref)
        # the read-back kernel (sccg_sums_copy) into device memory and into pinned host memory
    d = sccg.sums_copy(ref, torch.empty_like(ref))
    h = sccg.sums_copy(ref, torch.zeros(ref.shape, dtype=torch.int64).pin_memory())
    torch.cuda.synchronize()
    assert torch.equal(d, ref) and h.tolist() == ref.tolist()
    tiny = sccg.Pipeline(P, Q, cap=10, graph=False)
    tiny.run()
    with pytest.raises(sccg.SccgError) as e:
        tiny.check()
    assert e.value.code == sccg.E_CAPACITY


def test_missing_polygons_and_contains(sccg, tile_sets):
    """NEXT(f3)/(f4): missing-polygon counts from the kernels' hit
    bitmaps, and ST_Contains by areas (sccg_contains), against the
    oracle's pixel-set definitions."""
    A, B = tile_sets
    for cfg in ("tile", "skewed"):
        if cfg == "skewed":
            A, B = synth.generate("skewed", width=4096, height=4096)
        P, Q = dev(A, sccg), dev(B, sccg)
        pairs = sccg.filter_pairs(P, Q)
        hits = sccg.new_hits(P, Q)
        inter, uni, sums = sccg.pixelbox(P, Q, pairs, hits=hits)
        pn = pairs.cpu().numpy()
        ei, _ = oracle.pair_areas(A, B, pn)
        assert sccg.missing_polygons(hits, P, Q) == (oracle.missing(A.n, pn, ei, 0), oracle.missing(B.n, pn, ei, 1))
        got = sccg.contains(P, Q, pairs, inter).cpu().numpy()
        assert (got == oracle.contains_pairs(A, B, pn)).all()
    # hand-made containment cases: nested, identical, sharing sides, L-shape notch, overlap, disjoint MBR pair
    sq = lambda x, y, w, h: [[x, y], [x + w, y], [x + w, y + h], [x, y + h]]
    L = lambda x, y: [[x, y], [x + 6, y], [x + 6, y + 3], [x + 3, y + 3], [x + 3, y + 6], [x, y + 6]]
    cases = [(sq(0, 0, 8, 8), sq(2, 2, 3, 3), 1), (sq(2, 2, 3, 3), sq(0, 0, 8, 8), 2), (sq(0, 0, 4, 4), sq(0, 0, 4, 4), 3),
             (sq(0, 0, 8, 8), sq(0, 0, 8, 3), 1), (L(0, 0), sq(3, 3, 3, 3), 0), (L(0, 0), sq(0, 0, 3, 6), 1),
             (sq(0, 0, 4, 4), sq(2, 2, 4, 4), 0), (sq(0, 0, 40, 40), sq(5, 5, 30, 30), 1)]
    PP = synth.pack([np.asarray(a, np.int32) + np.array([100 * i, 0], np.int32) for i, (a, _, _) in enumerate(cases)])
    QQ = synth.pack([np.asarray(b, np.int32) + np.array([100 * i, 0], np.int32) for i, (_, b, _) in enumerate(cases)])
    P, Q = dev(PP, sccg), dev(QQ, sccg)
    pairs = torch.tensor([[i, i] for i in range(len(cases))], dtype=torch.int32, device="cuda")
    inter, _, _ = sccg.pixelbox(P, Q, pairs)
    got = sccg.contains(P, Q, pairs, inter).cpu().numpy().tolist()
    assert got == [c for _, _, c in cases]
    assert got == oracle.contains_pairs(PP, QQ, pairs.cpu().numpy()).tolist()


def _report_check(sccg, A, B, tiling):
    P, Q = dev(A, sccg), dev(B, sccg)
    pairs = sccg.filter_pairs(P, Q)
    hits = sccg.new_hits(P, Q)
    inter, uni, sums = sccg.pixelbox(P, Q, pairs, hits=hits)
    got = sccg.tile_report(P, Q, pairs, inter, uni, hits, tiling).cpu().numpy()
    pn = pairs.cpu().numpy()
    ei, eu = oracle.pair_areas(A, B, pn)
    want = oracle.report(A, B, pn, ei, eu, tiling)
    limbs = slice(6, 10)
    units = lambda r: sum(int(v) << (30 * k) for k, v in enumerate(r[limbs]))
    for t in range(got.shape[0]):
        g, w = got[t].tolist(), want[t].tolist()
        assert g[:6] == w[:6] and g[10:] == w[10:], (t, g, w)
        assert units(got[t]) == units(want[t]), t
    rep = sccg.similarity_report(P, Q, pairs, inter, uni, hits, tiling)
    ex = oracle.jaccard_exact(ei, eu)
    assert abs(rep["jaccard"] - float(ex)) <= 1e-12 * float(ex)
    assert (rep["missing_p"], rep["missing_q"]) == (oracle.missing(A.n, pn, ei, 0), oracle.missing(B.n, pn, ei, 1))
    for t in rep["tiles"]:
        row = want[t["tile_id"]]
        if row[1]:
            exact = Fraction(units(row), 1 << 116) / int(row[1])
            assert abs(t["jaccard"] - float(exact)) <= 1e-12 * float(exact)
        else:
            assert t["jaccard"] is None
    return got


def test_tile_report_matches_oracle(sccg, tile_sets):
    """NEXT(f3): the per-tile SimilarityReport (reading R22) --
    pair totals, exact ratio limbs, per-tile J', polygon and missing counts --
    against the oracle's report, on a 3 x 3 grid over the tile set, a grid with
    tiles outside the data (clamping), the skewed image and the whole slide
    (25 x 25 tiles of 4096)."""
    A, B = tile_sets
    _report_check(sccg, A, B, (0, 0, 1500, 1500, 3, 3))
    _report_check(sccg, A, B, (-1000, 500, 700, 900, 5, 4))
    _report_check(sccg, *synth.generate("skewed", width=8192, height=8192), (0, 0, 4096, 4096, 2, 2))
    got = _report_check(sccg, *synth.generate("slide"), (0, 0, 4096, 4096, 25, 25))
    assert (got[:, 0] > 0).sum() > 500


def test_maximum_sizes_closed_form(sccg):
    """Limits of the ABI (R20): MBR extents of 65535 pixels, coordinates near
    +-2^30, |p n q| > 2^31 -- pinned by rectangle closed forms and disjoint-
    rectangle-union combs (no oracle scan of 4e9 pixels)."""
    big = (1 << 30) - 70000
    rects_p = [(big, big, big + 65535, big + 65535), (-(1 << 30), 0, -(1 << 30) + 65535, 3),
               (0, -(1 << 30), 40000, -(1 << 30) + 65535)]
    rects_q = [(big + 1000, big + 999, big + 65535, big + 65535), (-(1 << 30) + 5, 1, -(1 << 30) + 65000, 2),
               (39999, -(1 << 30) + 1, 50000, -(1 << 30) + 65534)]
    ring = lambda r: [[r[0], r[1]], [r[2], r[1]], [r[2], r[3]], [r[0], r[3]]]
    A, B = synth.pack([ring(r) for r in rects_p]), synth.pack([ring(r) for r in rects_q])
    P, Q = dev(A, sccg), dev(B, sccg)
    pairs = sccg.filter_pairs(P, Q)
    assert pairs.cpu().numpy().tolist() == [[0, 0], [1, 1], [2, 2]]
    for T in (64, 2048):
        inter, uni, sums = sccg.pixelbox(P, Q, pairs, threshold=T)
        for k, (a, b) in enumerate(zip(rects_p, rects_q)):
            ow = max(0, min(a[2], b[2]) - max(a[0], b[0]))
            oh = max(0, min(a[3], b[3]) - max(a[1], b[1]))
            area = lambda r: (r[2] - r[0]) * (r[3] - r[1])
            assert inter[k].item() == ow * oh and uni[k].item() == area(a) + area(b) - ow * oh
        assert inter[0].item() > 1 << 31  # beyond int32
    # a comb spanning the full extent against its shifted copy (closed form)
    ra, Ra = combs.comb(-50000, 7, 16383, 2, 2, 60000, 5)  # W = 65534
    rb, Rb = combs.comb(-49999, 9, 16383, 2, 2, 60000, 5)
    C, D = synth.pack([ra]), synth.pack([rb])
    P, Q = dev(C, sccg), dev(D, sccg)
    pairs = sccg.filter_pairs(P, Q)
    inter, uni, _ = sccg.pixelbox(P, Q, pairs)
    want = combs.rect_decomp_intersection(Ra, Rb)
    assert inter.item() == want
    assert uni.item() == combs.rect_decomp_area(Ra) + combs.rect_decomp_area(Rb) - want


def test_abi_errors(sccg):
    bad = synth.pack([[[0, 0], [3, 1], [3, 3], [0, 3]]])  # diagonal edge
    good = synth.pack([[[0, 0], [3, 0], [3, 3], [0, 3]]])
    with pytest.raises(sccg.SccgError) as e:
        sccg.filter_pairs(dev(bad, sccg), dev(good, sccg))
    assert e.value.code == sccg.E_NOT_RECTILINEAR and e.value.index == 0
    wide = synth.pack([[[0, 0], [70000, 0], [70000, 3], [0, 3]]])
    with pytest.raises(sccg.SccgError) as e:
        sccg.filter_pairs(dev(good, sccg), dev(wide, sccg))
    assert e.value.code == sccg.E_RANGE
    tri = synth.PolygonSet(np.array([[0, 0], [1, 0], [1, 1]], np.int32), np.array([0, 3], np.int64))
    with pytest.raises(sccg.SccgError) as e:
        sccg.filter_pairs(dev(tri, sccg), dev(good, sccg))
    assert e.value.code == sccg.E_ARG
    # empty sets
    empty = synth.PolygonSet(np.zeros((0, 2), np.int32), np.zeros(1, np.int64))
    assert sccg.filter_pairs(dev(empty, sccg), dev(good, sccg)).shape[0] == 0
    assert sccg.filter_pairs(dev(good, sccg), dev(empty, sccg)).shape[0] == 0
    assert sccg.filter_pairs(dev(empty, sccg), dev(empty, sccg)).shape[0] == 0


# --------------------------------------------------- full bench configuration
def test_slide_full_size(sccg):
    """Config 2 (the bench workload) at full size, in the bench's launch
    configuration: the whole pair list equals the oracle's sweep join, EVERY
    pair's (I, U) equals the oracle's pixel counts, the integer sums and the
    ratio limbs equal the oracle-side totals, and J' is within 1e-12 of the
    exact rational mean."""
    A, B = synth.generate("slide")
    P, Q = dev(A, sccg), dev(B, sccg)
    pairs = sccg.filter_pairs(P, Q)
    pn = pairs.cpu().numpy()
    want = oracle.join(A, B)
    assert pn.shape == want.shape and (pn == want).all()
    inter, uni, sums = sccg.pixelbox(P, Q, pairs)
    ei, eu = check_batch(sccg, A, B, pn, inter, uni, sums)  # all pairs, sums, limbs, J'
    # determinism across thresholds and pixelization schedules: per-pair results identical
    i2, u2, s2 = sccg.pixelbox(P, Q, pairs, threshold=64)
    assert torch.equal(i2, inter) and torch.equal(s2, sums)
    i3, u3, s3 = sccg.pixelbox(P, Q, pairs, raster=False)
    assert torch.equal(i3, inter) and torch.equal(s3, sums)
    # the bench's launch configuration (device-resident pipeline, CUDA graphs, outputs written every step)
    pipe = sccg.Pipeline(P, Q, cap=3 * max(P.n, Q.n) + 1024, graph=True)
    for _ in range(2):
        ps = pipe.run()
    assert pipe.check() == len(pn)
    assert torch.equal(ps, sums)
    n = len(pn)
    assert torch.equal(pipe.inter[:n], inter) and torch.equal(pipe.uni[:n], uni)


def test_skewed_full_size(sccg):
    """Config 3 at full size (16384^2, nuclei + glands): every pair against the
    oracle (join, per-pair areas, sums, limbs, J')."""
    A, B = synth.generate("skewed")
    P, Q = dev(A, sccg), dev(B, sccg)
    pairs = sccg.filter_pairs(P, Q)
    pn = pairs.cpu().numpy()
    assert pn.tolist() == oracle.join(A, B).tolist()
    inter, uni, sums = sccg.pixelbox(P, Q, pairs)
    check_batch(sccg, A, B, pn, inter, uni, sums)
    pipe = sccg.Pipeline(P, Q, graph=True)
    pipe.run()
    assert pipe.check() == len(pn) and torch.equal(pipe.sums, sums)


def test_combs_full_size(sccg):
    """Config 5 analog at full size (16,384 comb pairs, 500-2000 vertices):
    EVERY pair pinned by its rectangle-decomposition closed form, and a seeded
    512-pair subset by the oracle's brute-force pixel counts."""
    A, B, (RA, RB) = combs.generate(want_rects=True)
    P, Q = dev(A, sccg), dev(B, sccg)
    pairs = sccg.filter_pairs(P, Q)
    n = A.n
    assert pairs.cpu().numpy().tolist() == [[k, k] for k in range(n)]
    inter, uni, sums = sccg.pixelbox(P, Q, pairs)
    gi, gu = inter.cpu().numpy(), uni.cpu().numpy()
    wi = np.array([combs.rect_decomp_intersection(RA[k], RB[k]) for k in range(n)], np.int64)
    wa = np.array([combs.rect_decomp_area(RA[k]) for k in range(n)], np.int64)
    wb = np.array([combs.rect_decomp_area(RB[k]) for k in range(n)], np.int64)
    bad = np.nonzero(gi != wi)[0]
    assert len(bad) == 0, (bad[:5], gi[bad[:5]], wi[bad[:5]])
    assert (gu == wa + wb - wi).all()
    s = sums.cpu().tolist()
    assert s[0] == n and s[1] == int((wi > 0).sum()) and s[2] == int(wi.sum()) and s[10] == 0
    assert s[4] == int(wa.sum()) and s[5] == int(wb.sum())
    assert sum(l << (30 * i) for i, l in enumerate(s[6:10])) == exact_ratio_units(wi, wa + wb - wi)
    idx = np.sort(np.random.default_rng(5).choice(n, size=512, replace=False))
    ei, eu = oracle.pair_areas(A, B, pairs.cpu().numpy()[idx])
    assert (ei == gi[idx]).all() and (eu == gu[idx]).all()


def _ring_variant(ring, rng, kind):
    """The same pixel set, written differently (DESIGN R2/R3): clockwise,
    duplicated consecutive vertices, extra collinear vertices, or the first
    vertex repeated at the end."""
    r = [tuple(int(c) for c in v) for v in np.asarray(ring)]
    if kind == "cw":
        return np.asarray(r[::-1], np.int32)
    if kind == "closing":
        return np.asarray(r + [r[0]], np.int32)
    out = []
    for i, a in enumerate(r):
        b = r[(i + 1) % len(r)]
        out.append(a)
        if kind == "dup" and rng.random() < 0.3:
            out.append(a)
        if kind == "collinear" and rng.random() < 0.5:
            dx, dy = np.sign(b[0] - a[0]), np.sign(b[1] - a[1])
            ln = abs(b[0] - a[0]) + abs(b[1] - a[1])
            if ln >= 2:
                t = int(rng.integers(1, ln))
                out.append((a[0] + t * dx, a[1] + t * dy))
    return np.asarray(out, np.int32)


@pytest.mark.parametrize("kind", ["cw", "dup", "collinear", "closing", "mixed"])
def test_ring_variants_same_results(sccg, tile_sets, kind):
    """Input contract (sccg.h, DESIGN R2/R3): either orientation, duplicate or
    collinear consecutive vertices and a repeated closing vertex are accepted
    (validation on) and change nothing: per-pair results equal the oracle's on
    the rewritten rings and the GPU's on the plain rings, bit for bit."""
    A, B = tile_sets
    rng = np.random.default_rng(hash(kind) & 0xFFFF)
    kinds = ["cw", "dup", "collinear", "closing"]
    pick = (lambda: kinds[int(rng.integers(4))]) if kind == "mixed" else (lambda: kind)
    A2 = synth.pack([_ring_variant(A.ring(i), rng, pick()) for i in range(A.n)])
    B2 = synth.pack([_ring_variant(B.ring(i), rng, pick()) for i in range(B.n)])
    P, Q = dev(A, sccg), dev(B, sccg)
    P2, Q2 = dev(A2, sccg), dev(B2, sccg)  # validate=True: no status bits
    assert P2.status.cpu().tolist()[0] == 0 and Q2.status.cpu().tolist()[0] == 0
    assert torch.equal(P2.area, P.area) and torch.equal(P2.mbr, P.mbr)
    pairs = sccg.filter_pairs(P, Q)
    pairs2 = sccg.filter_pairs(P2, Q2)
    assert torch.equal(pairs, pairs2)
    for T in (64, 2048):
        ref = sccg.pixelbox(P, Q, pairs, threshold=T)
        for raster in (True, False):
            got = sccg.pixelbox(P2, Q2, pairs2, threshold=T, raster=raster)
            assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1]) and torch.equal(got[2], ref[2])
    check_batch(sccg, A2, B2, pairs2.cpu().numpy(), *sccg.pixelbox(P2, Q2, pairs2))


def test_async_overflow_sets_status(sccg, tile_sets):
    """a join that overflows the pair buffer leaves it incomplete;
    sccg_pixelbox_async then processes nothing and flags SCCG_STATUS_CAPACITY,
    so the sums are never silently wrong, and sccg_jaccard rejects them."""
    A, B = tile_sets
    P, Q = dev(A, sccg), dev(B, sccg)
    pipe = sccg.Pipeline(P, Q, cap=10, graph=False)
    s = pipe.run().cpu().tolist()
    assert s[10] & sccg.STATUS_CAPACITY and s[0] == 0
    with pytest.raises(sccg.SccgError) as e:
        sccg.jaccard(s)
    assert e.value.code == sccg.E_CAPACITY
    # an out-of-range pair index: flagged, and pixelbox(check=True) raises
    bad = torch.tensor([[0, 10**6]], dtype=torch.int32, device="cuda")
    with pytest.raises(sccg.SccgError):
        sccg.pixelbox(P, Q, bad)


def test_sums_pack_unpack_and_nccl(sccg, tile_sets):
    """Row a9 on the GPU: sccg_sums_pack / unpack equal the host mirror, and the
    packed vector goes through a real NCCL all_reduce (world size 1, also
    captured in a CUDA graph) and unpacks to the same sums."""
    import os

    import torch.distributed as dist

    from paper_1208_0277_b200 import dist as sdist

    A, B = tile_sets
    P, Q = dev(A, sccg), dev(B, sccg)
    _, _, sums = sccg.pixelbox(P, Q, sccg.filter_pairs(P, Q))
    sums[10] = 0b10101
    vec = sccg.sums_pack(sums)
    assert vec.cpu().tolist() == sdist.pack_sums(sums.cpu()).tolist()
    back = sccg.sums_unpack(vec * 3, torch.zeros_like(sums))
    assert back.cpu().tolist() == sdist.unpack_sums(vec.cpu() * 3, torch.zeros(11, dtype=torch.int64)).tolist()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29731")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        ref = sums.clone()
        out = sdist.allreduce_sums(sums.clone(), force=True)
        assert torch.equal(out, ref)
        g = torch.cuda.CUDAGraph()
        buf = sums.clone()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            sdist.allreduce_sums(buf, force=True)  # warm-up outside capture
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            sdist.allreduce_sums(buf, force=True)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(buf, ref)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_study_many_images_one_graph(sccg):
    """configs[3] on one GPU (sccg.Study): images instanced from two tile bases
    under the 8 lattice symmetries run back to back in ONE graph with shared
    derived buffers and workspaces; the accumulated sums must equal the sum of
    the oracle's sums of each image's base (every field, exact ratio units),
    replays must be identical, and the last image's per-pair (I, U) must be its
    base's."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    bases = []
    for b in range(2):
        A, B = synth.generate("tile", image=10 + b)
        pairs = oracle.join(A, B)
        ei, eu = oracle.pair_areas(A, B, pairs)
        bases.append((A, B, pairs, ei, eu, oracle.sums(A, B, pairs, ei, eu)))
    plan = bench.study_images(9, 2)
    images = []
    for im in plan:
        A, B = bases[im["base"]][:2]
        xa, oa = sccg.to_device(A.xy, A.offsets)
        xb, ob = sccg.to_device(B.xy, B.offsets)
        images.append((bench.instance_xy(xa, im["sym"], im["dx"], im["dy"]), oa,
                       bench.instance_xy(xb, im["sym"], im["dx"], im["dy"]), ob))
    study = sccg.Study(images, graph=True)  # image i + 1's prep overlapped with image i's join and PixelBox
    s1 = study.run().clone()
    s2 = study.run().clone()
    s3 = sccg.Study(images, graph=True, overlap=False).run().clone()
    torch.cuda.synchronize()
    assert torch.equal(s1, s2) and torch.equal(s1, s3)
    study.check()
    got = s1.cpu().tolist()
    keys = ["n_pairs", "n_nonzero", "sum_inter", "sum_union", "sum_area_p", "sum_area_q"]
    want = [sum(bases[im["base"]][5][k] for im in plan) for k in keys]
    assert got[:6] == want
    units = sum(int(v) << (30 * k) for k, v in enumerate(got[6:10]))
    assert units == sum(exact_ratio_units(bases[im["base"]][3], bases[im["base"]][4]) for im in plan)
    last = bases[plan[-1]["base"]]
    n = len(last[2])
    assert np.array_equal(study.pairs[:n].cpu().numpy(), last[2])
    assert np.array_equal(study.inter[:n].cpu().numpy(), last[3])
    assert np.array_equal(study.uni[:n].cpu().numpy(), last[4])


_ABLATION_CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
import oracle, synth
import paper_1208_0277_b200 as sccg
A, B = synth.generate("tile", image=2)
for sf in (1, 3):
    P = sccg.DeviceSet(*sccg.to_device(A.xy * sf, A.offsets))
    Q = sccg.DeviceSet(*sccg.to_device(B.xy * sf, B.offsets))
    pairs = sccg.filter_pairs(P, Q)
    pn = pairs.cpu().numpy()
    assert np.array_equal(pn, oracle.join(synth.PolygonSet(A.xy * sf, A.offsets), synth.PolygonSet(B.xy * sf, B.offsets)))
    for raster, split in ((False, True), (True, False)):
        pipe = sccg.Pipeline(P, Q, raster=raster, paper_split=split)
        pipe.run()
        n = pipe.check()
        ei, eu = oracle.pair_areas(synth.PolygonSet(A.xy * sf, A.offsets), synth.PolygonSet(B.xy * sf, B.offsets), pn)
        assert np.array_equal(pipe.inter[:n].cpu().numpy(), ei) and np.array_equal(pipe.uni[:n].cpu().numpy(), eu)
print("ABLATION-OK", sccg.library_path())
"""


@pytest.mark.parametrize("variant,flags", [("noopt", ["-DSCCG_NO_PDL", "-DSCCG_PREP_NO_TMA"]),
                                           ("nopdl", ["-DSCCG_NO_PDL"])])
def test_ablation_builds_match_oracle(variant, flags):
    """The Fig. 9 analog's build variants (scripts/fig9.py: prep without TMA
    staging, launches without PDL) and runtime variants (no rasters, Alg. 1's
    split order) give the oracle's pair list and per-pair areas at SF 1 and 3."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    from paper_1208_0277_b200 import build as sbuild

    lib = os.path.join(root, "paper_1208_0277_b200", f"libsccg_{variant}.so")
    sbuild.build(extra=flags, out=lib)  # rebuilt when older than any source
    env = dict(os.environ, SCCG_LIB=lib)
    r = subprocess.run([sys.executable, "-c", _ABLATION_CHILD.format(root=root)], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ABLATION-OK" in r.stdout and lib in r.stdout, r.stdout + r.stderr


def test_filter_recycled_workspaces(sccg):
    """Joins of different sizes back to back, each with a freshly allocated
    (so recycled, stale) workspace, PixelBox in between: every pair list equals
    the oracle's.  (With kernels triggering their successors at entry, a probe
    CTA once read the previous join's grid descriptor from such a workspace
    and the next join found no pairs.)"""
    A, B = synth.generate("skewed", width=8192, height=8192)
    C, D = synth.generate("tile")
    ref_ab, ref_cd = oracle.join(A, B), oracle.join(C, D)
    for it in range(4):
        P2, Q2 = dev(C, sccg), dev(D, sccg)
        assert np.array_equal(sccg.filter_pairs(P2, Q2).cpu().numpy(), ref_cd)
        P, Q = dev(A, sccg), dev(B, sccg)  # no synchronisation: prep is still running when the join starts
        pairs = sccg.filter_pairs(P, Q)
        assert np.array_equal(pairs.cpu().numpy(), ref_ab), it
        counters = torch.zeros(8, dtype=torch.int64, device="cuda")
        sccg.pixelbox(P, Q, pairs, threshold=64, counters=counters)
        assert counters[sccg.CNT_SPLITS].item() > 0


@pytest.mark.parametrize("config", ["tile", "combs", "slide"])
def test_decode_rect_exact(sccg, config):
    """sccg_decode_rect (the compact host -> device encoding) reproduces every
    vertex of the plain layout exactly, and the path from the compact form
    gives the same pairs and sums as from the plain one."""
    if config == "combs":
        A, B = combs.generate(n_pairs=64)
    else:
        A, B = synth.generate(config)
    for S in (A, B):
        enc = sccg.encode_rect(S.xy, S.offsets)
        assert enc is not None
        start, move, fv = (torch.from_numpy(a).cuda() for a in enc)
        off = torch.from_numpy(S.offsets).cuda()
        xy = sccg.decode_rect(start, move, fv, off)
        assert torch.equal(xy.cpu(), torch.from_numpy(S.xy.astype(np.int32)))
    if config == "tile":
        P0, Q0 = dev(A, sccg), dev(B, sccg)
        dec = []
        for S in (A, B):
            start, move, fv = (torch.from_numpy(a).cuda() for a in sccg.encode_rect(S.xy, S.offsets))
            off = torch.from_numpy(S.offsets).cuda()
            dec.append(sccg.DeviceSet(sccg.decode_rect(start, move, fv, off), off))
        _, _, s0 = sccg.pixelbox(P0, Q0, sccg.filter_pairs(P0, Q0))
        _, _, s1 = sccg.pixelbox(dec[0], dec[1], sccg.filter_pairs(dec[0], dec[1]))
        assert torch.equal(s0, s1)


def _packed_to_device(enc):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in enc.items()}


@pytest.mark.parametrize("config", ["tile", "combs", "slide", "edge"])
def test_decode_rect_packed_exact(sccg, config):
    """sccg_decode_rect_packed (format 2: per-ring 4/8/16-bit moves, int16 start
    deltas, offsets rebuilt on the device) reproduces the plain rings and their
    offsets exactly -- including moves of every width, wide start blocks, empty
    rings and a partial last block -- and the path from it gives the same sums."""
    if config == "combs":
        A, B = combs.generate(n_pairs=64)
        sets = (A, B)
    elif config == "edge":
        from test_abi import _rect_ring

        rng = np.random.default_rng(11)
        rings = [_rect_ring(rng, int(rng.integers(-2**30, 2**30)) if i == 300 else int(rng.integers(-9000, 9000)),
                         int(rng.integers(-5000, 5000)), int(rng.integers(0, 60)) * 2 + 3,
                         (1, 8, 9, 128, 129, 32767)[i % 6]) for i in range(777)]
        rings.append(_rect_ring(rng, 0, 0, 8189, 3))  # 8190 vertices, the largest count a head holds
        P = synth.pack(rings)
        off = np.concatenate([P.offsets[:10], P.offsets[9:300], P.offsets[299:]])  # an empty ring
        sets = ((P.xy, off),)
    else:
        A, B = synth.generate(config)
        sets = (A, B)
    for S in sets:
        xy_h, off_h = (S if isinstance(S, tuple) else (S.xy, S.offsets))
        enc = sccg.encode_rect_packed(xy_h, off_h)
        assert enc is not None
        xy, off = sccg.decode_rect_packed(_packed_to_device(enc), int(off_h[-1]))
        assert torch.equal(off.cpu(), torch.from_numpy(np.asarray(off_h, np.int64)))
        assert torch.equal(xy.cpu(), torch.from_numpy(np.asarray(xy_h, np.int32)))
    # no rings: offsets[0] = 0
    e0 = sccg.encode_rect_packed(np.zeros((0, 2), np.int32), np.zeros(1, np.int64))
    out = (torch.empty((1, 2), dtype=torch.int32, device="cuda"), torch.full((1,), 7, dtype=torch.int64, device="cuda"))
    _, off0 = sccg.decode_rect_packed(_packed_to_device(e0), 0, out=out)
    assert off0.tolist() == [0]
    if config == "tile":
        P0, Q0 = dev(A, sccg), dev(B, sccg)
        dec = [sccg.DeviceSet(*sccg.decode_rect_packed(_packed_to_device(sccg.encode_rect_packed(S.xy, S.offsets)),
                                                       int(S.offsets[-1]))) for S in (A, B)]
        _, _, s0 = sccg.pixelbox(P0, Q0, sccg.filter_pairs(P0, Q0))
        _, _, s1 = sccg.pixelbox(dec[0], dec[1], sccg.filter_pairs(dec[0], dec[1]))
        assert torch.equal(s0, s1)


@pytest.mark.parametrize("config", ["tile", "skewed", "combs", "edge"])
def test_prep_sets_packed_matches_plain(sccg, config):
    """sccg_prep_sets_packed (prep decoding the packed encoding tile by tile,
    no decode kernel): xy and offsets exactly the plain rings, and every
    derived output (MBR, area, edge counts and rebases, records and rasters,
    status) identical to sccg_prep_sets on the plain sets -- thread-path
    tiles, rings over 192 vertices (warp path), tiles too large to stage
    (combs: decoded straight to global memory), every coding class."""
    if config == "combs":
        sets = combs.generate(n_pairs=48)
    elif config == "edge":
        from test_abi import _rect_ring

        rng = np.random.default_rng(5)
        rings = [_rect_ring(rng, int(rng.integers(-9000, 9000)), int(rng.integers(-5000, 5000)),
                            int(rng.integers(2, 60)) * 2 + 2, (1, 8, 9, 128, 129, 300)[i % 6]) for i in range(600)]
        sets = (synth.pack(rings),)
    else:
        sets = synth.generate(config)
    for S in sets:
        for vlc in (True, False):
            enc = sccg.encode_rect_packed(S.xy, S.offsets, vlc=vlc)
            assert enc is not None
            ed = _packed_to_device(enc)
            xy = torch.zeros((len(S.xy), 2), dtype=torch.int32, device="cuda")
            off = torch.zeros(S.n + 1, dtype=torch.int64, device="cuda")
            D = sccg.DeviceSet(xy, off, prep=False)
            sccg.prep_sets_packed([D], [ed])
            torch.cuda.synchronize()
            assert torch.equal(off.cpu(), torch.from_numpy(np.asarray(S.offsets, np.int64)))
            assert torch.equal(xy.cpu(), torch.from_numpy(np.asarray(S.xy, np.int32)))
            R = dev(S, sccg)
            for f in ("mbr", "area", "ecount", "status"):
                assert torch.equal(getattr(D, f), getattr(R, f)), (config, vlc, f)
            assert torch.equal(D.used_edge_words(), R.used_edge_words())


def test_prep_sets_packed_empty_set(sccg):
    """A set with no rings in packed mode: offsets[0] = 0 is still written."""
    e0 = _packed_to_device(sccg.encode_rect_packed(np.zeros((0, 2), np.int32), np.zeros(1, np.int64)))
    A, _ = synth.generate("tile")
    ea = _packed_to_device(sccg.encode_rect_packed(A.xy, A.offsets))
    xy0 = torch.zeros((1, 2), dtype=torch.int32, device="cuda")
    off0 = torch.full((1,), 7, dtype=torch.int64, device="cuda")
    xya = torch.zeros((len(A.xy), 2), dtype=torch.int32, device="cuda")
    offa = torch.zeros(A.n + 1, dtype=torch.int64, device="cuda")
    D0, Da = sccg.DeviceSet(xy0[:0], off0, prep=False), sccg.DeviceSet(xya, offa, prep=False)
    sccg.prep_sets_packed([Da, D0], [ea, e0])
    torch.cuda.synchronize()
    assert off0.tolist() == [0]
    assert torch.equal(offa.cpu(), torch.from_numpy(np.asarray(A.offsets, np.int64)))


def test_streamer_fused_matches_pipeline(sccg):
    """sccg.Streamer(fused=...): the step graph's prep decodes the packed
    rings itself; every step's sums equal the device-resident Pipeline's."""
    A, B = synth.generate("tile", image=33)
    P, Q = dev(A, sccg), dev(B, sccg)
    pipe = sccg.Pipeline(P, Q, graph=False)
    pipe.run()
    torch.cuda.synchronize()
    ref = pipe.sums.cpu().tolist()
    step = sccg.PackedStep(*(sccg.encode_rect_packed(S.xy, S.offsets) for S in (A, B)))
    st = sccg.Streamer(A.n, int(A.offsets[-1]), B.n, int(B.offsets[-1]), depth=3, fused=step)
    tickets = [st.submit_step(step) for _ in range(5)]
    got = [st.result(t) for t in tickets[2:]]
    for g in got:
        assert [getattr(g, f) for f in sccg.SUMS_FIELDS] == ref


def _study_rank(rank, world, port, out):
    import os
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist

    import bench
    import paper_1208_0277_b200 as sccg
    from paper_1208_0277_b200 import dist as sdist
    import synth

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    plan = bench.study_images(7, 2)
    mine = [plan[i] for i in sdist.shard_for_rank(len(plan), world, rank)]
    bases = {b: synth.generate("tile", image=20 + b) for b in (0, 1)}
    images = []
    for im in mine:
        A, B = bases[im["base"]]
        xa, oa = sccg.to_device(A.xy, A.offsets)
        xb, ob = sccg.to_device(B.xy, B.offsets)
        images.append((bench.instance_xy(xa, im["sym"], im["dx"], im["dy"]), oa,
                       bench.instance_xy(xb, im["sym"], im["dx"], im["dy"]), ob))
    sums = sccg.Study(images).run().clone() if images else sccg.new_sums("cuda")
    sdist.allreduce_sums(sums, force=True)
    out[rank] = sums.cpu().tolist()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_study_gloo_ranks_bit_identical(sccg):
    """configs[3] over 1, 2 and 3 ranks (gloo, sharing cuda:0): LPT shards of
    the same 7 instanced images, each rank's pass one Study graph, one
    all-reduce -- the reduced sums are bit-identical for every rank count."""
    import socket

    import torch.multiprocessing as tmp

    results = {}
    for world in (1, 2, 3):
        ctx = tmp.get_context("spawn")
        mgr = ctx.Manager()
        out = mgr.dict()
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        procs = [ctx.Process(target=_study_rank, args=(r, world, port, out)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(500)
            assert p.exitcode == 0
        assert all(out[r] == out[0] for r in range(world))
        results[world] = out[0]
    assert results[1] == results[2] == results[3]
    assert results[1][10] == 0 and results[1][0] > 0


def test_streamer_matches_pipeline(sccg):
    """sccg.Streamer (packed host -> device transfer on a copy stream, decode,
    the step graph, read-back; two slots in flight): every step's sums equal
    the device-resident Pipeline's for the same sets, steps of two different
    images interleaved."""
    imgs = []
    for image in (30, 31):
        A, B = synth.generate("tile", image=image)
        P, Q = dev(A, sccg), dev(B, sccg)
        pipe = sccg.Pipeline(P, Q, graph=False)
        pipe.run()
        torch.cuda.synchronize()
        enc = [sccg.pin_packed(sccg.encode_rect_packed(S.xy, S.offsets)) for S in (A, B)]
        imgs.append((A, B, enc, pipe.sums.cpu().tolist()))
    # one Streamer per shape (slots are shaped by the first sets); same-shaped repeats of each image
    for A, B, enc, ref in imgs:
        st = sccg.Streamer(A.n, int(A.offsets[-1]), B.n, int(B.offsets[-1]))
        tickets = [st.submit(enc[0], enc[1]) for _ in range(2)]
        got = [st.result(t) for t in tickets]
        tickets = [st.submit(enc[0], enc[1]) for _ in range(2)]
        got += [st.result(t) for t in tickets]
        step = sccg.PackedStep(*(sccg.encode_rect_packed(S.xy, S.offsets) for S in (A, B)))  # one copy per step
        tickets = [st.submit_step(step) for _ in range(3)]
        got += [st.result(t) for t in tickets[1:]]
        for g in got:
            assert [getattr(g, f) for f in sccg.SUMS_FIELDS] == ref
