"""Pins for the CPU oracle (``-m "not gpu"``).

Each test ties the oracle to something other than itself (the task's rule ③):
SPEC worked examples (tests/golden/spec_examples.json, each cited), the
generator's own pixel masks (built without any ray casting), closed forms
(rectangles, combs as disjoint rectangle unions), exhaustive enumeration of tiny
polyominoes against plain set arithmetic, the identity |p n q| + |p u q| =
|p| + |q| with all four counted directly, grid symmetries, and nested-loop vs
plane-sweep joins.  A dropped term, flipped sign, wrong index or transposed
operand in oracle.c fails at least one of these.
"""
import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from synth import combs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


# ---------------------------------------------------------------- golden
def test_golden_areas(golden):
    for e in golden["areas"]:
        assert oracle.area_shoelace(e["ring"]) == e["area"], e["cite"]
        assert oracle.area_pixels(e["ring"], 0) == e["area"], e["cite"]
        assert oracle.area_pixels(e["ring"], 1) == e["area"], e["cite"]


def test_golden_pixels_and_mbrs(golden):
    for e in golden["pixels"]:
        assert oracle.pixel_in(e["ring"], *e["pixel"]) == e["inside"], e["cite"]
    for e in golden["mbrs"]:
        assert list(oracle.mbr(e["ring"])) == e["mbr"], e["cite"]


def test_golden_pairs(golden):
    for e in golden["pairs"]:
        assert oracle.area_shoelace(e["p"]) == e["area_p"], e["cite"]
        assert oracle.area_shoelace(e["q"]) == e["area_q"], e["cite"]
        for mode in (0, 1):
            assert oracle.pair(e["p"], e["q"], mode) == (e["inter"], e["union"]), e["cite"]
            assert oracle.pair(e["q"], e["p"], mode) == (e["inter"], e["union"]), e["cite"]


def test_golden_jaccard(golden):
    for e in golden["jaccard"]:
        j = oracle.jaccard(e["inter"], e["union"])
        ex = oracle.jaccard_exact(e["inter"], e["union"])
        if e["jprime_num"] is None:
            assert math.isnan(j) and ex is None, e["cite"]
        else:
            assert ex == Fraction(e["jprime_num"], e["jprime_den"]), e["cite"]
            assert j == e["jprime_num"] / e["jprime_den"], e["cite"]


# ------------------------------------------------- generator masks (no PIP)
def test_generator_masks_pin_pixel_test_and_shoelace(tile_sets):
    """The generator builds each ring by tracing a pixel mask; the oracle's ray
    casting must reproduce that mask exactly and the shoelace must equal its
    cell count (pixel areas are exact for raster polygons)."""
    for s in tile_sets:
        for i in range(s.n):
            x0, y0, m = s.masks[i]
            h, w = m.shape
            ring = s.ring(i)
            # window one pixel larger on every side: nothing leaks outside
            om = oracle.mask(ring, x0 - 1, y0 - 1, w + 2, h + 2, mode=1)
            assert om[1:-1, 1:-1].tolist() == m.tolist()
            assert om.sum() == m.sum()
            assert oracle.area_shoelace(ring) == int(m.sum())
            assert oracle.mbr(ring) == (x0, y0, x0 + w, y0 + h)


def test_plain_and_prefilter_agree(tile_sets):
    a, b = tile_sets
    for i in range(0, a.n, 7):
        x0, y0, m = a.masks[i]
        h, w = m.shape
        assert (oracle.mask(a.ring(i), x0 - 2, y0 - 2, w + 4, h + 4, 0) ==
                oracle.mask(a.ring(i), x0 - 2, y0 - 2, w + 4, h + 4, 1)).all()
    pairs = oracle.join(a, b)[::3]
    i0, u0 = oracle.pair_areas(a, b, pairs, mode=0)
    i1, u1 = oracle.pair_areas(a, b, pairs, mode=1)
    assert (i0 == i1).all() and (u0 == u1).all()


# ------------------------------------------------------------ closed forms
def _rect(x0, y0, x1, y1):
    return [[x0, y0], [x1, y0], [x1, y1], [x0, y1]]


def test_rectangle_pairs_closed_form():
    rng = np.random.default_rng(7)
    for _ in range(400):
        a = rng.integers(-20, 20, 2)
        wa = rng.integers(1, 15, 2)
        b = a + rng.integers(-16, 16, 2)
        wb = rng.integers(1, 15, 2)
        ra = _rect(a[0], a[1], a[0] + wa[0], a[1] + wa[1])
        rb = _rect(b[0], b[1], b[0] + wb[0], b[1] + wb[1])
        ow = max(0, min(a[0] + wa[0], b[0] + wb[0]) - max(a[0], b[0]))
        oh = max(0, min(a[1] + wa[1], b[1] + wb[1]) - max(a[1], b[1]))
        inter = ow * oh
        uni = wa[0] * wa[1] + wb[0] * wb[1] - inter
        assert oracle.pair(ra, rb) == (inter, uni)
        assert oracle.area_shoelace(ra) == wa[0] * wa[1]


def test_comb_closed_form():
    """Combs are disjoint rectangle unions: |A| = sum |R_i|, |A n B| =
    sum_ij |R_i n S_j| (SURVEY §8c pins), and comb area = W*b + k*w*h."""
    for two in (False, True):
        for k, w, g, h, b in [(3, 1, 1, 5, 2), (7, 2, 3, 9, 4), (12, 3, 1, 4, 1)]:
            ring, rects = combs.comb(10, -5, k, w, g, h, b, two)
            W = k * w + (k - 1) * g
            expect = W * b + k * w * h * (2 if two else 1)
            assert combs.rect_decomp_area(rects) == expect
            assert oracle.area_shoelace(ring) == expect
            assert oracle.area_pixels(ring, 0) == expect
            assert len(ring) == (8 * k - 4 if two else 4 * k)
    A, B, (RA, RB) = combs.generate(n_pairs=24, want_rects=True, max_vertices=800)
    pairs = np.stack([np.arange(24), np.arange(24)], 1).astype(np.int32)
    inter, uni = oracle.pair_areas(A, B, pairs)
    for k in range(24):
        ik = combs.rect_decomp_intersection(RA[k], RB[k])
        assert inter[k] == ik
        assert uni[k] == combs.rect_decomp_area(RA[k]) + combs.rect_decomp_area(RB[k]) - ik


# ------------------------------------------------------------- exhaustive
def _clean_polyominoes(k):
    """All k x k masks that are one simply-connected, pinch-free 4-connected
    region (the generator's clean() leaves them unchanged), with their rings."""
    out = []
    for bits in range(1, 1 << (k * k)):
        m = np.array([(bits >> i) & 1 for i in range(k * k)], np.uint8).reshape(k, k)
        ring, cleaned = synth.trace_mask(m)
        if ring is not None and (cleaned == m).all():
            out.append((m, ring))
    return out


def test_exhaustive_3x3_pairs():
    polys = _clean_polyominoes(3)
    assert len(polys) > 150
    for m, ring in polys:
        assert (oracle.mask(ring, -1, -1, 5, 5, 0)[1:4, 1:4] == m).all()
        assert oracle.mask(ring, -1, -1, 5, 5, 0).sum() == m.sum() == oracle.area_shoelace(ring)
    # bitboards on a 7x7 board: p at offset (2,2), q at (2+dx, 2+dy), |d| <= 2
    def board(m, dx, dy):
        v = 0
        for (y, x) in zip(*np.nonzero(m)):
            v |= 1 << ((y + 2 + dy) * 7 + (x + 2 + dx))
        return v

    rings_q, exp_i, exp_u, pairs = [], [], [], []
    offs = list(itertools.product(range(-2, 3), repeat=2))
    for qi, (mq, rq) in enumerate(polys):
        for dx, dy in offs:
            rings_q.append(rq + np.array([dx, dy], np.int32))
    P = synth.pack([r for _, r in polys])
    Q = synth.pack(rings_q)
    bp = [board(m, 0, 0) for m, _ in polys]
    for pi in range(len(polys)):
        for qi, (mq, _) in enumerate(polys):
            for oi, (dx, dy) in enumerate(offs):
                bq = board(mq, dx, dy)
                pairs.append((pi, qi * len(offs) + oi))
                exp_i.append(bin(bp[pi] & bq).count("1"))
                exp_u.append(bin(bp[pi] | bq).count("1"))
    pairs = np.asarray(pairs, np.int32)
    inter, uni = oracle.pair_areas(P, Q, pairs)
    assert (inter == np.asarray(exp_i)).all()
    assert (uni == np.asarray(exp_u)).all()


def test_touches_rectangles_closed_form():
    """ST_Touches (R21) of two rectangles: their closed boxes meet and
    their open boxes do not -- interval arithmetic, no pixels."""
    rng = np.random.default_rng(41)
    for _ in range(400):
        ax, ay, bx, by = (int(v) for v in rng.integers(0, 12, 4))
        aw, ah, bw, bh = (int(v) for v in rng.integers(1, 6, 4))
        A, B = _rect(ax, ay, ax + aw, ay + ah), _rect(bx, by, bx + bw, by + bh)
        closed = ax <= bx + bw and bx <= ax + aw and ay <= by + bh and by <= ay + ah
        opened = ax < bx + bw and bx < ax + aw and ay < by + bh and by < ay + ah
        assert oracle.touches(A, B) == (closed and not opened), (A, B)
        assert oracle.touches(B, A) == oracle.touches(A, B)
    # the P:277 literal rule calls identical / contained-with-shared-edge rings
    # touching; they overlap, so they do not touch (R21)
    assert not oracle.touches(_rect(0, 0, 2, 2), _rect(0, 0, 2, 2))
    assert not oracle.touches(_rect(0, 0, 2, 2), _rect(0, 0, 2, 1))


def test_touches_exhaustive_polyominoes_and_symmetry():
    """Pairs of clean 3x3 polyominoes at offsets in [-3, 3]^2: touches iff the
    cell sets are disjoint and the 8-neighbourhood of one meets the other
    (bitboards); invariant under the 8 grid symmetries."""
    polys = _clean_polyominoes(3)[::2]
    B = 11

    def board(m, dx, dy):
        v = 0
        for (y, x) in zip(*np.nonzero(m)):
            v |= 1 << ((int(y) + 4 + dy) * B + (int(x) + 4 + dx))
        return v

    def dilate(v):
        out = 0
        for y in range(B):
            for x in range(B):
                if v >> (y * B + x) & 1:
                    for dy in (-1, 0, 1):
                        for dx in (-1, 0, 1):
                            if 0 <= y + dy < B and 0 <= x + dx < B:
                                out |= 1 << ((y + dy) * B + (x + dx))
        return out

    offs = list(itertools.product(range(-3, 4), repeat=2))
    for mp, rp in polys:
        bp = board(mp, 0, 0)
        dp = dilate(bp)
        for mq, rq in polys[::3]:
            for dx, dy in offs:
                bq = board(mq, dx, dy)
                want = (bp & bq) == 0 and (dp & bq) != 0
                got = oracle.touches(rp, rq + np.array([dx, dy], np.int32))
                assert got == want, (rp.tolist(), rq.tolist(), dx, dy)
    rng = np.random.default_rng(43)
    for _ in range(60):
        (mp, rp), (mq, rq) = polys[int(rng.integers(len(polys)))], polys[int(rng.integers(len(polys)))]
        rq = rq + np.array([int(v) for v in rng.integers(-3, 4, 2)], np.int32)
        t = oracle.touches(rp, rq)
        for sx, sy, sw in itertools.product((1, -1), (1, -1), (False, True)):
            f = lambda r: (r[:, ::-1] if sw else r) * np.array([sx, sy], np.int32)
            assert oracle.touches(f(rp), f(rq)) == t


def test_exhaustive_4x4_single():
    polys = _clean_polyominoes(4)
    assert len(polys) > 5000
    for m, ring in polys:
        om = oracle.mask(ring, -1, -1, 6, 6, 1)
        assert (om[1:5, 1:5] == m).all() and om.sum() == m.sum()
        assert oracle.area_shoelace(ring) == m.sum()


# ------------------------------------------------------ invariants / symmetry
def test_union_identity_counted_directly(tile_sets):
    """|p n q| + |p u q| = |p| + |q| with all four counted pixel by pixel."""
    a, b = tile_sets
    pairs = oracle.join(a, b)
    inter, uni = oracle.pair_areas(a, b, pairs, mode=0)
    ap = np.array([oracle.area_pixels(a.ring(i), 0) for i in range(a.n)])
    aq = np.array([oracle.area_pixels(b.ring(i), 0) for i in range(b.n)])
    assert (inter + uni == ap[pairs[:, 0]] + aq[pairs[:, 1]]).all()
    assert (inter <= np.minimum(ap[pairs[:, 0]], aq[pairs[:, 1]])).all()
    assert (uni >= np.maximum(ap[pairs[:, 0]], aq[pairs[:, 1]])).all()
    assert (inter > 0).sum() > 0.8 * len(pairs)


D4 = [
    lambda x, y: (x, y), lambda x, y: (-y, x), lambda x, y: (-x, -y), lambda x, y: (y, -x),
    lambda x, y: (-x, y), lambda x, y: (x, -y), lambda x, y: (y, x), lambda x, y: (-y, -x),
]


def test_grid_symmetries_translation_scale(tile_sets):
    a, b = tile_sets
    pairs = oracle.join(a, b)[:150]
    base_i, base_u = oracle.pair_areas(a, b, pairs)
    for k, (p, q) in enumerate(pairs):
        rp, rq = a.ring(int(p)).astype(np.int64), b.ring(int(q)).astype(np.int64)
        assert oracle.pair(rq, rp) == (base_i[k], base_u[k])  # symmetry
        for T in D4:
            tp = np.array([T(x, y) for x, y in rp], np.int32)
            tq = np.array([T(x, y) for x, y in rq], np.int32)
            assert oracle.pair(tp, tq) == (base_i[k], base_u[k])
        d = np.array([-1234, 777])
        assert oracle.pair(rp + d, rq + d) == (base_i[k], base_u[k])  # translation
        if k % 10 == 0:
            for s in (2, 3):
                assert oracle.pair(rp * s, rq * s) == (base_i[k] * s * s, base_u[k] * s * s)  # scale law
    # idempotence
    for i in range(0, a.n, 25):
        ar = oracle.area_shoelace(a.ring(i))
        assert oracle.pair(a.ring(i), a.ring(i)) == (ar, ar)


# -------------------------------------------------------------------- join
def test_join_nested_equals_sweep_and_transpose(tile_sets):
    a, b = tile_sets
    s = oracle.join(a, b, "sweep")
    n = oracle.join(a, b, "nested")
    assert s.tolist() == n.tolist()
    t = oracle.join(b, a, "sweep")
    assert sorted(t[:, ::-1].tolist()) == s.tolist()
    keys = s[:, 0].astype(np.int64) * (1 << 32) + s[:, 1]
    assert (np.diff(keys) > 0).all()


def test_join_random_boxes_half_open():
    rng = np.random.default_rng(3)
    for trial in range(30):
        n, m = rng.integers(1, 60, 2)
        def boxes(k):
            lo = rng.integers(0, 40, (k, 2))
            wh = rng.integers(1, 12, (k, 2))
            return np.concatenate([lo, lo + wh], 1).astype(np.int32)
        bp, bq = boxes(n), boxes(m)
        got = oracle.join_mbrs(bp, bq, "sweep").tolist()
        exp = [[i, j] for i in range(n) for j in range(m)
               if bp[i, 0] < bq[j, 2] and bq[j, 0] < bp[i, 2] and bp[i, 1] < bq[j, 3] and bq[j, 1] < bp[i, 3]]
        assert got == exp
    # touching boxes share no pixel: no pair (reading R4)
    assert oracle.join_mbrs(np.array([[0, 0, 2, 2]], np.int32), np.array([[2, 0, 4, 2]], np.int32)).shape[0] == 0


# ----------------------------------------------------------------- Eq. (1)
def test_jaccard_exact_and_edge_cases(tile_sets):
    a, b = tile_sets
    pairs = oracle.join(a, b)
    inter, uni = oracle.pair_areas(a, b, pairs)
    j = oracle.jaccard(inter, uni)
    ex = oracle.jaccard_exact(inter, uni)
    assert abs(j - float(ex)) <= 1e-15 * float(ex)
    # identical sets -> exactly 1
    pa = oracle.join(a, a)
    ia, ua = oracle.pair_areas(a, a, pa)
    # pixel sets within one segmentation are disjoint, so only (p, p) has I > 0
    assert oracle.jaccard(ia, ua) == 1.0
    self_pairs = pa[pa[:, 0] == pa[:, 1]]
    i2, u2 = oracle.pair_areas(a, a, self_pairs)
    assert oracle.jaccard(i2, u2) == 1.0
    # disjoint sets -> none
    far = synth.pack([a.ring(i) + np.array([10**6, 0], np.int32) for i in range(a.n)])
    assert len(oracle.join(a, far)) == 0
    assert math.isnan(oracle.jaccard([], []))


def test_sums_fields(tile_sets):
    a, b = tile_sets
    pairs = oracle.join(a, b)
    inter, uni = oracle.pair_areas(a, b, pairs)
    s = oracle.sums(a, b, pairs, inter, uni)
    nz = inter > 0
    assert s["n_pairs"] == len(pairs) and s["n_nonzero"] == int(nz.sum())
    # all-pairs check: sum|p| + sum|q| - sum I = sum over all pairs of U
    assert s["sum_area_p"] + s["sum_area_q"] - s["sum_inter"] == int(uni.sum())


def test_missing_polygons(tile_sets):
    a, b = tile_sets
    pa = oracle.join(a, a)
    ia, _ = oracle.pair_areas(a, a, pa)
    assert oracle.missing(a.n, pa, ia, 0) == 0 and oracle.missing(a.n, pa, ia, 1) == 0  # identical sets
    pairs = oracle.join(a, b)
    inter, _ = oracle.pair_areas(a, b, pairs)
    ma, mb = oracle.missing(a.n, pairs, inter, 0), oracle.missing(b.n, pairs, inter, 1)
    # set B drops ~5 % of A's nuclei (synth recipe): A has about that many missing
    assert 0.02 * a.n < ma < 0.10 * a.n and 0 <= mb < 0.15 * b.n
    assert oracle.missing(7, np.zeros((0, 2)), [], 0) == 7


# ------------------------------------------- closed join, missing, contains, report
def test_join_closed_pinned_by_lattice_points():
    """The closed-box join (oracle_join_nested_closed, the ST_Touches
    candidates) against brute force on lattice points: two closed integer boxes
    meet iff some integer point lies in both -- touching sides and corners
    included, gaps excluded."""
    rng = np.random.default_rng(41)
    for trial in range(25):
        n, m = (int(v) for v in rng.integers(1, 25, 2))

        def boxes(k):
            lo = rng.integers(0, 16, (k, 2))
            wh = rng.integers(1, 6, (k, 2))
            return np.concatenate([lo, lo + wh], 1).astype(np.int32)

        bp, bq = boxes(n), boxes(m)
        pts = lambda b: {(x, y) for x in range(b[0], b[2] + 1) for y in range(b[1], b[3] + 1)}
        sp, sq = [pts(b) for b in bp], [pts(b) for b in bq]
        exp = [[i, j] for i in range(n) for j in range(m) if sp[i] & sq[j]]
        assert oracle.join_mbrs(bp, bq, "closed").tolist() == exp
    side = np.array([[0, 0, 2, 2]], np.int32)
    assert oracle.join_mbrs(side, np.array([[2, 0, 4, 2]], np.int32), "closed").tolist() == [[0, 0]]  # shared side
    assert oracle.join_mbrs(side, np.array([[2, 2, 3, 3]], np.int32), "closed").tolist() == [[0, 0]]  # corner
    assert oracle.join_mbrs(side, np.array([[3, 0, 4, 2]], np.int32), "closed").shape[0] == 0  # gap


def _sq(x, y, w, h):
    return [[x, y], [x + w, y], [x + w, y + h], [x, y + h]]


def test_missing_hand_built():
    """P:63 missing polygons on a hand-built pair of sets with known answers:
    P = five squares; Q matches square 0 exactly, splits square 1 into two
    halves, drops square 2, overlaps square 3 and adds a spurious far square,
    and only touches square 4 (a shared side: no common pixel)."""
    P = synth.pack([_sq(0, 0, 4, 4), _sq(10, 0, 4, 4), _sq(20, 0, 4, 4), _sq(30, 0, 4, 4), _sq(40, 0, 4, 4)])
    Q = synth.pack([_sq(0, 0, 4, 4), _sq(10, 0, 2, 4), _sq(12, 0, 2, 4), _sq(31, 1, 4, 4), _sq(100, 100, 3, 3),
                    _sq(44, 0, 2, 4)])
    for kind in ("sweep", "closed"):
        pairs = oracle.join(P, Q, kind)
        inter, _ = oracle.pair_areas(P, Q, pairs)
        assert oracle.missing(P.n, pairs, inter, 0) == 2  # squares 2 and 4
        assert oracle.missing(Q.n, pairs, inter, 1) == 2  # the spurious and the touching square
    assert oracle.join(P, Q, "closed").tolist() == [[0, 0], [1, 1], [1, 2], [3, 3], [4, 5]]


def test_contains_rectangles_and_polyominoes():
    """ST_Contains on the pixel model, pinned by interval containment of
    rectangles (closed form) and by bitboard subset tests on all pairs of clean
    3x3 polyominoes at offsets in [-1, 1]^2."""
    rng = np.random.default_rng(43)
    for _ in range(300):
        a = [int(v) for v in rng.integers(0, 10, 2)] + [int(v) for v in rng.integers(1, 8, 2)]
        b = [int(v) for v in rng.integers(0, 10, 2)] + [int(v) for v in rng.integers(1, 8, 2)]
        inside = lambda u, v: u[0] <= v[0] and v[0] + v[2] <= u[0] + u[2] and u[1] <= v[1] and v[1] + v[3] <= u[1] + u[3]
        assert oracle.contains(_sq(*a), _sq(*b)) == inside(a, b)
    polys = []
    for bits in range(1, 512):
        m = np.array([(bits >> i) & 1 for i in range(9)], np.uint8).reshape(3, 3)
        ring, cleaned = synth.trace_mask(m)
        if ring is not None and (cleaned == m).all():
            polys.append((ring, bits))
    cells = lambda bits, dx, dy: {(i % 3 + dx, i // 3 + dy) for i in range(9) if (bits >> i) & 1}
    for (ra, ba), (rb, bb) in itertools.product(polys[::4], polys[::5]):
        for dx, dy in itertools.product((-1, 0, 1), repeat=2):
            got = oracle.contains(ra, rb + np.array([dx, dy], np.int32))
            assert got == (cells(bb, dx, dy) <= cells(ba, 0, 0)), (ba, bb, dx, dy)


def test_report_hand_built_and_totals(tile_sets):
    """The per-tile report (reading R22) on a hand-built 2 x 2
    grid with known per-tile answers, and on the tile sets: the tiles add up to
    the global sums, J' and missing counts (each pinned on its own)."""
    P = synth.pack([_sq(0, 0, 4, 4), _sq(10, 0, 4, 4), _sq(60, 5, 4, 4), _sq(5, 60, 2, 2)])
    Q = synth.pack([_sq(1, 1, 4, 4), _sq(10, 0, 4, 4), _sq(58, 5, 4, 2), _sq(90, 90, 2, 2)])
    pairs = oracle.join(P, Q)
    assert pairs.tolist() == [[0, 0], [1, 1], [2, 2]]
    inter, uni = oracle.pair_areas(P, Q, pairs)
    assert inter.tolist() == [9, 16, 4] and uni.tolist() == [23, 16, 20]
    rows = oracle.report(P, Q, pairs, inter, uni, (0, 0, 50, 50, 2, 2))
    f = {k: i for i, k in enumerate(oracle.REPORT_FIELDS)}
    # tile 0 (x < 50, y < 50): pairs (0, 0), (1, 1); tile 1: pair (2, 2) (p = square at x 60); tile 2: P's
    # square at (5, 60), missing; tile 3: Q's far square, missing
    assert rows[:, f["n_pairs"]].tolist() == [2, 1, 0, 0]
    assert rows[:, f["n_nonzero"]].tolist() == [2, 1, 0, 0]
    assert rows[:, f["sum_inter"]].tolist() == [25, 4, 0, 0]
    assert rows[:, f["sum_union"]].tolist() == [39, 20, 0, 0]
    assert rows[:, f["n_poly_p"]].tolist() == [2, 1, 1, 0] and rows[:, f["n_poly_q"]].tolist() == [2, 1, 0, 1]
    assert rows[:, f["missing_p"]].tolist() == [0, 0, 1, 0] and rows[:, f["missing_q"]].tolist() == [0, 0, 0, 1]
    units = lambda r: sum(int(r[f["limb0"] + k]) << (30 * k) for k in range(4))
    assert units(rows[0]) == int(Fraction(9 / 23) * (1 << 116)) + (1 << 116)  # 9/23 and exactly 1
    assert units(rows[1]) == int(Fraction(4 / 20) * (1 << 116))
    # tile sets over a 3 x 3 grid: the tiles add up to the global totals
    a, b = tile_sets
    pairs = oracle.join(a, b)
    inter, uni = oracle.pair_areas(a, b, pairs)
    rows = oracle.report(a, b, pairs, inter, uni, (0, 0, 1500, 1500, 3, 3))
    s = oracle.sums(a, b, pairs, inter, uni)
    for k in ("n_pairs", "n_nonzero", "sum_inter", "sum_union", "sum_area_p", "sum_area_q"):
        assert int(rows[:, f[k]].sum()) == s[k], k
    assert int(rows[:, f["missing_p"]].sum()) == oracle.missing(a.n, pairs, inter, 0)
    assert int(rows[:, f["missing_q"]].sum()) == oracle.missing(b.n, pairs, inter, 1)
    assert int(rows[:, f["n_poly_p"]].sum()) == a.n and int(rows[:, f["n_poly_q"]].sum()) == b.n
    tot = sum(units(r) for r in rows)
    assert abs(Fraction(tot, 1 << 116) / s["n_nonzero"] - oracle.jaccard_exact(inter, uni)) < Fraction(1, 10**12)
