"""CPU oracle for the SCCG / PixelBox hot path (arXiv 1208.0277).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  It shares no code with ``paper_1208_0277_b200`` and is never called by
the product path.

What it computes, each the plain definition from PAPER.md (citations are
``P:<line>`` of /root/reference/PAPER.md; readings R1..R12 are listed in
DESIGN.md):

* ``pixel_in`` / ``mask`` -- even-odd ray casting from the pixel center
  (§3.1), textbook PNPOLY in ``oracle.c``.
* ``area_shoelace`` -- A = 1/2 |sum x_i y_{i+1} - x_{i+1} y_i| (§3.2).
* ``pair_areas`` -- |p n q| and |p u q| counted pixel by pixel over the pair's
  bounding region (§3.1).  The union is counted directly, not derived.
* ``join`` -- every (p, q) with overlapping half-open MBRs (the ``&&`` filter,
  §2.2, reading R4), nested loop or plane sweep, sorted by (p, q).
* ``jaccard`` -- J' of Eq. 1 (§2.1): the mean of r = I/U over the
  pairs with I != 0 (a multiset over pairs, reading R9), by ``math.fsum`` of
  the IEEE-rounded ratios and, for checks, exactly with ``fractions``.
* ``sums`` -- the integer totals the C-ABI reports in ``sccg_sums``.
* ``touches`` -- ST_Touches (reading R21) on the pixel model: no common
  pixel and some pixel of each polygon sharing at least a corner.
* ``contains`` -- ST_Contains on the pixel model: every pixel of the
  contained ring is a pixel of the other (checked pixel by pixel over its MBR).
* ``report`` -- the per-tile SimilarityReport (reading R22 for
  the tile of a polygon / pair), from per-pair areas.

Pins (tests/test_oracle.py) tie each of these to something other than itself:
generator masks, the shoelace closed form, rectangles / combs / the SPEC
worked examples, exhaustive tiny polyominoes, the identity I + U = |p| + |q|,
grid symmetries, nested-loop vs sweep.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_i32p = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile oracle.c (gcc -O2, no fast-math, -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-o", tmp, _SRC,
             "-lm", "-lpthread"]
        )
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            vp, i64, i32, dbl, cint = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_int
            lib.oracle_pip.argtypes = [vp, i64, dbl, dbl]
            lib.oracle_pip.restype = cint
            lib.oracle_pixel_in.argtypes = [vp, i64, i32, i32]
            lib.oracle_pixel_in.restype = cint
            lib.oracle_area_shoelace.argtypes = [vp, i64]
            lib.oracle_area_shoelace.restype = i64
            lib.oracle_mbr.argtypes = [vp, i64, vp]
            lib.oracle_mbr.restype = None
            lib.oracle_mask.argtypes = [vp, i64, i32, i32, i32, i32, vp, cint]
            lib.oracle_mask.restype = i64
            lib.oracle_area_pixels.argtypes = [vp, i64, cint]
            lib.oracle_area_pixels.restype = i64
            lib.oracle_pair.argtypes = [vp, i64, vp, i64, vp, vp, cint]
            lib.oracle_pair.restype = None
            lib.oracle_pairs.argtypes = [vp, vp, vp, vp, vp, i64, vp, vp, cint, cint]
            lib.oracle_pairs.restype = None
            lib.oracle_set_props.argtypes = [vp, vp, i64, vp, vp]
            lib.oracle_set_props.restype = None
            lib.oracle_join_nested.argtypes = [vp, i64, vp, i64, vp, i64]
            lib.oracle_join_nested.restype = i64
            lib.oracle_join_sweep.argtypes = [vp, i64, vp, i64, vp, i64]
            lib.oracle_join_sweep.restype = i64
            lib.oracle_join_nested_closed.argtypes = [vp, i64, vp, i64, vp, i64]
            lib.oracle_join_nested_closed.restype = i64
            lib.oracle_touches.argtypes = [vp, i64, vp, i64]
            lib.oracle_touches.restype = cint
            _lib = lib
    return _lib


def _ring(r) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(r, dtype=np.int32).reshape(-1, 2))


# ----------------------------------------------------------- single polygons
def pixel_in(ring, x: int, y: int) -> bool:
    """Pixel (x, y) = cell [x, x+1) x [y, y+1) inside the ring."""
    r = _ring(ring)
    return bool(_load().oracle_pixel_in(r.ctypes.data, len(r), x, y))


def area_shoelace(ring) -> int:
    r = _ring(ring)
    return int(_load().oracle_area_shoelace(r.ctypes.data, len(r)))


def mbr(ring) -> tuple[int, int, int, int]:
    r = _ring(ring)
    out = np.zeros(4, np.int32)
    _load().oracle_mbr(r.ctypes.data, len(r), out.ctypes.data)
    return tuple(int(v) for v in out)


def mask(ring, x0: int, y0: int, w: int, h: int, mode: int = 1) -> np.ndarray:
    """uint8[h, w] pixel mask over the window; mode 0 plain, 1 row prefilter."""
    r = _ring(ring)
    out = np.zeros((h, w), np.uint8)
    _load().oracle_mask(r.ctypes.data, len(r), x0, y0, w, h, out.ctypes.data, mode)
    return out


def area_pixels(ring, mode: int = 1) -> int:
    r = _ring(ring)
    return int(_load().oracle_area_pixels(r.ctypes.data, len(r), mode))


def pair(ring_p, ring_q, mode: int = 1) -> tuple[int, int]:
    """(|p n q|, |p u q|), both counted pixel by pixel."""
    a, b = _ring(ring_p), _ring(ring_q)
    i, u = ctypes.c_int64(), ctypes.c_int64()
    _load().oracle_pair(a.ctypes.data, len(a), b.ctypes.data, len(b), ctypes.byref(i), ctypes.byref(u), mode)
    return int(i.value), int(u.value)


# ------------------------------------------------------------------- sets
def set_props(pset) -> tuple[np.ndarray, np.ndarray]:
    """Shoelace areas int64[n] and MBRs int32[n, 4] of a PolygonSet."""
    n = pset.n
    area = np.zeros(n, np.int64)
    m = np.zeros((n, 4), np.int32)
    xy = np.ascontiguousarray(pset.xy, np.int32)
    off = np.ascontiguousarray(pset.offsets, np.int64)
    _load().oracle_set_props(xy.ctypes.data, off.ctypes.data, n, area.ctypes.data, m.ctypes.data)
    return area, m


def pair_areas(pset, qset, pairs, threads: int | None = None, mode: int = 1) -> tuple[np.ndarray, np.ndarray]:
    """Per-pair (I, U) int64 arrays for pairs int32[n, 2] (input order)."""
    pairs = np.ascontiguousarray(np.asarray(pairs, np.int32).reshape(-1, 2))
    n = len(pairs)
    inter = np.zeros(n, np.int64)
    uni = np.zeros(n, np.int64)
    if n:
        xp = np.ascontiguousarray(pset.xy, np.int32)
        xq = np.ascontiguousarray(qset.xy, np.int32)
        op = np.ascontiguousarray(pset.offsets, np.int64)
        oq = np.ascontiguousarray(qset.offsets, np.int64)
        t = threads if threads is not None else (os.cpu_count() or 1)
        t = max(1, min(t, n))
        _load().oracle_pairs(xp.ctypes.data, op.ctypes.data, xq.ctypes.data, oq.ctypes.data, pairs.ctypes.data, n,
                             inter.ctypes.data, uni.ctypes.data, t, mode)
    return inter, uni


def join(pset, qset, method: str = "sweep") -> np.ndarray:
    """Candidate pairs int32[n, 2] with overlapping half-open MBRs, sorted by (p, q)."""
    _, mp = set_props(pset)
    _, mq = set_props(qset)
    return join_mbrs(mp, mq, method)


def join_mbrs(mp: np.ndarray, mq: np.ndarray, method: str = "sweep") -> np.ndarray:
    """method: "sweep" / "nested" (half-open boxes, R4) or "closed" (touching
    boxes pair too; nested loop -- the ST_Touches candidates)."""
    lib = _load()
    fn = {"sweep": lib.oracle_join_sweep, "nested": lib.oracle_join_nested,
          "closed": lib.oracle_join_nested_closed}[method]
    mp = np.ascontiguousarray(mp, np.int32)
    mq = np.ascontiguousarray(mq, np.int32)
    n = fn(mp.ctypes.data, len(mp), mq.ctypes.data, len(mq), None, 0)
    out = np.zeros((max(n, 1), 2), np.int32)
    n2 = fn(mp.ctypes.data, len(mp), mq.ctypes.data, len(mq), out.ctypes.data, n)
    assert n2 == n
    return out[:n]


def touches(ring_p, ring_q) -> bool:
    """ST_Touches (reading R21): no common pixel, and some pixel of p
    and some pixel of q share at least a corner (closed squares meet)."""
    a, b = _ring(ring_p), _ring(ring_q)
    return bool(_load().oracle_touches(a.ctypes.data, len(a), b.ctypes.data, len(b)))


def touches_pairs(pset, qset, pairs) -> np.ndarray:
    """uint8 [n]: touches(p, q) for each pair of a batch."""
    pairs = np.asarray(pairs, np.int64).reshape(-1, 2)
    out = np.zeros(len(pairs), np.uint8)
    for k, (p, q) in enumerate(pairs):
        out[k] = touches(pset.ring(int(p)), qset.ring(int(q)))
    return out


# ---------------------------------------------------------------- Eq. (1)
def jaccard(inter, uni) -> float:
    """J' (Eq. 1): mean of r = I/U over pairs with I != 0; NaN if none.

    r is the IEEE binary64 quotient (round to nearest); the mean is the
    correctly rounded sum (math.fsum) divided by the count."""
    inter = np.asarray(inter, np.int64)
    uni = np.asarray(uni, np.int64)
    keep = inter != 0
    if not keep.any():
        return float("nan")
    r = [int(i) / int(u) for i, u in zip(inter[keep], uni[keep])]
    return math.fsum(r) / len(r)


def jaccard_exact(inter, uni) -> Fraction | None:
    """J' with exact rational arithmetic (for the 1e-12 check); None if empty.
    The ratios are grouped by their union first (sum_u (sum I) / u: the same
    rational, with one Fraction addition per distinct u instead of per pair)."""
    by_u: dict[int, int] = {}
    n = 0
    for i, u in zip(np.asarray(inter, np.int64).tolist(), np.asarray(uni, np.int64).tolist()):
        if i != 0:
            by_u[u] = by_u.get(u, 0) + i
            n += 1
    if not n:
        return None
    return sum((Fraction(i, u) for u, i in sorted(by_u.items())), Fraction(0)) / n


def sums(pset, qset, pairs, inter, uni) -> dict:
    """Integer totals over a pair batch, as reported in ``sccg_sums``:
    n_pairs, n_nonzero, sum_inter, sum_union (over I > 0), sum_area_p and
    sum_area_q (shoelace areas, with pair multiplicity)."""
    pairs = np.asarray(pairs, np.int64).reshape(-1, 2)
    inter = np.asarray(inter, np.int64)
    uni = np.asarray(uni, np.int64)
    ap, _ = set_props(pset)
    aq, _ = set_props(qset)
    nz = inter != 0
    return dict(
        n_pairs=int(len(pairs)),
        n_nonzero=int(nz.sum()),
        sum_inter=int(inter.sum()),
        sum_union=int(uni[nz].sum()),
        sum_area_p=int(ap[pairs[:, 0]].sum()) if len(pairs) else 0,
        sum_area_q=int(aq[pairs[:, 1]].sum()) if len(pairs) else 0,
    )


def missing(n: int, pairs, inter, side: int) -> int:
    """Missing polygons: polygons of a set (side 0 = P, 1 = Q) of size n
    that appear in no pair with |p n q| != 0."""
    pairs = np.asarray(pairs, np.int64).reshape(-1, 2)
    inter = np.asarray(inter, np.int64)
    seen = set(pairs[inter != 0, side].tolist())
    return int(n - len(seen))


# ------------------------------------------------------------ ST_Contains
def contains(ring_p, ring_q) -> bool:
    """ST_Contains on the pixel model: q is non-empty and every pixel
    of q (scanned over q's MBR) is a pixel of p."""
    x0, y0, x1, y1 = mbr(ring_q)
    if x1 <= x0 or y1 <= y0:
        return False
    mq = mask(ring_q, x0, y0, x1 - x0, y1 - y0)
    if not mq.any():
        return False
    mp = mask(ring_p, x0, y0, x1 - x0, y1 - y0)
    return bool(((mq == 1) <= (mp == 1)).all())


def contains_pairs(pset, qset, pairs) -> np.ndarray:
    """uint8 [n]: bit 0 = p contains q, bit 1 = q contains p."""
    pairs = np.asarray(pairs, np.int64).reshape(-1, 2)
    out = np.zeros(len(pairs), np.uint8)
    for k, (p, q) in enumerate(pairs):
        rp, rq = pset.ring(int(p)), qset.ring(int(q))
        out[k] = (1 if contains(rp, rq) else 0) | (2 if contains(rq, rp) else 0)
    return out


# ------------------------------------------------------------------ report
REPORT_FIELDS = ("n_pairs", "n_nonzero", "sum_inter", "sum_union", "sum_area_p", "sum_area_q", "limb0", "limb1",
                 "limb2", "limb3", "status", "n_poly_p", "n_poly_q", "missing_p", "missing_q")


def ratio_units(i: int, u: int) -> int:
    """RN64(I/U) as an exact integer count of 2^-116 (reading R12): Python's
    int / int is the correctly rounded binary64 quotient."""
    return int(Fraction(int(i) / int(u)) * (1 << 116))


def tile_index(xlo: int, ylo: int, tiling) -> int:
    """Reading R22: the tile holding (xlo, ylo), clamped into the grid."""
    x0, y0, tw, th, ntx, nty = tiling
    tx = min(max((xlo - x0) // tw, 0), ntx - 1)
    ty = min(max((ylo - y0) // th, 0), nty - 1)
    return ty * ntx + tx


def report(pset, qset, pairs, inter, uni, tiling) -> np.ndarray:
    """Per-tile SimilarityReport rows int64 [ntx * nty, 15] (REPORT_FIELDS):
    a pair counts in the tile of its p, a polygon in its own tile; missing =
    polygons in no pair with I != 0; ratio limbs = the exact sum of
    RN64(I/U) over the tile's pairs with I != 0 in 30-bit limbs (Eq. 1)."""
    pairs = np.asarray(pairs, np.int64).reshape(-1, 2)
    inter = np.asarray(inter, np.int64)
    uni = np.asarray(uni, np.int64)
    ap, mp = set_props(pset)
    aq, mq = set_props(qset)
    nt = tiling[4] * tiling[5]
    rows = [[0] * len(REPORT_FIELDS) for _ in range(nt)]
    units = [0] * nt
    hit_p, hit_q = set(), set()
    for (p, q), i, u in zip(pairs.tolist(), inter.tolist(), uni.tolist()):
        t = tile_index(int(mp[p, 0]), int(mp[p, 1]), tiling)
        r = rows[t]
        r[0] += 1
        r[2] += i
        r[4] += int(ap[p])
        r[5] += int(aq[q])
        if i != 0:
            r[1] += 1
            r[3] += u
            units[t] += ratio_units(i, u)
            hit_p.add(p)
            hit_q.add(q)
    for t in range(nt):
        for k in range(4):
            rows[t][6 + k] = (units[t] >> (30 * k)) & ((1 << 30) - 1) if k < 3 else units[t] >> 90
    for side, (m, hit) in enumerate(((mp, hit_p), (mq, hit_q))):
        for i in range(len(m)):
            t = tile_index(int(m[i, 0]), int(m[i, 1]), tiling)
            rows[t][11 + side] += 1
            if i not in hit:
                rows[t][13 + side] += 1
    return np.array(rows, np.int64).reshape(nt, len(REPORT_FIELDS))
