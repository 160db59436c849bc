"""Highly concave rectilinear combs (config 5, "adversarial shapes").

INPUT GENERATION ONLY (no method arithmetic).  A comb is built as a union of
disjoint axis-aligned rectangles -- a base bar plus k teeth (optionally on both
sides) -- and its ring is written down vertex by vertex, so every pair also
carries its rectangle decomposition for the closed-form pin
``|A n B| = sum_i sum_j |R_i n S_j|`` used in tests.

Shape: base [x0, x0+W) x [y0, y0+b) with W = k*w + (k-1)*g; tooth i is
[x0 + i*(w+g), x0 + i*(w+g) + w) x [y0+b, y0+b+h) (and, two-sided, mirrored
below the base).  One-sided rings have 4k vertices.
"""
from __future__ import annotations

import numpy as np


def comb(x0: int, y0: int, k: int, w: int, g: int, h: int, b: int, two_sided: bool = False):
    """Return (ring int32[V, 2] CCW, rects [(x0, y0, x1, y1)] disjoint)."""
    p = w + g
    W = k * w + (k - 1) * g
    hb = h if two_sided else 0  # teeth below the base
    yb0, yb1 = y0 + hb, y0 + hb + b  # base bar
    rects = [(x0, yb0, x0 + W, yb1)]
    for i in range(k):
        tx = x0 + i * p
        rects.append((tx, yb1, tx + w, yb1 + h))
        if two_sided:
            rects.append((tx, y0, tx + w, yb0))
    # the ring, vertex by vertex (vectorised): bottom side left to right, then
    # the top side right to left; the left and right ends are straight columns
    txs = x0 + np.arange(k, dtype=np.int64) * p
    if two_sided:  # per tooth i: (tx, y0), (tx + w, y0), then (tx + w, yb0), (tx + p, yb0) between teeth
        bot = np.empty((k, 4, 2), np.int64)
        bot[:, 0] = np.stack([txs, np.full(k, y0)], 1)
        bot[:, 1] = np.stack([txs + w, np.full(k, y0)], 1)
        bot[:, 2] = np.stack([txs + w, np.full(k, yb0)], 1)
        bot[:, 3] = np.stack([txs + p, np.full(k, yb0)], 1)
        bot = bot.reshape(-1, 2)[:-2]
    else:
        bot = np.array([(x0, yb0), (x0 + W, yb0)], np.int64)
    rt = txs[::-1]  # top side, right to left: (tx + w, top), (tx, top), then (tx, yb1), (tx - g, yb1) between teeth
    top = np.empty((k, 4, 2), np.int64)
    top[:, 0] = np.stack([rt + w, np.full(k, yb1 + h)], 1)
    top[:, 1] = np.stack([rt, np.full(k, yb1 + h)], 1)
    top[:, 2] = np.stack([rt, np.full(k, yb1)], 1)
    top[:, 3] = np.stack([rt - g, np.full(k, yb1)], 1)
    top = top.reshape(-1, 2)[:-2]
    r = np.concatenate([bot, top]).astype(np.int32)
    # drop collinear vertices
    a, d = np.roll(r, 1, axis=0), np.roll(r, -1, axis=0)
    col = ((a[:, 0] == r[:, 0]) & (r[:, 0] == d[:, 0])) | ((a[:, 1] == r[:, 1]) & (r[:, 1] == d[:, 1]))
    return np.ascontiguousarray(r[~col], np.int32), rects


def _rng(seed: int, i: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[seed & 0xFFFFFFFFFFFFFFFF, i]))


def generate(image: int = 0, seed: int | None = None, n_pairs: int = 16384, cell: int = 2048, cols: int = 128,
             max_vertices: int = 2000, want_rects: bool = False):
    """Config 5 analog: n_pairs independent comb pairs, each in its own
    cell x cell square so only the intended pairs' MBRs overlap.
    Returns (A, B) PolygonSets; with want_rects, also (rects_A, rects_B)."""
    from . import pack

    seed = seed if seed is not None else 5000 + image
    ra, rb, RA, RB = [], [], [], []
    for i in range(n_pairs):
        r = _rng(seed, i)
        cx, cy = (i % cols) * cell + 16, (i // cols) * cell + 16
        while True:
            w, g = int(r.integers(1, 4)), int(r.integers(1, 4))
            two = bool(r.random() < 0.3)
            kmax = min(1024 // (w + g), max_vertices // (8 if two else 4))
            kmin = max(2, 500 // (8 if two else 4))
            if kmax >= kmin:
                break
        k = int(r.integers(kmin, kmax + 1))
        h = int(r.integers(64, 257)) if not two else int(r.integers(64, 129))
        b = int(r.integers(4, 33))
        ring, rects = comb(cx + 8, cy + 8, k, w, g, h, b, two)
        if r.random() < 0.5:
            dx, dy = (int(v) for v in r.integers(-3, 4, size=2))
            ring2, rects2 = comb(cx + 8 + dx, cy + 8 + dy, k, w, g, h, b, two)
        else:
            w2 = max(1, min(w + g - 1, w + (1 if r.random() < 0.5 else -1)))
            ring2, rects2 = comb(cx + 8, cy + 8, k, w2, w + g - w2, h, b, two)
        ra.append(ring)
        rb.append(ring2)
        RA.append(rects)
        RB.append(rects2)
    A, B = pack(ra), pack(rb)
    if want_rects:
        return A, B, (RA, RB)
    return A, B


def rect_decomp_intersection(ra, rb) -> int:
    """Closed form: |A n B| for disjoint rectangle decompositions of A and B,
    sum_i sum_j |R_i n S_j| (only x-overlapping candidates are visited)."""
    a = np.asarray(ra, np.int64).reshape(-1, 4)
    b = np.asarray(rb, np.int64).reshape(-1, 4)
    if len(a) * len(b) <= 1 << 20:
        ow = np.minimum(a[:, None, 2], b[None, :, 2]) - np.maximum(a[:, None, 0], b[None, :, 0])
        oh = np.minimum(a[:, None, 3], b[None, :, 3]) - np.maximum(a[:, None, 1], b[None, :, 1])
        return int((np.clip(ow, 0, None) * np.clip(oh, 0, None)).sum())
    b = b[np.argsort(b[:, 0], kind="stable")]
    wmax = int((b[:, 2] - b[:, 0]).max())
    tot = 0
    for r in a:
        lo = np.searchsorted(b[:, 0], r[0] - wmax, side="left")
        hi = np.searchsorted(b[:, 0], r[2], side="left")
        c = b[lo:hi]
        ow = np.minimum(c[:, 2], r[2]) - np.maximum(c[:, 0], r[0])
        oh = np.minimum(c[:, 3], r[3]) - np.maximum(c[:, 1], r[1])
        tot += int((np.clip(ow, 0, None) * np.clip(oh, 0, None)).sum())
    return tot


def rect_decomp_area(ra) -> int:
    a = np.asarray(ra, np.int64).reshape(-1, 4)
    return int(((a[:, 2] - a[:, 0]) * (a[:, 3] - a[:, 1])).sum())
