"""Pure-Python model of the CUDA PixelBox kernel's bit-parallel logic.

A CPU pre-screen only (tests/test_kernel_model.py): it mirrors the formulas in
paper_1208_0277_b200/csrc/pixelbox.cu (row-word crossing masks, edge-parallel
Lemma-1 classification over power-of-two sub-box grids, DFS stack) so logic
errors surface before GPU time is spent.  It is not the oracle and proves
nothing about the GPU; the GPU parity tests compare the real kernels against
oracle/.
"""
from __future__ import annotations

M32 = 0xFFFFFFFF


def suffix_mask(k):
    k = max(k, 0)
    return 0 if k >= 32 else (M32 << k) & M32


def low_bits(n):
    n = max(n, 0)
    return M32 if n >= 32 else (1 << n) - 1


def edges_of(ring):
    """(vertical [(x, ylo, yhi)], horizontal [(y, xlo, xhi)]) in absolute coords."""
    v, h = [], []
    n = len(ring)
    for i in range(n):
        a, c = ring[i], ring[(i + 1) % n]
        if a[0] == c[0] and a[1] != c[1]:
            v.append((int(a[0]), int(min(a[1], c[1])), int(max(a[1], c[1]))))
        elif a[1] == c[1] and a[0] != c[0]:
            h.append((int(a[1]), int(min(a[0], c[0])), int(max(a[0], c[0]))))
    return v, h


def pixelize(X0, Y0, X1, Y1, pv, qv):
    """pv/qv: vertical edges relative to the root origin.  Returns |box n p n q|."""
    Wb, Hb = X1 - X0, Y1 - Y0
    nw = (Wb + 31) >> 5
    acc = 0
    for row in range(Hb):
        for w in range(nw):
            xs = 32 * w
            m = []
            for E in (pv, qv):
                mm = 0
                for (x, yl, yh) in E:
                    x, yl, yh = x - X0, yl - Y0, yh - Y0
                    if not (yl < Hb and yh > 0):
                        continue
                    if (row - yl) & M32 < (yh - yl) & M32:
                        mm ^= suffix_mask(x - xs)
                m.append(mm)
            acc += bin(m[0] & m[1] & low_bits(Wb - xs)).count("1")
    return acc


def ceil_log2(v):
    return 0 if v <= 1 else (v - 1).bit_length()


def make_split(Wb, Hb):
    kx, lkx = (8, 3) if Wb >= Hb else (4, 2)
    ky = 32 // kx
    lsx = ceil_log2((Wb + kx - 1) // kx)
    lsy = ceil_log2((Hb + ky - 1) // ky)
    ncols = (Wb + (1 << lsx) - 1) >> lsx
    nrows = (Hb + (1 << lsy) - 1) >> lsy
    colpat = 0x01010101 if kx == 8 else 0x11111111
    return dict(kx=kx, lkx=lkx, lsx=lsx, lsy=lsy, ncols=ncols, nrows=nrows, colpat=colpat)


def row_range(r_lo, r_hi, g):
    return (low_bits((r_hi - r_lo + 1) << g["lkx"]) << (max(r_lo, 0) << g["lkx"])) & M32


def classify(V, H, X0, Y0, Wb, Hb, g):
    sx, sy = 1 << g["lsx"], 1 << g["lsy"]
    h = p = 0
    for (x, yl, yh) in V:
        x, yl, yh = x - X0, yl - Y0, yh - Y0
        if yl < Hb and yh > 0:
            r_hi = min(g["nrows"] - 1, (yh - 1) >> g["lsy"])
            if 0 < x < Wb and (x & (sx - 1)) != 0:
                h |= ((g["colpat"] << (x >> g["lsx"])) & M32) & row_range(max(0, yl >> g["lsy"]), r_hi, g)
            if x > 0:
                c_hi = min(g["ncols"] - 1, (x - 1) >> g["lsx"])
                p ^= ((low_bits(c_hi + 1) * g["colpat"]) & M32) & row_range(max(0, (yl + sy - 1) >> g["lsy"]), r_hi, g)
    for (y, xl, xh) in H:
        y, xl, xh = y - Y0, xl - X0, xh - X0
        if 0 < y < Hb and (y & (sy - 1)) != 0 and xl < Wb and xh > 0:
            c_lo = max(0, xl >> g["lsx"])
            c_hi = min(g["ncols"] - 1, (xh - 1) >> g["lsx"])
            h |= (low_bits(c_hi - c_lo + 1) << (((y >> g["lsy"]) << g["lkx"]) + c_lo)) & M32
    return h, p


def pair_intersection(ring_p, ring_q, T=2048, mode=0, stats=None):
    ring_p = [(int(x), int(y)) for x, y in ring_p]
    ring_q = [(int(x), int(y)) for x, y in ring_q]
    pv, ph = edges_of(ring_p)
    qv, qh = edges_of(ring_q)
    xs = [v[0] for v in ring_p]
    ys = [v[1] for v in ring_p]
    mp = (min(xs), min(ys), max(xs), max(ys))
    xs = [v[0] for v in ring_q]
    ys = [v[1] for v in ring_q]
    mq = (min(xs), min(ys), max(xs), max(ys))
    bx0, by0 = max(mp[0], mq[0]), max(mp[1], mq[1])
    bx1, by1 = min(mp[2], mq[2]), min(mp[3], mq[3])
    if not (bx0 < bx1 and by0 < by1):
        return 0

    def rel(E, vert):
        if vert:
            return [(x - bx0, a - by0, b - by0) for (x, a, b) in E]
        return [(y - by0, a - bx0, b - bx0) for (y, a, b) in E]

    PV, PH, QV, QH = rel(pv, True), rel(ph, False), rel(qv, True), rel(qh, False)
    W, H = bx1 - bx0, by1 - by0
    if mode == 1 or W * H < T:
        return pixelize(0, 0, W, H, PV, QV)
    acc = 0
    stack = [(0, 0, W, H)]
    while stack:
        X0, Y0, X1, Y1 = stack.pop()
        Wb, Hb = X1 - X0, Y1 - Y0
        if Wb * Hb < T:
            acc += pixelize(X0, Y0, X1, Y1, PV, QV)
            if stats is not None:
                stats["pix"] = stats.get("pix", 0) + 1
            continue
        g = make_split(Wb, Hb)
        hp, pp = classify(PV, PH, X0, Y0, Wb, Hb, g)
        hq, pq = classify(QV, QH, X0, Y0, Wb, Hb, g)
        valid = 0
        for lane in range(32):
            cc, rr = lane & (g["kx"] - 1), lane >> g["lkx"]
            if cc < g["ncols"] and rr < g["nrows"]:
                valid |= 1 << lane
        in_p, out_p = ~hp & pp & M32, ~hp & ~pp & M32
        in_q, out_q = ~hq & pq & M32, ~hq & ~pq & M32
        contrib = valid & in_p & in_q
        cont = valid & ~(out_p | out_q) & ~contrib & M32
        if stats is not None:
            stats["splits"] = stats.get("splits", 0) + 1
        for lane in range(32):
            cc, rr = lane & (g["kx"] - 1), lane >> g["lkx"]
            x0, y0 = cc << g["lsx"], rr << g["lsy"]
            x1, y1 = min(x0 + (1 << g["lsx"]), Wb), min(y0 + (1 << g["lsy"]), Hb)
            if (contrib >> lane) & 1:
                acc += (x1 - x0) * (y1 - y0)
            if (cont >> lane) & 1:
                stack.append((X0 + x0, Y0 + y0, X0 + x1, Y0 + y1))
    return acc
