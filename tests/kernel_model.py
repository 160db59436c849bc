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


# ------------------------------------------------------------------------
# Large-pair path (large.cu): region items with local edge culling.
def _corner_parity(V, X0, Y0):
    return sum(1 for (x, yl, yh) in V if x > X0 and yl <= Y0 < yh) & 1


def build_local(V, H, X0, Y0, X1, Y1):
    """Local lists (region coords, clamped as in pack_loc) and corner parity."""
    Wr, Hr = X1 - X0, Y1 - Y0
    lv = [(x - X0, max(yl - Y0, -1), min(yh - Y0, Hr + 1)) for (x, yl, yh) in V
          if X0 < x < X1 and yl < Y1 and yh > Y0]
    lh = [(f - Y0, max(xl - X0, -1), min(xh - X0, Wr + 1)) for (f, xl, xh) in H
          if Y0 < f < Y1 and xl < X1 and xh > X0]
    return lv, lh, _corner_parity(V, X0, Y0)


def classify_local(lv, lh, x0, y0, Wb, Hb, g, pi):
    sx, sy = 1 << g["lsx"], 1 << g["lsy"]
    kxmask = low_bits(g["kx"])
    h = p = 0
    for (x, yl, yh) in lv:
        x, yl, yh = x - x0, yl - y0, yh - y0
        if yl < Hb and yh > 0:
            r_hi = min(g["nrows"] - 1, (yh - 1) >> g["lsy"])
            if 0 < x < Wb and (x & (sx - 1)) != 0:
                h |= ((g["colpat"] << (x >> g["lsx"])) & M32) & row_range(max(0, yl >> g["lsy"]), r_hi, g)
            if x > 0:
                c_lo = (x + sx - 1) >> g["lsx"]
                if c_lo < g["ncols"]:
                    p ^= (((kxmask & ~low_bits(c_lo)) * g["colpat"]) & M32) & row_range(max(0, (yl + sy - 1) >> g["lsy"]), r_hi, g)
    for (y, xl, xh) in lh:
        y, xl, xh = y - y0, xl - x0, xh - x0
        if 0 < y < Hb and (y & (sy - 1)) != 0 and xl < Wb and xh > 0:
            c_lo = max(0, xl >> g["lsx"])
            c_hi = min(g["ncols"] - 1, (xh - 1) >> g["lsx"])
            h |= (low_bits(c_hi - c_lo + 1) << (((y >> g["lsy"]) << g["lkx"]) + c_lo)) & M32
        if xl <= 0 and xh > 0 and y > 0:
            r_lo = (y + sy - 1) >> g["lsy"]
            if r_lo < g["nrows"]:
                p ^= row_range(r_lo, g["nrows"] - 1, g)
    return h, (p ^ (M32 if pi else 0)) & M32


def pixelize_local(lp, lq, x0, y0, x1, y1, pip, piq):
    Wb, Hb = x1 - x0, y1 - y0
    nw = (Wb + 31) >> 5
    acc = 0
    for row in range(Hb):
        for w in range(nw):
            xs = 32 * w
            ms = []
            for (lv, lh), pi in ((lp, pip), (lq, piq)):
                par = pi
                for (y, xl, xh) in lh:
                    if xl <= x0 < xh and y0 < y < y1 and y - y0 <= row:
                        par ^= 1
                m = 0
                for (x, yl, yh) in lv:
                    if x0 < x < x1 and yl <= row + y0 < yh:
                        m ^= suffix_mask(x - x0 - xs)
                ms.append(m ^ (M32 if par else 0))
            acc += bin(ms[0] & ms[1] & low_bits(Wb - xs)).count("1")
    return acc


def region_pixelbox(lp, lq, Wr, Hr, pip, piq, T, mode=0, stats=None):
    if mode == 1 or Wr * Hr < T:
        return pixelize_local(lp, lq, 0, 0, Wr, Hr, pip, piq)
    acc = 0
    stack = [(0, 0, Wr, Hr, pip, piq)]
    while stack:
        x0, y0, x1, y1, pp, pq = stack.pop()
        Wb, Hb = x1 - x0, y1 - y0
        if Wb * Hb < T:
            acc += pixelize_local(lp, lq, x0, y0, x1, y1, pp, pq)
            continue
        g = make_split(Wb, Hb)
        hp, parp = classify_local(lp[0], lp[1], x0, y0, Wb, Hb, g, pp)
        hq, parq = classify_local(lq[0], lq[1], x0, y0, Wb, Hb, g, pq)
        if stats is not None:
            stats["splits"] = stats.get("splits", 0) + 1
        for lane in range(32):
            cc, rr = lane & (g["kx"] - 1), lane >> g["lkx"]
            if not (cc < g["ncols"] and rr < g["nrows"]):
                continue
            ip = not (hp >> lane) & 1 and (parp >> lane) & 1
            op = not (hp >> lane) & 1 and not (parp >> lane) & 1
            iq = not (hq >> lane) & 1 and (parq >> lane) & 1
            oq = not (hq >> lane) & 1 and not (parq >> lane) & 1
            sx0, sy0 = cc << g["lsx"], rr << g["lsy"]
            sx1, sy1 = min(sx0 + (1 << g["lsx"]), Wb), min(sy0 + (1 << g["lsy"]), Hb)
            if ip and iq:
                acc += (sx1 - sx0) * (sy1 - sy0)
            elif not (op or oq):
                stack.append((x0 + sx0, y0 + sy0, x0 + sx1, y0 + sy1, (parp >> lane) & 1, (parq >> lane) & 1))
    return acc


def pair_intersection_regions(ring_p, ring_q, T=2048, region=128, mode=0, stats=None):
    """Model of expand + item kernels: the root box cut into regions, each
    processed with local lists."""
    ring_p = [(int(x), int(y)) for x, y in ring_p]
    ring_q = [(int(x), int(y)) for x, y in ring_q]
    pv, ph = edges_of(ring_p)
    qv, qh = edges_of(ring_q)
    mp = (min(v[0] for v in ring_p), min(v[1] for v in ring_p), max(v[0] for v in ring_p), max(v[1] for v in ring_p))
    mq = (min(v[0] for v in ring_q), min(v[1] for v in ring_q), max(v[0] for v in ring_q), max(v[1] for v in ring_q))
    bx0, by0 = max(mp[0], mq[0]), max(mp[1], mq[1])
    bx1, by1 = min(mp[2], mq[2]), min(mp[3], mq[3])
    if not (bx0 < bx1 and by0 < by1):
        return 0
    rel = lambda E, vert: [((x - bx0, a - by0, b - by0) if vert else (x - by0, a - bx0, b - bx0)) for (x, a, b) in E]
    PV, PH, QV, QH = rel(pv, True), rel(ph, False), rel(qv, True), rel(qh, False)
    W, H = bx1 - bx0, by1 - by0
    nx, ny = min(32, -(-W // region)), min(32, -(-H // region))
    acc = 0
    for ry in range(ny):
        for rx in range(nx):
            X0, X1 = rx * W // nx, (rx + 1) * W // nx
            Y0, Y1 = ry * H // ny, (ry + 1) * H // ny
            lpv, lph, pip = build_local(PV, PH, X0, Y0, X1, Y1)
            lqv, lqh, piq = build_local(QV, QH, X0, Y0, X1, Y1)
            acc += region_pixelbox((lpv, lph), (lqv, lqh), X1 - X0, Y1 - Y0, pip, piq, T, mode, stats)
    return acc
