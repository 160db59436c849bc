"""C-ABI checks that need no GPU (``-m "not gpu"``): the sm_100a library builds,
loads, exports exactly the symbols include/sccg.h declares, and its host-only
logic (argument checking, workspace carving, sccg_jaccard on integer sums)
behaves as documented."""
import ctypes
import math
import os
import re
import subprocess
from fractions import Fraction

import numpy as np
import pytest

import oracle
import paper_1208_0277_b200 as sccg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "sccg.h")) as f:
        return sorted(set(re.findall(r"SCCG_API [^;(]*?\b(sccg_\w+)\(", f.read())))


def test_library_exports_exactly_the_header():
    lib = sccg.load()
    assert lib.sccg_version() == 1
    syms = header_symbols()
    assert set(syms) == set(sccg.SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", sccg.library_path()], capture_output=True, text=True).stdout
    exported = sorted(l.split()[-1] for l in out.splitlines() if " T " in l)
    assert exported == syms


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", sccg.library_path()], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches


def test_strerror_and_error_slot():
    lib = sccg.load()
    for code in range(9):
        assert lib.sccg_strerror(code)
    assert lib.sccg_strerror(sccg.E_EMPTY).decode().startswith("no pair")


def _sums_from(inter, uni):
    units = 0
    nz = 0
    for i, u in zip(inter, uni):
        if i:
            units += int(Fraction(int(i) / int(u)) * (1 << 116))
            nz += 1
    limbs = []
    for k in range(3):
        limbs.append(units & ((1 << 30) - 1))
        units >>= 30
    limbs.append(units)
    s = sccg.Sums()
    s.n_pairs = len(inter)
    s.n_nonzero = nz
    s.sum_inter = int(sum(inter))
    s.sum_union = int(sum(u for i, u in zip(inter, uni) if i))
    s.limb0, s.limb1, s.limb2, s.limb3 = limbs
    return s


def test_jaccard_host_logic_against_oracle():
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 1000, 20000):
        uni = rng.integers(1, 10**6, n)
        inter = (uni * rng.random(n)).astype(np.int64)
        inter[rng.random(n) < 0.2] = 0
        if not inter.any():
            inter[0] = 1
        s = _sums_from(inter, uni)
        j, pooled = sccg.jaccard(s)
        ex = oracle.jaccard_exact(inter, uni)
        assert abs(j - float(ex)) <= 1e-12 * float(ex)
        assert pooled == s.sum_inter / s.sum_union
    # SPEC S:364 example {(1,7),(1,1)} -> 4/7
    j, _ = sccg.jaccard(_sums_from([1, 1], [7, 1]))
    assert abs(j - 4 / 7) <= 1e-15
    # Eq. 1 over an empty set: NaN + SCCG_E_EMPTY
    j, p = sccg.jaccard(sccg.Sums())
    assert math.isnan(j) and math.isnan(p)
    lib = sccg.load()
    jj = ctypes.c_double()
    assert lib.sccg_jaccard(ctypes.byref(sccg.Sums()), ctypes.byref(jj), None) == sccg.E_EMPTY
    # sccg_sums_copy: null / misaligned pointers are rejected before anything is enqueued
    assert lib.sccg_sums_copy(None, None, None) == sccg.E_ARG
    assert lib.sccg_sums_copy(8, 12, None) == sccg.E_ARG


def test_host_argument_checks():
    lib = sccg.load()
    assert lib.sccg_polyset_bytes(-1, 0) == 0
    b1 = lib.sccg_polyset_bytes(10, 100)
    b2 = lib.sccg_polyset_bytes(20, 200)
    assert 0 < b1 < b2
    s = sccg.PolySet()
    s.n_polygons, s.n_vertices = 10, 100
    assert lib.sccg_polyset_bind(ctypes.byref(s), None, b1) == sccg.E_ARG
    assert lib.sccg_polyset_bind(ctypes.byref(s), 0x1001, b1) == sccg.E_WORKSPACE  # misaligned
    assert lib.sccg_polyset_bind(ctypes.byref(s), 0x100000, b1 - 512) == sccg.E_WORKSPACE  # too small
    assert lib.sccg_polyset_bind(ctypes.byref(s), 0x100000, b1) == sccg.OK
    assert s.mbr % 256 == 0 and s.edges % 8 == 0
    assert lib.sccg_prep(None, 1, None) == sccg.E_ARG
    sets = (sccg.PolySet * 2)()
    assert lib.sccg_prep_sets(None, 1, 1, None) == sccg.E_ARG
    assert lib.sccg_prep_sets(sets, 0, 1, None) == sccg.E_ARG
    assert lib.sccg_prep_sets(sets, 5, 1, None) == sccg.E_ARG
    n = ctypes.c_int64()
    assert lib.sccg_filter_pairs(None, None, None, 0, ctypes.byref(n), None, 0, None) == sccg.E_ARG
    cfg = sccg.Config(-1, 0, 0, 0, None, None, None)
    assert lib.sccg_pixelbox(None, None, None, 0, None, None, None, ctypes.byref(cfg), None, 0, None) == sccg.E_ARG
    # the compact-transfer decode and the index-pool sizer: argument checks (nothing enqueued)
    assert lib.sccg_decode_rect(None, None, None, None, -1, None, None) == sccg.E_ARG
    assert lib.sccg_decode_rect(None, None, None, None, 3, None, None) == sccg.E_ARG
    assert lib.sccg_decode_rect(0x1004, 0x2000, 0x3000, 0x4000, 3, 0x5000, None) == sccg.E_ARG  # start misaligned
    assert lib.sccg_decode_rect(0x1000, 0x2001, 0x3000, 0x4000, 3, 0x5000, None) == sccg.E_ARG  # move misaligned
    assert lib.sccg_decode_rect(None, None, None, None, 0, None, None) == sccg.OK  # nothing to decode
    # packed decode / packed prep: argument checks before anything is enqueued
    assert lib.sccg_decode_rect_packed(None, None, None, None, None, -1, None, None, None) == sccg.E_ARG
    assert lib.sccg_decode_rect_packed(None, None, None, None, None, 3, 0x1000, None, None) == sccg.E_ARG
    assert lib.sccg_decode_rect_packed(0x1001, None, 0x2000, 0x3000, 0x4000, 3, 0x5000, 0x6000, None) == sccg.E_ARG
    assert lib.sccg_prep_sets_packed(None, None, 1, 1, None) == sccg.E_ARG
    ps = sccg.PolySet()
    assert lib.sccg_prep_sets_packed(ctypes.byref(ps), None, 1, 1, None) == sccg.E_ARG
    enc = sccg.RectPacked()
    assert lib.sccg_prep_sets_packed(ctypes.byref(ps), ctypes.byref(enc), 0, 1, None) == sccg.E_ARG
    assert lib.sccg_prep_sets_packed(ctypes.byref(ps), ctypes.byref(enc), 5, 1, None) == sccg.E_ARG
    assert lib.sccg_pixelbox_index_bytes(-1, 5) == 0
    assert lib.sccg_pixelbox_index_bytes(100, 200) == 8 * 300 + (1 << 24)


def test_jaccard_rejects_status_bits_and_new_entry_points():
    """sums carrying device status bits never yield a J' (NaN and
    the matching code, checked in the documented order); argument checks of
    sccg_contains / sccg_report / sccg_sums_pack / unpack (host-only)."""
    lib = sccg.load()
    base = _sums_from([1, 1], [7, 1])
    for bits, code in ((sccg.STATUS_ARG, sccg.E_ARG), (sccg.STATUS_NOT_RECTILINEAR, sccg.E_NOT_RECTILINEAR),
                       (sccg.STATUS_RANGE, sccg.E_RANGE), (sccg.STATUS_STACK, sccg.E_STACK),
                       (sccg.STATUS_CAPACITY, sccg.E_CAPACITY), (sccg.STATUS_STACK | sccg.STATUS_RANGE, sccg.E_RANGE),
                       (1 << 9, sccg.E_ARG)):
        s = sccg.Sums(*[getattr(base, f) for f in sccg.SUMS_FIELDS])
        s.status = bits
        jj, pp = ctypes.c_double(0.0), ctypes.c_double(0.0)
        assert lib.sccg_jaccard(ctypes.byref(s), ctypes.byref(jj), ctypes.byref(pp)) == code
        assert math.isnan(jj.value) and math.isnan(pp.value)
        with pytest.raises(sccg.SccgError):
            sccg.jaccard(s)
    assert lib.sccg_contains(None, None, None, 0, None, None, None) == sccg.E_ARG
    t = sccg.Tiling(0, 0, 0, 10, 1, 1)
    assert lib.sccg_report(None, None, None, 0, None, None, None, None, ctypes.byref(t), None, None) == sccg.E_ARG
    assert lib.sccg_sums_pack(None, None, None) == sccg.E_ARG
    assert lib.sccg_sums_unpack(8, 12, None) == sccg.E_ARG


def _decode_rect_host(start, move, fv, off):
    """Plain loop mirror of sccg_decode_rect (include/sccg.h)."""
    n = len(off) - 1
    xy = np.zeros((int(off[-1]), 2), np.int64)
    for i in range(n):
        x, y = (int(v) for v in start[i])
        xy[off[i]] = (x, y)
        mb = int(off[i]) - i
        for k in range(1, int(off[i + 1] - off[i])):
            d = int(move[mb + k - 1])
            if ((k & 1) == 1) == (fv[i] == 1):
                y += d
            else:
                x += d
            xy[off[i] + k] = (x, y)
    return xy


def test_encode_rect_roundtrip_and_rejects(tile_sets):
    """The compact rectilinear encoding (sccg_decode_rect's input): lossless on
    clean rectilinear rings of either orientation and either first-edge axis;
    rings it cannot express (a duplicate vertex, a collinear vertex, a move
    beyond int16) are refused, never mis-encoded."""
    import synth

    for S in tile_sets:
        start, move, fv = sccg.encode_rect(S.xy, S.offsets)
        assert move.dtype == np.int16 and len(move) == len(S.xy) - S.n
        assert np.array_equal(_decode_rect_host(start, move, fv, S.offsets), S.xy)
    sq = [[0, 0], [5, 0], [5, 3], [0, 3]]
    rings = [sq, sq[::-1], [[2, 2], [2, 9], [7, 9], [7, 2]]]  # CCW, CW, first edge vertical
    P = synth.pack(rings)
    start, move, fv = sccg.encode_rect(P.xy, P.offsets)
    assert fv.tolist() == [0, 0, 1]
    assert np.array_equal(_decode_rect_host(start, move, fv, P.offsets), P.xy)
    for bad in ([[0, 0], [0, 0], [5, 0], [5, 3], [0, 3]],  # duplicate vertex
                [[0, 0], [2, 0], [5, 0], [5, 3], [0, 3]],  # collinear vertex
                [[0, 0], [40000, 0], [40000, 3], [0, 3]]):  # move beyond int16
        Q = synth.pack([sq, bad])
        assert sccg.encode_rect(Q.xy, Q.offsets) is None


def _decode_rect_packed_host(enc, n):
    """Plain loop reading of the packed format as include/sccg.h states it
    (sccg_decode_rect_packed): returns (xy, offsets)."""
    head, start, units, block = (enc[k] for k in ("head", "start", "units", "block"))
    start_u = start.view(np.uint16)
    offs, xy = [0], []
    for b in range((n + sccg.RECTP_BLOCK - 1) // sccg.RECTP_BLOCK):
        v_off, u, sw, org = (int(t) for t in block[b])
        org &= (1 << 64) - 1
        assert v_off == offs[-1]
        wide, s = (sw >> 62) & 1, sw & ((1 << 62) - 1)
        x0 = int(np.uint32(org & 0xFFFFFFFF).view(np.int32))
        y0 = int(np.uint32((org >> 32) & 0xFFFFFFFF).view(np.int32))
        for jr in range(min(sccg.RECTP_BLOCK, n - b * sccg.RECTP_BLOCK)):
            h = int(head[b * sccg.RECTP_BLOCK + jr])
            V, wc, vert = h & 0x1FFF, (h >> 13) & 3, h >> 15
            if wide:
                q = [int(t) for t in start_u[s + 4 * jr: s + 4 * jr + 4]]
                x = int(np.uint32(q[0] | q[1] << 16).view(np.int32))
                y = int(np.uint32(q[2] | q[3] << 16).view(np.int32))
            else:
                x, y = x0 + int(start[s + 2 * jr]), y0 + int(start[s + 2 * jr + 1])
            if V > 0:
                xy.append((x, y))
            if wc == 3:  # variable length: a bit stream over vlen units, exp-Golomb symbols LSB first
                nu = int(enc["vlen"][b * sccg.RECTP_BLOCK + jr])
                stream = 0
                for t in range(nu):
                    stream |= int(units[u + t]) << (16 * t)
                bit, sign = 0, [0, 0]
                for k in range(1, V):
                    L = 0
                    while not (stream >> (bit + L)) & 1:
                        L += 1
                    low = (stream >> (bit + L + 1)) & ((1 << L) - 1)
                    bit += 2 * L + 1
                    sym = ((1 << L) | low) - 1
                    ax = (k - 1) & 1
                    sign[ax] ^= sym & 1
                    dv = -((sym >> 1) + 1) if sign[ax] else (sym >> 1) + 1
                    if ((k & 1) == 1) == (vert == 1):
                        y += dv
                    else:
                        x += dv
                    xy.append((x, y))
                assert bit <= 16 * nu
                u += nu
                offs.append(offs[-1] + V)
                continue
            c = (4, 2, 1)[wc]
            bits = 16 // c
            for k in range(1, V):
                jm = k - 1
                word = int(units[u + jm // c])
                code = (word >> (bits * (jm % c))) & ((1 << bits) - 1)
                if bits == 16:
                    dv = code - (1 << 16) if code >= 1 << 15 else code
                else:
                    mag = (code & ((1 << (bits - 1)) - 1)) + 1
                    dv = -mag if code >> (bits - 1) else mag
                if ((k & 1) == 1) == (vert == 1):
                    y += dv
                else:
                    x += dv
                xy.append((x, y))
            u += (V - 1 + c - 1) // c if V > 1 else 0
            offs.append(offs[-1] + V)
    return np.array(xy, np.int64).reshape(-1, 2), np.array(offs, np.int64)


def _rect_ring(rng, x0, y0, steps, big=1):
    """A closed rectilinear ring-like vertex walk (not necessarily simple --
    the encoding does not care): alternating axis moves, nonzero."""
    pts = [(x0, y0)]
    x, y = x0, y0
    for k in range(steps):
        d = int(rng.integers(1, big + 1)) * (1 if rng.random() < 0.5 else -1)
        if k % 2 == 0:
            x += d
        else:
            y += d
        pts.append((x, y))
    return pts


def test_encode_rect_packed_roundtrip_and_rejects(tile_sets):
    """The packed rectilinear encoding (sccg_decode_rect_packed's input),
    against a plain reading of the header's layout: lossless on the tile sets,
    on rings whose moves need 4, 8 and 16 bits, on blocks whose starts need
    int32 (wide) and on empty rings / a partial last block / no rings; rings it
    cannot express are refused."""
    import synth

    for S in tile_sets:
        for vlc in (True, False):
            enc = sccg.encode_rect_packed(S.xy, S.offsets, vlc=vlc)
            xy, off = _decode_rect_packed_host(enc, S.n)
            assert np.array_equal(off, S.offsets) and np.array_equal(xy, S.xy)
            if vlc:  # ~2.2 bits per move
                assert enc["units"].nbytes < 0.05 * S.xy.nbytes and ((enc["head"] >> 13) & 3 == 3).all()
            else:
                assert enc["units"].nbytes < 0.3 * S.xy.nbytes  # ~ 4-bit moves
                assert ((enc["head"] >> 13 & 3) == 0).mean() > 0.5  # most rings: 4-bit moves
    rng = np.random.default_rng(7)
    rings = []
    for i in range(700):  # > 2 blocks, the last partial
        big = (1, 8, 9, 128, 129, 32767)[i % 6]
        x0 = int(rng.integers(-2**30, 2**30)) if i == 300 else 5000 + int(rng.integers(-10000, 10000))
        rings.append(_rect_ring(rng, x0, int(rng.integers(-5000, 5000)), int(rng.integers(0, 40)) * 2 + 3, big))
    rings[3] = rings[3][::-1]
    P = synth.pack(rings)
    # empty rings in the middle: offsets repeat
    off = np.concatenate([P.offsets[:10], P.offsets[9:300], P.offsets[299:]])
    enc = sccg.encode_rect_packed(P.xy, off)
    n = len(off) - 1
    xy, off2 = _decode_rect_packed_host(enc, n)
    assert np.array_equal(off2, off) and np.array_equal(xy, P.xy)
    widths = set(((enc["head"] >> 13) & 3).tolist())
    assert {2, 3} <= widths  # variable length where |d| <= 127 (and <= 255 units), else the narrowest fixed width
    enc_f = sccg.encode_rect_packed(P.xy, off, vlc=False)
    assert set(((enc_f["head"] >> 13) & 3).tolist()) == {0, 1, 2}
    xy, off2 = _decode_rect_packed_host(enc_f, n)
    assert np.array_equal(off2, off) and np.array_equal(xy, P.xy)
    assert any((enc["block"][:, 2] >> 62) & 1) and not all((enc["block"][:, 2] >> 62) & 1)
    e0 = sccg.encode_rect_packed(np.zeros((0, 2), np.int32), np.zeros(1, np.int64))
    assert e0["head"].size == 0 and e0["block"].shape == (0, 4)
    sq = [[0, 0], [5, 0], [5, 3], [0, 3]]
    for bad in ([[0, 0], [0, 0], [5, 0], [5, 3], [0, 3]],  # duplicate vertex
                [[0, 0], [2, 0], [5, 0], [5, 3], [0, 3]],  # collinear vertex
                [[0, 0], [40000, 0], [40000, 3], [0, 3]],  # move beyond int16
                _rect_ring(rng, 0, 0, 8191)):  # 8192 vertices
        Q = synth.pack([sq, bad])
        assert sccg.encode_rect_packed(Q.xy, Q.offsets) is None


def test_packed_step_layout(tile_sets):
    """sccg.PackedStep (both sets' packed encodings in one host buffer, one
    host -> device copy per step): every field comes back bit-identical through
    the typed views, 16-byte aligned."""
    A, B = tile_sets[0], tile_sets[1]
    encs = [sccg.encode_rect_packed(S.xy, S.offsets) for S in (A, B)]
    st = sccg.PackedStep(*encs)
    v = st.views(st.host)
    for side, e in zip(("p", "q"), encs):
        for k, a in e.items():
            assert st.layout[side][k][0] % 16 == 0
            assert np.array_equal(v[side][k].numpy().view(a.dtype), a), (side, k)
    assert st.n == {"p": A.n, "q": B.n}
