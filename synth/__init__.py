"""Seeded synthetic inputs for the SCCG / PixelBox hot path (tests and bench).

INPUT GENERATION ONLY -- this package holds none of the method's arithmetic (no
point-in-polygon, area, intersection, join or Jaccard).  It is the one module
that both ``oracle/`` and the CUDA path consume, per the independence rule.

The C core (``gen.c``) draws nucleus / gland blobs on pixel masks and traces
each mask into a counter-clockwise rectilinear ring.  The configurations mirror
BASELINE.json ``configs`` and the recipe in DESIGN.md ("Input recipe"):

* ``tile``   -- config 1: one 4096x4096 tile, ~1,000 nuclei per set.
* ``slide``  -- config 2: one 100k x 100k whole-slide image, ~500k nuclei per set.
* ``skewed`` -- config 3: 4x4 tiles, nuclei plus 16 glands per tile (MBR side up
  to 512) so deep box subdivision is exercised.
* ``combs``  -- config 5 analog: independent highly concave comb pairs.

Area statistics follow PAPER.md §5.1: mean ~150 px, sd ~100.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libsynth.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile gen.c into libsynth.so (gcc, -O2).  Returns the library path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm", "-lpthread"]
        )
        os.replace(tmp, _LIB)
    return _LIB


class _Spec(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("x0", ctypes.c_int32),
        ("y0", ctypes.c_int32),
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("tile", ctypes.c_int32),
        ("margin", ctypes.c_int32),
        ("nuclei_per_tile", ctypes.c_double),
        ("cluster_frac", ctypes.c_double),
        ("spacing", ctypes.c_double),
        ("cl_lo", ctypes.c_double),
        ("cl_hi", ctypes.c_double),
        ("glands_per_tile", ctypes.c_int32),
        ("gland_split_frac", ctypes.c_double),
        ("drop_frac", ctypes.c_double),
        ("split_frac", ctypes.c_double),
        ("spur_frac", ctypes.c_double),
        ("threads", ctypes.c_int32),
        ("want_masks", ctypes.c_int32),
    ]


class _Set(ctypes.Structure):
    _fields_ = [
        ("xy", ctypes.POINTER(ctypes.c_int32)),
        ("off", ctypes.POINTER(ctypes.c_int64)),
        ("n_polygons", ctypes.c_int64),
        ("n_vertices", ctypes.c_int64),
        ("mbox", ctypes.POINTER(ctypes.c_int32)),
        ("mbits", ctypes.POINTER(ctypes.c_uint8)),
        ("moff", ctypes.POINTER(ctypes.c_int64)),
        ("n_maskbytes", ctypes.c_int64),
    ]


class _Result(ctypes.Structure):
    _fields_ = [("a", _Set), ("b", _Set), ("rejected", ctypes.c_int64)]


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.synth_generate.argtypes = [ctypes.POINTER(_Spec), ctypes.POINTER(_Result)]
            lib.synth_generate.restype = ctypes.c_int
            lib.synth_free.argtypes = [ctypes.POINTER(_Result)]
            lib.synth_free.restype = None
            lib.synth_trace_mask.argtypes = [
                ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
            ]
            lib.synth_trace_mask.restype = ctypes.c_int
            _lib = lib
    return _lib


@dataclass
class PolygonSet:
    """Packed rings: polygon i has vertices ``xy[offsets[i]:offsets[i+1]]``
    (int32 x, y pixel-corner coordinates, ring implicitly closed, CCW)."""

    xy: np.ndarray  # int32 [V, 2]
    offsets: np.ndarray  # int64 [n + 1]
    masks: list | None = None  # optional [(x0, y0, mask uint8[h, w])] per polygon

    @property
    def n(self) -> int:
        return int(self.offsets.shape[0] - 1)

    def ring(self, i: int) -> np.ndarray:
        return self.xy[self.offsets[i] : self.offsets[i + 1]]

    def subset(self, idx) -> "PolygonSet":
        idx = np.asarray(idx, dtype=np.int64)
        lens = self.offsets[idx + 1] - self.offsets[idx]
        off = np.zeros(len(idx) + 1, np.int64)
        np.cumsum(lens, out=off[1:])
        xy = np.concatenate([self.ring(int(i)) for i in idx]) if len(idx) else np.zeros((0, 2), np.int32)
        masks = [self.masks[int(i)] for i in idx] if self.masks is not None else None
        return PolygonSet(np.ascontiguousarray(xy, dtype=np.int32), off, masks)


def _copy_set(s: _Set, want_masks: bool) -> PolygonSet:
    n, nv = int(s.n_polygons), int(s.n_vertices)
    off = np.ctypeslib.as_array(s.off, shape=(n + 1,)).copy()
    xy = np.ctypeslib.as_array(s.xy, shape=(nv, 2)).copy() if nv else np.zeros((0, 2), np.int32)
    masks = None
    if want_masks and n:
        mbox = np.ctypeslib.as_array(s.mbox, shape=(n, 4)).copy()
        moff = np.ctypeslib.as_array(s.moff, shape=(n + 1,)).copy()
        bits = np.ctypeslib.as_array(s.mbits, shape=(int(s.n_maskbytes),)).copy()
        masks = []
        for i in range(n):
            x0, y0, w, h = (int(v) for v in mbox[i])
            masks.append((x0, y0, bits[moff[i] : moff[i + 1]].reshape(h, w)))
    return PolygonSet(xy.astype(np.int32, copy=False), off.astype(np.int64, copy=False), masks)


# Configurations (BASELINE.json "configs"); seeds: config k uses 1000*k + image.
CONFIGS = {
    "tile": dict(width=4096, height=4096, tile=4096, margin=64, nuclei_per_tile=1000.0, cluster_frac=0.0,
                 spacing=40.0, glands_per_tile=0),
    "slide": dict(width=100_000, height=100_000, tile=4096, margin=32, nuclei_per_tile=875.0, cluster_frac=0.33,
                  spacing=40.0, glands_per_tile=0),
    "skewed": dict(width=16384, height=16384, tile=4096, margin=64, nuclei_per_tile=1000.0, cluster_frac=0.0,
                   spacing=40.0, glands_per_tile=16, gland_split_frac=0.30),
}
CONFIG_INDEX = {"tile": 1, "slide": 2, "skewed": 3, "study": 4, "combs": 5}


def generate(config: str = "tile", image: int = 0, seed: int | None = None, want_masks: bool = False,
             threads: int | None = None, **overrides) -> tuple[PolygonSet, PolygonSet]:
    """Generate the two result sets (A, B) of one synthetic image."""
    if config == "combs":
        from . import combs

        return combs.generate(image=image, seed=seed, **overrides)
    base = dict(CONFIGS["slide" if config == "study" else config])
    base.update(overrides)
    spec = _Spec()
    spec.seed = seed if seed is not None else 1000 * CONFIG_INDEX[config] + image
    spec.x0 = base.get("x0", 0)
    spec.y0 = base.get("y0", 0)
    spec.width = base["width"]
    spec.height = base["height"]
    spec.tile = base["tile"]
    spec.margin = base["margin"]
    spec.nuclei_per_tile = base["nuclei_per_tile"]
    spec.cluster_frac = base["cluster_frac"]
    spec.spacing = base["spacing"]
    spec.cl_lo = base.get("cl_lo", 14.0)
    spec.cl_hi = base.get("cl_hi", 20.0)
    spec.glands_per_tile = base.get("glands_per_tile", 0)
    spec.gland_split_frac = base.get("gland_split_frac", 0.0)
    spec.drop_frac = base.get("drop_frac", 0.05)
    spec.split_frac = base.get("split_frac", 0.05)
    spec.spur_frac = base.get("spur_frac", 0.05)
    spec.threads = threads if threads is not None else max(1, min(32, os.cpu_count() or 1))
    spec.want_masks = 1 if want_masks else 0
    lib = _load()
    res = _Result()
    lib.synth_generate(ctypes.byref(spec), ctypes.byref(res))
    try:
        a = _copy_set(res.a, want_masks)
        b = _copy_set(res.b, want_masks)
    finally:
        lib.synth_free(ctypes.byref(res))
    return a, b


def trace_mask(mask: np.ndarray, ox: int = 0, oy: int = 0):
    """Clean a binary mask (h x w) into one simply-connected region and trace
    its CCW ring.  Returns (ring int32[V, 2] or None if empty, cleaned mask)."""
    lib = _load()
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    h, w = m.shape
    cleaned = np.zeros_like(m)
    cap = 4 * (w + 1) * (h + 1) + 8
    xy = np.zeros((cap, 2), np.int32)
    nv = lib.synth_trace_mask(m.ctypes.data, w, h, ox, oy, cleaned.ctypes.data, xy.ctypes.data, cap)
    if nv < 0:
        raise RuntimeError("trace buffer too small")
    return (xy[:nv].copy() if nv else None), cleaned


def pack(rings) -> PolygonSet:
    """Pack a list of int rings [(V_i, 2)] into a PolygonSet."""
    off = np.zeros(len(rings) + 1, np.int64)
    np.cumsum([len(r) for r in rings], out=off[1:])
    xy = np.concatenate([np.asarray(r, np.int32).reshape(-1, 2) for r in rings]) if rings else np.zeros((0, 2), np.int32)
    return PolygonSet(np.ascontiguousarray(xy, np.int32), off)


def partition(seed: int, n: int = 96, k: int = 60, ox: int = 0, oy: int = 0) -> "PolygonSet":
    """A seeded partition of the n x n square into rectilinear pieces (region
    growing from k seeds in random order), keeping the pieces that trace to one
    clean ring.  Neighbouring pieces share sides, T-junctions and corners: the
    ST_Touches workload.  Input generation only."""
    rng = np.random.default_rng(seed)
    lab = -np.ones((n, n), np.int32)
    front = []
    for i, (y, x) in enumerate(rng.integers(0, n, (k, 2))):
        if lab[y, x] < 0:
            lab[y, x] = i
            front.append((int(y), int(x)))
    while front:
        j = int(rng.integers(len(front)))
        y, x = front[j]
        front[j] = front[-1]
        front.pop()
        for dy, dx in ((0, 1), (1, 0), (0, -1), (-1, 0)):
            yy, xx = y + dy, x + dx
            if 0 <= yy < n and 0 <= xx < n and lab[yy, xx] < 0:
                lab[yy, xx] = lab[y, x]
                front.append((yy, xx))
    rings = []
    for i in range(k):
        m = (lab == i).astype(np.uint8)
        if not m.any():
            continue
        ys, xs = np.nonzero(m)
        y0, x0 = int(ys.min()), int(xs.min())
        sub = m[y0:ys.max() + 1, x0:xs.max() + 1]
        ring, cleaned = trace_mask(sub)
        if ring is not None and (cleaned == sub).all():
            rings.append(ring + np.array([x0 + ox, y0 + oy], np.int32))
    return pack(rings)
