"""paper_1208_0277_b200 -- B200-native PixelBox hot path of SCCG (arXiv 1208.0277).

A thin ctypes binding over the C ABI in ``include/sccg.h`` (``libsccg.so``,
built for sm_100a).  Argument marshalling only: every step of the path -- prep,
MBR join, PixelBox, the integer sums -- runs in the library's CUDA kernels.
There is no CPU fallback: if the library or a GPU is missing, these functions
raise.

PyTorch supplies device memory, streams and process groups::

    import paper_1208_0277_b200 as sccg
    P = sccg.DeviceSet(xy_p, off_p)           # torch cuda tensors (int32 [V,2], int64 [n+1])
    Q = sccg.DeviceSet(xy_q, off_q)
    pairs = sccg.filter_pairs(P, Q)           # int32 [N, 2], sorted by (p, q)
    inter, uni, sums = sccg.pixelbox(P, Q, pairs)
    jprime, pooled = sccg.jaccard(sums)       # Eq. (1)

``compare`` runs the whole path from host arrays (the end-to-end API).
"""
from __future__ import annotations

import ctypes
import math
import os
import threading

from . import build as _build

_lock = threading.Lock()
_lib = None

# status codes (include/sccg.h)
OK, E_ARG, E_NOT_RECTILINEAR, E_RANGE, E_CAPACITY, E_STACK, E_EMPTY, E_CUDA, E_WORKSPACE = range(9)
RASTER_FLAG = 1 << 30  # ecount[i, 0] bit: prep stored polygon i's raster rows (the count is the low 30 bits)
FLAG_NO_RASTER = 1
FLAG_PAPER_SPLIT = 2
CNT_PIXELS, CNT_ROWTESTS, CNT_BOXES, CNT_BOXEDGES, CNT_SPLITS, CNT_PIXBOXES, CNT_ROOTPX = range(7)
SUMS_FIELDS = ("n_pairs", "n_nonzero", "sum_inter", "sum_union", "sum_area_p", "sum_area_q", "limb0", "limb1",
               "limb2", "limb3", "status")
SYMBOLS = ("sccg_polyset_bytes", "sccg_polyset_bind", "sccg_prep", "sccg_prep_sets", "sccg_filter_workspace_bytes",
           "sccg_filter_pairs", "sccg_filter_pairs_closed", "sccg_filter_pairs_async", "sccg_touches", "sccg_pixelbox_workspace_bytes", "sccg_pixelbox_index_bytes", "sccg_pixelbox",
           "sccg_pixelbox_async", "sccg_count_missing", "sccg_contains", "sccg_report", "sccg_jaccard", "sccg_sums_copy", "sccg_decode_rect",
           "sccg_decode_rect_packed", "sccg_prep_sets_packed",
           "sccg_sums_pack", "sccg_sums_unpack", "sccg_strerror", "sccg_last_error_string", "sccg_last_error_index",
           "sccg_version")
STATUS_ARG, STATUS_NOT_RECTILINEAR, STATUS_RANGE, STATUS_STACK, STATUS_CAPACITY = 1, 2, 4, 8, 16
REDUCE_WORDS = 26  # SCCG_REDUCE_WORDS
REPORT_FIELDS = SUMS_FIELDS[:10] + ("status", "n_poly_p", "n_poly_q", "missing_p", "missing_q")


class SccgError(RuntimeError):
    def __init__(self, code: int, where: str):
        lib = _lib
        self.code = code
        self.detail = lib.sccg_last_error_string().decode() if lib else ""
        self.index = int(lib.sccg_last_error_index()) if lib else -1
        name = lib.sccg_strerror(code).decode() if lib else str(code)
        super().__init__(f"{where}: {name} ({self.detail}) [index {self.index}]")


class PolySet(ctypes.Structure):
    _fields_ = [
        ("xy", ctypes.c_void_p),
        ("offsets", ctypes.c_void_p),
        ("n_polygons", ctypes.c_int64),
        ("n_vertices", ctypes.c_int64),
        ("mbr", ctypes.c_void_p),
        ("area", ctypes.c_void_p),
        ("ecount", ctypes.c_void_p),
        ("edges", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
        ("stats", ctypes.c_void_p),
    ]


class Sums(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in SUMS_FIELDS]


class Tiling(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in ("x0", "y0", "tile_w", "tile_h", "ntx", "nty")]


class Config(ctypes.Structure):
    _fields_ = [
        ("threshold", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("grid", ctypes.c_int32),
        ("counters", ctypes.c_void_p),
        ("hit_p", ctypes.c_void_p),
        ("hit_q", ctypes.c_void_p),
    ]


def library_path() -> str:
    v = os.environ.get("SCCG_LIB")
    if v:
        return v if os.path.isabs(v) else os.path.join(os.path.dirname(_build.LIB), v)
    return _build.LIB


def load(build: bool = True):
    """Load libsccg.so (building it first if stale and nvcc exists)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = _build.LIB
        variant = os.environ.get("SCCG_LIB")  # experiment variant built by build.py --variant
        if variant:
            path = variant if os.path.isabs(variant) else os.path.join(os.path.dirname(_build.LIB), variant)
            build = False
        if build:
            try:
                path = _build.build()
            except (OSError, RuntimeError) as e:  # no nvcc: fall through to an existing library
                if not os.path.exists(path):
                    raise ImportError(f"libsccg.so missing and cannot be built: {e}") from e
        if not os.path.exists(path):
            raise ImportError(f"libsccg.so not found at {path}; run paper_1208_0277_b200/build.py")
        lib = ctypes.CDLL(path)
        vp, i64, i32, sz, cint = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t, ctypes.c_int
        ps = ctypes.POINTER(PolySet)
        lib.sccg_polyset_bytes.argtypes = [i64, i64]
        lib.sccg_polyset_bytes.restype = sz
        lib.sccg_polyset_bind.argtypes = [ps, vp, sz]
        lib.sccg_polyset_bind.restype = cint
        lib.sccg_prep.argtypes = [ps, i32, vp]
        lib.sccg_prep.restype = cint
        lib.sccg_prep_sets.argtypes = [ps, i32, i32, vp]
        lib.sccg_prep_sets.restype = cint
        lib.sccg_filter_workspace_bytes.argtypes = [i64, i64]
        lib.sccg_filter_workspace_bytes.restype = sz
        lib.sccg_filter_pairs.argtypes = [ps, ps, vp, i64, ctypes.POINTER(i64), vp, sz, vp]
        lib.sccg_filter_pairs_closed.argtypes = [ps, ps, vp, i64, ctypes.POINTER(i64), vp, sz, vp]
        lib.sccg_filter_pairs_closed.restype = cint
        lib.sccg_touches.argtypes = [ps, ps, vp, i64, vp, vp, vp]
        lib.sccg_touches.restype = cint
        lib.sccg_filter_pairs.restype = cint
        lib.sccg_filter_pairs_async.argtypes = [ps, ps, vp, i64, vp, vp, sz, vp]
        lib.sccg_filter_pairs_async.restype = cint
        lib.sccg_pixelbox_async.argtypes = [ps, ps, vp, vp, i64, vp, vp, vp, ctypes.POINTER(Config), vp, sz, vp]
        lib.sccg_pixelbox_async.restype = cint
        lib.sccg_pixelbox_workspace_bytes.argtypes = [i64]
        lib.sccg_pixelbox_workspace_bytes.restype = sz
        lib.sccg_pixelbox_index_bytes.argtypes = [i64, i64]
        lib.sccg_pixelbox_index_bytes.restype = sz
        lib.sccg_decode_rect.argtypes = [vp, vp, vp, vp, i64, vp, vp]
        lib.sccg_decode_rect.restype = cint
        lib.sccg_decode_rect_packed.argtypes = [vp, vp, vp, vp, vp, i64, vp, vp, vp]
        lib.sccg_prep_sets_packed.argtypes = [vp, vp, ctypes.c_int32, ctypes.c_int32, vp]
        lib.sccg_prep_sets_packed.restype = cint
        lib.sccg_decode_rect_packed.restype = cint
        lib.sccg_pixelbox.argtypes = [ps, ps, vp, i64, vp, vp, vp, ctypes.POINTER(Config), vp, sz, vp]
        lib.sccg_pixelbox.restype = cint
        lib.sccg_count_missing.argtypes = [vp, i64, vp, vp]
        lib.sccg_count_missing.restype = cint
        lib.sccg_contains.argtypes = [ps, ps, vp, i64, vp, vp, vp]
        lib.sccg_contains.restype = cint
        lib.sccg_report.argtypes = [ps, ps, vp, i64, vp, vp, vp, vp, ctypes.POINTER(Tiling), vp, vp]
        lib.sccg_report.restype = cint
        lib.sccg_sums_pack.argtypes = [vp, vp, vp]
        lib.sccg_sums_pack.restype = cint
        lib.sccg_sums_unpack.argtypes = [vp, vp, vp]
        lib.sccg_sums_unpack.restype = cint
        lib.sccg_jaccard.argtypes = [ctypes.POINTER(Sums), ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(ctypes.c_double)]
        lib.sccg_jaccard.restype = cint
        lib.sccg_sums_copy.argtypes = [vp, vp, vp]
        lib.sccg_sums_copy.restype = cint
        lib.sccg_strerror.argtypes = [cint]
        lib.sccg_strerror.restype = ctypes.c_char_p
        lib.sccg_last_error_string.argtypes = []
        lib.sccg_last_error_string.restype = ctypes.c_char_p
        lib.sccg_last_error_index.argtypes = []
        lib.sccg_last_error_index.restype = i64
        lib.sccg_version.argtypes = []
        lib.sccg_version.restype = cint
        _lib = lib
        return lib


def _check(code: int, where: str):
    if code != OK:
        raise SccgError(code, where)


def _torch():
    import torch

    return torch


def _stream_ptr(stream=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _require_cuda(t, name, dtype):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


class RectPacked(ctypes.Structure):
    """sccg_rect_packed: a set's rings in the packed transfer encoding (device pointers)."""
    _fields_ = [("head", ctypes.c_void_p), ("vlen", ctypes.c_void_p), ("start", ctypes.c_void_p),
                ("units", ctypes.c_void_p), ("block", ctypes.c_void_p)]


def rect_packed(enc) -> RectPacked:
    """RectPacked of an encode_rect_packed dict already on the device (tensors)."""
    ptr = lambda t: t.data_ptr() if t is not None and t.numel() else None  # noqa: E731
    return RectPacked(ptr(enc["head"]), ptr(enc.get("vlen")), ptr(enc["start"]), ptr(enc["units"]),
                      ptr(enc["block"]))


def prep_sets_packed(sets, encs, validate: bool = True, stream=None):
    """sccg_prep_sets_packed: prep the DeviceSets (built with prep=False over
    writable xy / offsets buffers) from their packed encodings (device dicts):
    decodes xy and offsets into the sets' buffers and derives everything
    sccg_prep_sets does, in one launch."""
    arr = (PolySet * len(sets))(*[S.c for S in sets])
    enc = (RectPacked * len(sets))(*[rect_packed(e) for e in encs])
    _check(load().sccg_prep_sets_packed(arr, enc, len(sets), 1 if validate else 0, _stream_ptr(stream)),
           "sccg_prep_sets_packed")


class DeviceSet:
    """One polygon set resident on the GPU plus the buffers sccg_prep fills.

    xy: int32 [V, 2] CUDA tensor; offsets: int64 [n + 1] CUDA tensor."""

    def __init__(self, xy, offsets, prep: bool = True, validate: bool = True, stream=None):
        torch = _torch()
        lib = load()
        _require_cuda(xy, "xy", torch.int32)
        _require_cuda(offsets, "offsets", torch.int64)
        self.xy, self.offsets = xy, offsets
        n = int(offsets.numel()) - 1
        nv = int(xy.numel()) // 2
        self.n, self.nv = n, nv
        nbytes = int(lib.sccg_polyset_bytes(n, nv))
        self._buf = torch.empty(nbytes, dtype=torch.uint8, device=xy.device)
        self.c = PolySet(xy.data_ptr(), offsets.data_ptr(), n, nv, None, None, None, None, None, None)
        _check(lib.sccg_polyset_bind(ctypes.byref(self.c), self._buf.data_ptr(), nbytes), "sccg_polyset_bind")
        if prep:
            self.prep(validate, stream)

    def prep(self, validate: bool = True, stream=None):
        _check(load().sccg_prep(ctypes.byref(self.c), 1 if validate else 0, _stream_ptr(stream)), "sccg_prep")
        return self

    def _view(self, ptr_field, dtype, shape):
        torch = _torch()
        base = self._buf.data_ptr()
        off = getattr(self.c, ptr_field) - base
        count = 1
        for s in shape:
            count *= s
        esz = torch.empty((), dtype=dtype).element_size()
        return self._buf[off: off + count * esz].view(dtype).view(*shape)

    @property
    def mbr(self):
        return self._view("mbr", _torch().int32, (self.n, 4))

    @property
    def area(self):
        return self._view("area", _torch().int64, (self.n,))

    @property
    def ecount(self):
        """int32 [n, 2]: vertical-edge records | RASTER_FLAG, the records' 16-bit rebase
        (x0 - xlo) | (y0 - ylo) << 16 (include/sccg.h, internal.cuh decode_edge)."""
        return self._view("ecount", _torch().int32, (self.n, 2))

    @property
    def status(self):
        return self._view("status", _torch().int32, (2,))

    def stats_bytes(self):
        """The 128-byte join statistics block (internal layout)."""
        return self._view("stats", _torch().uint8, (128,))

    def used_edge_words(self):
        """The defined part of `edges` after prep, concatenated over polygons:
        each polygon's vertical-edge records, then its raster rows (as 32-bit
        words, when ecount flags one).  For tests and diagnostics."""
        torch = _torch()
        edges = self._view("edges", torch.int64, (self.nv,))
        ec = self.ecount.long()
        m = self.mbr.long()
        rast = (ec[:, 0] & RASTER_FLAG) != 0
        used = (ec[:, 0] & (RASTER_FLAG - 1)) + torch.where(rast, (m[:, 3] - m[:, 1] + 1) // 2, torch.zeros_like(ec[:, 0]))
        off = self.offsets[:-1]
        idx = torch.repeat_interleave(off, used) + (
            torch.arange(int(used.sum()), device=used.device) - torch.repeat_interleave(torch.cumsum(used, 0) - used, used))
        words = edges[idx].clone()
        # an odd raster row count leaves the upper half of the last slot undefined
        odd = rast & ((m[:, 3] - m[:, 1]) % 2 == 1)
        last = (torch.cumsum(used, 0) - 1)[odd]
        words[last] &= 0xFFFFFFFF
        return words


def filter_pairs(P: DeviceSet, Q: DeviceSet, cap: int | None = None, stream=None, closed: bool = False):
    """Candidate pairs (overlapping half-open MBRs; closed=True: closed MBRs
    that meet, touching included), int32 [N, 2] sorted by (p, q)."""
    torch = _torch()
    lib = load()
    fn = lib.sccg_filter_pairs_closed if closed else lib.sccg_filter_pairs
    wsb = int(lib.sccg_filter_workspace_bytes(P.n, Q.n))
    ws = torch.empty(wsb, dtype=torch.uint8, device=P.xy.device)
    if cap is None:
        cap = 2 * max(P.n, Q.n) + 1024
    for _ in range(2):
        out = torch.empty((max(cap, 1), 2), dtype=torch.int32, device=P.xy.device)
        n = ctypes.c_int64(0)
        code = fn(ctypes.byref(P.c), ctypes.byref(Q.c), out.data_ptr(), cap, ctypes.byref(n), ws.data_ptr(), wsb,
                  _stream_ptr(stream))
        if code == E_CAPACITY:
            cap = int(n.value)
            continue
        _check(code, "sccg_filter_pairs")
        return out[: int(n.value)]
    raise SccgError(E_CAPACITY, "sccg_filter_pairs")


class Pipeline:
    """A device-resident, host-sync-free cross-comparison step for fixed sets:
    prep(P), prep(Q), MBR join and PixelBox enqueued back to back on one stream
    (sccg_filter_pairs_async / sccg_pixelbox_async: the pair count never leaves
    the GPU), so the whole step is captured and replayed as ONE CUDA graph
    (and as three stage graphs, used when run() is asked for stage events).
    ``run()`` returns the device sums vector; read it (one sync) for J'."""

    def __init__(self, P: "DeviceSet", Q: "DeviceSet", cap: int | None = None, threshold: int = 0, graph: bool = True,
                 validate: bool = True, raster: bool = True, readback=(), outputs: bool = True,
                 paper_split: bool = False, index: bool = True, allreduce=None, packed=None):
        torch = _torch()
        self.lib = load()
        self.P, self.Q = P, Q
        # packed = (enc_p, enc_q): device dicts of the packed encoding at fixed addresses; the step's prep then
        # decodes the rings itself (sccg_prep_sets_packed) into P's and Q's xy / offsets buffers
        self._packed = (RectPacked * 2)(*[rect_packed(e) for e in packed]) if packed is not None else None
        dev = P.xy.device
        self.cap = int(cap) if cap is not None else 2 * max(P.n, Q.n) + 1024
        self.pairs = torch.empty((max(self.cap, 1), 2), dtype=torch.int32, device=dev)
        self.result = torch.zeros(2, dtype=torch.int64, device=dev)
        self.sums = new_sums(dev)
        self._zero = new_sums(dev)  # the step's sums are reset by our copy kernel (no torch fill kernel in the graph)
        # per-pair |p n q| and |p u q| (row a7's outputs), written every step; valid for pairs[:n]
        self.inter = torch.empty(max(self.cap, 1), dtype=torch.int64, device=dev) if outputs else None
        self.uni = torch.empty(max(self.cap, 1), dtype=torch.int64, device=dev) if outputs else None
        self.fws_bytes = int(self.lib.sccg_filter_workspace_bytes(P.n, Q.n))
        self.fws = torch.empty(self.fws_bytes, dtype=torch.uint8, device=dev)
        # required PixelBox workspace plus the large path's edge-index pool (sccg_pixelbox_index_bytes)
        self.pws_bytes = int(self.lib.sccg_pixelbox_workspace_bytes(self.cap)) + (
            int(self.lib.sccg_pixelbox_index_bytes(P.nv, Q.nv)) if index else 0)
        self.pws = torch.empty(max(self.pws_bytes, 256), dtype=torch.uint8, device=dev)
        self.cfg = Config(threshold, 0, (0 if raster else FLAG_NO_RASTER) | (FLAG_PAPER_SPLIT if paper_split else 0), 0,
                          None, None, None)
        self.validate = 1 if validate else 0
        self._sets = (PolySet * 2)(P.c, Q.c)  # copies of the bound descriptors (pointers only)
        # allreduce: a callable (e.g. dist.allreduce_sums over NCCL) enqueued after PixelBox and before the
        # read-back, so the multi-GPU step's one collective is inside the step graph
        self.allreduce = allreduce
        # readback: pinned host int64 [11] buffers; run(slot=k) ends the step by
        # writing the sums into readback[k] from the GPU (sccg_sums_copy inside
        # the PixelBox graph: no copy-engine transfer, no extra launch)
        self.readback = tuple(readback)
        self._slot = 0
        self.graphs = None
        if graph:
            s = torch.cuda.Stream(device=dev)
            s.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(s):  # warm-up outside capture (one-time attribute setup)
                for stage in self._stages:
                    stage()
            torch.cuda.current_stream(dev).wait_stream(s)
            torch.cuda.synchronize(dev)
            graphs = []
            for stage in self._stages:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    stage()
                graphs.append(g)
            self.graphs = tuple(graphs)
            self._pix_rb = []
            for k in range(len(self.readback)):
                self._slot = k
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._enqueue_pixelbox()
                self._pix_rb.append(g)
            # the whole step as ONE graph (per read-back slot): no graph-to-graph
            # gaps, and the stages chain by programmatic dependent launch too;
            # run() uses it whenever no per-stage events are asked for
            self._full = []
            for k in range(max(1, len(self.readback))):
                self._slot = k
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for stage in self._stages:
                        stage()
                self._full.append(g)

    @property
    def _stages(self):
        return (self._enqueue_prep, self._enqueue_join, self._enqueue_pixelbox)

    def _enqueue_prep(self):
        st = _stream_ptr()
        lib = self.lib
        sums_copy(self._zero, self.sums)
        if self._packed is not None:
            _check(lib.sccg_prep_sets_packed(self._sets, self._packed, 2, self.validate, st), "sccg_prep_sets_packed")
        else:
            _check(lib.sccg_prep_sets(self._sets, 2, self.validate, st), "sccg_prep_sets")

    def _enqueue_join(self):
        _check(self.lib.sccg_filter_pairs_async(ctypes.byref(self.P.c), ctypes.byref(self.Q.c), self.pairs.data_ptr(),
                                                self.cap, self.result.data_ptr(), self.fws.data_ptr(), self.fws_bytes,
                                                _stream_ptr()), "sccg_filter_pairs_async")

    def _enqueue_pixelbox(self):
        _check(self.lib.sccg_pixelbox_async(ctypes.byref(self.P.c), ctypes.byref(self.Q.c), self.pairs.data_ptr(),
                                            self.result.data_ptr(), self.cap,
                                            self.inter.data_ptr() if self.inter is not None else None,
                                            self.uni.data_ptr() if self.uni is not None else None, self.sums.data_ptr(),
                                            ctypes.byref(self.cfg), self.pws.data_ptr(), self.pws_bytes, _stream_ptr()),
               "sccg_pixelbox_async")
        if self.allreduce is not None:
            self.allreduce(self.sums)
        if self.readback:
            sums_copy(self.sums, self.readback[self._slot])

    def run(self, events=None, slot: int = 0):
        """One step: prep(P) + prep(Q) | MBR join | PixelBox, three graphs (or
        eager launches) back to back on the current stream.  events = four CUDA
        events recorded before prep, after prep, after the join and after
        PixelBox (per-stage device times).  With readback buffers, the step's
        sums also land in readback[slot] (read them after an event recorded
        after run() has completed)."""
        self._slot = slot
        if self.graphs is not None and not events:
            self._full[slot if self.readback else 0].replay()
            return self.sums
        for k, stage in enumerate(self._stages):
            if events:
                events[k].record()
            if self.graphs is not None:
                (self._pix_rb[slot] if k == 2 and self.readback else self.graphs[k]).replay()
            else:
                stage()
        if events:
            events[3].record()
        return self.sums

    def check(self):
        """After a run: raise if the pair buffer overflowed, prep flagged input or
        PixelBox flagged a device-side error (the sums' status word)."""
        n, status = (int(v) for v in self.result.tolist())
        if n > self.cap:
            raise SccgError(E_CAPACITY, f"Pipeline: {n} pairs > cap {self.cap}")
        if status:
            raise SccgError(E_ARG, f"Pipeline: prep status bits {status:#x}")
        check_status(self.sums.cpu(), "Pipeline")
        return n


class Study:
    """Many image pairs on one GPU (configs[3]: a multi-image study, "hundreds
    of whole slide images are common"; image-granularity tasks).

    Each image's inputs (xy, offsets of both sets) stay resident in HBM; the
    derived buffers, the pair buffer, the per-pair outputs and the workspaces
    are sized for the largest image and shared -- the images run one after the
    other on one stream (prep, MBR join, PixelBox per image, the async ABI: no
    host sync) and every image's PixelBox adds into ONE device sums vector.  The
    rank's whole pass -- optionally followed by the all-reduce of the sums
    (``allreduce``: a callable enqueued after the last image, e.g. NCCL, which
    graphs can capture) and the read-back -- is ONE CUDA graph.

    images: list of (xy_p, off_p, xy_q, off_q) CUDA tensors (int32 [V, 2], int64 [n + 1])."""

    def __init__(self, images, cap: int | None = None, threshold: int = 0, graph: bool = True, validate: bool = True,
                 raster: bool = True, readback=(), allreduce=None, overlap: bool = True):
        torch = _torch()
        self.lib = lib = load()
        if not images:
            raise ValueError("Study needs at least one image")
        dev = images[0][0].device
        for t4 in images:
            for t, name, dt in zip(t4, ("xy_p", "off_p", "xy_q", "off_q"), (torch.int32, torch.int64, torch.int32,
                                                                            torch.int64)):
                _require_cuda(t, name, dt)
        self.images = list(images)
        dims = [(int(op.numel()) - 1, int(xp.numel()) // 2, int(oq.numel()) - 1, int(xq.numel()) // 2)
                for xp, op, xq, oq in self.images]
        self.n_images = len(dims)
        # shared derived buffers bound per image (the layout is carved from each image's sizes); with overlap,
        # two sets used alternately: image i + 1's prep (HBM-bound) runs on a side stream while image i's join
        # and PixelBox (latency-bound) run on the main one
        self.overlap = bool(overlap) and len(dims) > 1
        nbuf = 2 if self.overlap else 1
        bp = max(int(lib.sccg_polyset_bytes(a, b)) for a, b, _, _ in dims)
        bq = max(int(lib.sccg_polyset_bytes(c, d)) for _, _, c, d in dims)
        self._bufs = [(torch.empty(bp, dtype=torch.uint8, device=dev), torch.empty(bq, dtype=torch.uint8, device=dev))
                      for _ in range(nbuf)]
        self._sets = []
        for i, ((xp, op, xq, oq), (n_p, nv_p, n_q, nv_q)) in enumerate(zip(self.images, dims)):
            cp = PolySet(xp.data_ptr(), op.data_ptr(), n_p, nv_p, None, None, None, None, None, None)
            cq = PolySet(xq.data_ptr(), oq.data_ptr(), n_q, nv_q, None, None, None, None, None, None)
            b = self._bufs[i % nbuf]
            _check(lib.sccg_polyset_bind(ctypes.byref(cp), b[0].data_ptr(), bp), "sccg_polyset_bind")
            _check(lib.sccg_polyset_bind(ctypes.byref(cq), b[1].data_ptr(), bq), "sccg_polyset_bind")
            self._sets.append((PolySet * 2)(cp, cq))
        if self.overlap:
            self._side = torch.cuda.Stream(device=dev)
            self._ev_prep = [torch.cuda.Event() for _ in dims]
            self._ev_done = [torch.cuda.Event() for _ in dims]
        self.cap = int(cap) if cap is not None else max(3 * max(a, c) + 1024 for a, _, c, _ in dims)
        self.pairs = torch.empty((self.cap, 2), dtype=torch.int32, device=dev)
        self.result = torch.zeros(2, dtype=torch.int64, device=dev)
        self.inter = torch.empty(self.cap, dtype=torch.int64, device=dev)  # each image's (I, U) per pair (row a7)
        self.uni = torch.empty(self.cap, dtype=torch.int64, device=dev)
        self.fws_bytes = max(int(lib.sccg_filter_workspace_bytes(a, c)) for a, _, c, _ in dims)
        self.fws = torch.empty(self.fws_bytes, dtype=torch.uint8, device=dev)
        self.pws_bytes = int(lib.sccg_pixelbox_workspace_bytes(self.cap)) + max(
            int(lib.sccg_pixelbox_index_bytes(b, d)) for _, b, _, d in dims)
        self.pws = torch.empty(max(self.pws_bytes, 256), dtype=torch.uint8, device=dev)
        self.sums = new_sums(dev)
        self._zero = new_sums(dev)
        self.cfg = Config(threshold, 0, 0 if raster else FLAG_NO_RASTER, 0, None, None, None)
        self.validate = 1 if validate else 0
        self.readback = tuple(readback)
        self.allreduce = allreduce
        self._slot = 0
        self._graphs = None
        if graph:
            s = torch.cuda.Stream(device=dev)
            s.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(s):  # warm-up outside capture
                self._enqueue()
            torch.cuda.current_stream(dev).wait_stream(s)
            torch.cuda.synchronize(dev)
            self._graphs = []
            for k in range(max(1, len(self.readback))):
                self._slot = k
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._enqueue()
                self._graphs.append(g)

    def _image(self, i, stage):
        lib, st = self.lib, _stream_ptr()
        sets = self._sets[i]
        if stage == 0:
            _check(lib.sccg_prep_sets(sets, 2, self.validate, st), "sccg_prep_sets")
        elif stage == 1:
            _check(lib.sccg_filter_pairs_async(ctypes.byref(sets[0]), ctypes.byref(sets[1]), self.pairs.data_ptr(),
                                               self.cap, self.result.data_ptr(), self.fws.data_ptr(), self.fws_bytes,
                                               st), "sccg_filter_pairs_async")
        else:
            _check(lib.sccg_pixelbox_async(ctypes.byref(sets[0]), ctypes.byref(sets[1]), self.pairs.data_ptr(),
                                           self.result.data_ptr(), self.cap, self.inter.data_ptr(),
                                           self.uni.data_ptr(), self.sums.data_ptr(), ctypes.byref(self.cfg),
                                           self.pws.data_ptr(), self.pws_bytes, st), "sccg_pixelbox_async")

    def _enqueue(self, events=None):
        torch = _torch()
        sums_copy(self._zero, self.sums)
        if self.overlap and events is None:
            main = torch.cuda.current_stream()
            side = self._side
            side.wait_stream(main)  # fork
            for i in range(self.n_images):
                if i >= 2:
                    side.wait_event(self._ev_done[i - 2])  # image i - 2's join and PixelBox are done with this buffer set
                with torch.cuda.stream(side):
                    self._image(i, 0)
                    self._ev_prep[i].record(side)
                main.wait_event(self._ev_prep[i])
                self._image(i, 1)
                self._image(i, 2)
                self._ev_done[i].record(main)
            main.wait_stream(side)  # join
        else:
            for i in range(self.n_images):
                for stage in range(3):
                    if events is not None:
                        events[i][stage].record()
                    self._image(i, stage)
                if events is not None:
                    events[i][3].record()
        if self.allreduce is not None:
            self.allreduce(self.sums)
        if self.readback:
            sums_copy(self.sums, self.readback[self._slot])

    def run(self, events=None, slot: int = 0):
        """One pass over all images (one graph replay).  events: per image four
        CUDA events (before prep, after prep, after the join, after PixelBox):
        that pass is launched eagerly, without the prep overlap, with the
        events between its stages."""
        self._slot = slot
        if self._graphs is not None and events is None:
            self._graphs[slot if self.readback else 0].replay()
        else:
            self._enqueue(events)
        return self.sums

    def check(self):
        """After a run: raise on any device status bit (a join that overflowed
        the pair buffer, invalid input, a PixelBox error) in the summed status."""
        check_status(self.sums.cpu(), "Study")
        return int(self.sums[0])


class Streamer:
    """End-to-end comparison of image pairs arriving in host memory, pipelined.

    Each submitted pair of sets travels host -> device in the packed
    rectilinear encoding (encode_rect_packed: ~0.8 bytes per vertex instead of
    8, and no offsets), is decoded on the GPU (sccg_decode_rect_packed, which
    also rebuilds the offsets) and runs the whole step (a Pipeline graph: prep,
    join, PixelBox, the sums written into pinned host memory by the GPU).
    `depth` slots of device buffers rotate: the host -> device copy of step
    i + 1 runs on a copy stream while step i computes, so a PCIe-bound stream
    of images moves at the link's speed.  Shapes are fixed per slot (n
    polygons and vertices of each set); the encoded buffers grow as needed.

        st = Streamer(A.n, A.nv, B.n, B.nv)
        t = st.submit(packed_a, packed_b)   # encode_rect_packed dicts of pinned tensors
        sums = st.result(t)                 # waits for that step"""

    def __init__(self, n_p: int, nv_p: int, n_q: int, nv_q: int, cap: int | None = None, threshold: int = 0,
                 depth: int = 2, device=None, fused: "PackedStep | None" = None, allreduce=None):
        """fused: a PackedStep whose layout every submit_step shares; the step
        graph's prep then decodes the rings itself (sccg_prep_sets_packed: no
        decode kernels, no read of xy) -- submit_step only.  allreduce: the
        multi-GPU step's collective (e.g. dist.allreduce_sums over NCCL),
        captured in each slot's step graph before the read-back."""
        torch = _torch()
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.depth = depth
        self.shapes = (n_p, nv_p, n_q, nv_q)
        self.fused = fused
        cap = int(cap) if cap is not None else 3 * max(n_p, n_q) + 1024
        self.slots = []
        for _ in range(depth):
            sl = {}
            for side, n, nv in (("p", n_p, nv_p), ("q", n_q, nv_q)):
                sl["off_" + side] = torch.zeros(n + 1, dtype=torch.int64, device=dev)
                sl["xy_" + side] = torch.empty((max(nv, 1), 2), dtype=torch.int32, device=dev)
                sl["enc_" + side] = {}
            sl["rb"] = torch.zeros(len(SUMS_FIELDS), dtype=torch.int64).pin_memory()
            P = DeviceSet(sl["xy_p"][:nv_p], sl["off_p"], prep=False)
            Q = DeviceSet(sl["xy_q"][:nv_q], sl["off_q"], prep=False)
            sl["sets"] = (P, Q)
            packed = None
            if fused is not None:  # the slot's step buffer at a fixed address, captured in the graph
                # zeroed: the graph capture's warm-up run decodes it (all rings empty)
                sl["step_buf"] = torch.zeros(max(fused.nbytes, 16), dtype=torch.uint8, device=dev)
                v = fused.views(sl["step_buf"])
                sl["step_views"] = v
                packed = (v["p"], v["q"])
            sl["pipe"] = Pipeline(P, Q, cap=cap, threshold=threshold, graph=True, readback=[sl["rb"]], packed=packed,
                                  allreduce=allreduce)
            sl["copied"], sl["done"], sl["decoded"] = torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()
            self.slots.append(sl)
        self.copy_stream = torch.cuda.Stream(device=dev)
        self.decode_stream = torch.cuda.Stream(device=dev)
        self.count = 0

    def submit(self, enc_p, enc_q) -> int:
        """Enqueue one step for host sets given as encode_rect_packed dicts of
        (pinned) CPU tensors.  Returns a ticket for result()."""
        torch = _torch()
        k = self.count % self.depth
        sl = self.slots[k]
        main = torch.cuda.current_stream()
        cs = self.copy_stream
        cs.wait_event(sl["done"])  # the slot's previous step no longer reads its buffers
        n_p, nv_p, n_q, nv_q = self.shapes
        views = {}
        with torch.cuda.stream(cs):
            for side, enc, n in (("p", enc_p, n_p), ("q", enc_q, n_q)):
                if int(enc["head"].numel()) != n:
                    raise ValueError(f"Streamer: set {side} has {int(enc['head'].numel())} rings, the slots {n}")
                buf, v = sl["enc_" + side], {}
                for key, t in enc.items():
                    if key not in buf or buf[key].numel() < t.numel():
                        buf[key] = torch.empty(max(t.numel(), 1), dtype=t.dtype, device=self.device)
                    d = buf[key].view(-1)[: t.numel()].view(t.shape)
                    if t.numel():
                        d.copy_(t, non_blocking=True)
                    v[key] = d
                views[side] = v
            sl["copied"].record(cs)
        main.wait_event(sl["copied"])
        for side, nv in (("p", nv_p), ("q", nv_q)):
            decode_rect_packed(views[side], nv, out=(sl["xy_" + side], sl["off_" + side]))
        sl["pipe"].run(slot=0)
        sl["done"].record(main)
        self.count += 1
        return self.count - 1

    def submit_step(self, step: "PackedStep") -> int:
        """Enqueue one step whose inputs are a PackedStep (both sets in one
        pinned buffer: one host -> device copy).  Returns a ticket for result()."""
        torch = _torch()
        k = self.count % self.depth
        sl = self.slots[k]
        main = torch.cuda.current_stream()
        cs = self.copy_stream
        n_p, nv_p, n_q, nv_q = self.shapes
        if step.n["p"] != n_p or step.n["q"] != n_q:
            raise ValueError("Streamer: the step's ring counts differ from the slots'")
        if self.fused is not None and (step.nbytes != self.fused.nbytes or step.layout != self.fused.layout):
            raise ValueError("Streamer(fused=...): the step's packed layout differs from the slots'")
        cs.wait_event(sl["done"])  # the slot's previous step no longer reads its buffers
        with torch.cuda.stream(cs):
            buf = sl.get("step_buf")
            if buf is None or buf.numel() < step.nbytes:
                buf = sl["step_buf"] = torch.empty(max(step.nbytes, 16), dtype=torch.uint8, device=self.device)
            buf[: step.nbytes].copy_(step.host[: step.nbytes], non_blocking=True)
            sl["copied"].record(cs)
        if self.fused is not None:  # prep decodes inside the step graph
            main.wait_event(sl["copied"])
            sl["pipe"].run(slot=0)
            sl["done"].record(main)
            self.count += 1
            return self.count - 1
        # the decode runs on its own stream: step i + 1's decode overlaps step i's graph
        ds = self.decode_stream
        ds.wait_event(sl["copied"])
        v = step.views(buf)
        with torch.cuda.stream(ds):
            for side, nv in (("p", nv_p), ("q", nv_q)):
                decode_rect_packed(v[side], nv, stream=ds, out=(sl["xy_" + side], sl["off_" + side]))
            sl["decoded"].record(ds)
        main.wait_event(sl["decoded"])
        sl["pipe"].run(slot=0)
        sl["done"].record(main)
        self.count += 1
        return self.count - 1

    def result(self, ticket: int):
        """The sums of step `ticket` (waits for it; its slot must not have been
        reused since: at most `depth` steps in flight)."""
        if ticket < self.count - self.depth:
            raise ValueError("Streamer: that step's slot has been reused")
        sl = self.slots[ticket % self.depth]
        sl["done"].synchronize()
        return sums_to_host(sl["rb"])


def pin_packed(enc):
    """An encode_rect_packed dict as pinned CPU tensors (Streamer.submit's input)."""
    import numpy as np

    torch = _torch()
    return {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in enc.items()}


class PackedStep:
    """Both sets' packed encodings of one step in ONE pinned host buffer (16-byte
    aligned fields), so a step's inputs cross PCIe as one copy
    (Streamer.submit_step).  layout[side][key] = (byte offset, dtype, shape)."""

    _KEYS = ("head", "vlen", "start", "units", "block")

    def __init__(self, enc_p, enc_q):
        import numpy as np

        torch = _torch()
        self.layout, off, parts = {}, 0, []
        for side, enc in (("p", enc_p), ("q", enc_q)):
            lay = {}
            for k in self._KEYS:
                a = np.ascontiguousarray(enc[k])
                lay[k] = (off, a.dtype, a.shape)
                parts.append((off, a))
                off += (a.nbytes + 15) & ~15
            self.layout[side] = lay
        self.nbytes = off
        self.host = torch.empty(max(off, 16), dtype=torch.uint8)
        if torch.cuda.is_available():
            self.host = self.host.pin_memory()
        hv = self.host.numpy()
        for o, a in parts:
            hv[o: o + a.nbytes] = a.view(np.uint8).reshape(-1)
        self.n = {side: int(self.layout[side]["head"][2][0]) for side in ("p", "q")}

    def views(self, dev_buf):
        """Typed views of a device byte buffer holding a copy of self.host."""
        import numpy as np

        torch = _torch()
        tmap = {np.dtype(np.uint16): torch.int16, np.dtype(np.int16): torch.int16, np.dtype(np.int64): torch.int64,
                np.dtype(np.uint8): torch.uint8}
        out = {}
        for side, lay in self.layout.items():
            out[side] = {}
            for k, (o, dt, shape) in lay.items():
                nb = int(np.prod(shape)) * np.dtype(dt).itemsize
                out[side][k] = dev_buf[o: o + nb].view(tmap[np.dtype(dt)]).view(shape)
        return out


def touches(P: DeviceSet, Q: DeviceSet, pairs, inter, stream=None):
    """ST_Touches (reading R21) per pair: uint8 [N], 1 iff |p n q| == 0
    (inter: the pairs' intersections from pixelbox) and the boundaries meet.
    Use pairs from filter_pairs(..., closed=True)."""
    torch = _torch()
    _require_cuda(pairs, "pairs", torch.int32)
    _require_cuda(inter, "inter", torch.int64)
    n = int(pairs.shape[0])
    out = torch.empty(n, dtype=torch.uint8, device=pairs.device)
    _check(load().sccg_touches(ctypes.byref(P.c), ctypes.byref(Q.c), pairs.data_ptr(), n, inter.data_ptr(),
                               out.data_ptr(), _stream_ptr(stream)), "sccg_touches")
    return out


def new_sums(device=None):
    """A zeroed device sums vector (int64[11], the sccg_sums layout)."""
    torch = _torch()
    return torch.zeros(len(SUMS_FIELDS), dtype=torch.int64, device=device or "cuda")


def pixelbox(P: DeviceSet, Q: DeviceSet, pairs, threshold: int = 0, mode: int = 0, sums=None, want_inter=True,
             want_union=True, counters=None, grid: int = 0, hits=None, raster: bool = True, paper_split: bool = False,
             stream=None, check: bool = True, index: bool = True):
    """Per-pair |p n q| and |p u q| (int64, input order) + accumulated sums.
    check: read the sums' status word after the call (one sync) and raise
    SccgError if a device-side error was flagged (check=False: stay async).
    paper_split: push every continuing sub-box (Alg. 1 as written) instead of
    pixelizing dense splits whole (SCCG_FLAG_PAPER_SPLIT; same results).
    hits = (hit_p, hit_q): optional int32 bitmaps (new_hits) marking polygons
    with a non-zero intersection, for missing_polygons()."""
    torch = _torch()
    lib = load()
    _require_cuda(pairs, "pairs", torch.int32)
    n = int(pairs.shape[0])
    dev = P.xy.device
    inter = torch.empty(n, dtype=torch.int64, device=dev) if want_inter else None
    uni = torch.empty(n, dtype=torch.int64, device=dev) if want_union else None
    if sums is None:
        sums = new_sums(dev)
    _require_cuda(sums, "sums", torch.int64)
    cfg = Config(threshold, mode, (0 if raster else FLAG_NO_RASTER) | (FLAG_PAPER_SPLIT if paper_split else 0), grid,
                 counters.data_ptr() if counters is not None else None,
                 hits[0].data_ptr() if hits is not None else None, hits[1].data_ptr() if hits is not None else None)
    wsb = int(lib.sccg_pixelbox_workspace_bytes(n)) + (int(lib.sccg_pixelbox_index_bytes(P.nv, Q.nv)) if index else 0)
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)
    code = lib.sccg_pixelbox(ctypes.byref(P.c), ctypes.byref(Q.c), pairs.data_ptr(), n,
                             inter.data_ptr() if inter is not None else None,
                             uni.data_ptr() if uni is not None else None, sums.data_ptr(), ctypes.byref(cfg),
                             ws.data_ptr(), wsb, _stream_ptr(stream))
    _check(code, "sccg_pixelbox")
    if check:
        check_status(sums, "sccg_pixelbox")
    return inter, uni, sums


def check_status(sums, where="sums"):
    """Raise SccgError if a sums vector carries device status bits (one sync)."""
    st = int(sums[10]) if not isinstance(sums, Sums) else int(sums.status)
    if st:
        code = (E_ARG if st & STATUS_ARG else E_NOT_RECTILINEAR if st & STATUS_NOT_RECTILINEAR else
                E_RANGE if st & STATUS_RANGE else E_STACK if st & STATUS_STACK else
                E_CAPACITY if st & STATUS_CAPACITY else E_ARG)
        raise SccgError(code, f"{where}: device status bits {st:#x}")


def new_hits(P: "DeviceSet", Q: "DeviceSet"):
    """Zeroed hit bitmaps (int32 words) for sets P and Q."""
    torch = _torch()
    dev = P.xy.device
    return (torch.zeros((P.n + 31) // 32 + 1, dtype=torch.int32, device=dev),
            torch.zeros((Q.n + 31) // 32 + 1, dtype=torch.int32, device=dev))


def missing_polygons(hits, P: "DeviceSet", Q: "DeviceSet", stream=None) -> tuple[int, int]:
    """(missing in P, missing in Q): polygons with no intersecting counterpart
    (P:63), from the bitmaps pixelbox(..., hits=...) filled."""
    torch = _torch()
    lib = load()
    out = torch.zeros(2, dtype=torch.int64, device=P.xy.device)
    _check(lib.sccg_count_missing(hits[0].data_ptr(), P.n, out.data_ptr(), _stream_ptr(stream)), "sccg_count_missing")
    _check(lib.sccg_count_missing(hits[1].data_ptr(), Q.n, out.data_ptr() + 8, _stream_ptr(stream)),
           "sccg_count_missing")
    a, b = out.tolist()
    return int(a), int(b)


def contains(P: DeviceSet, Q: DeviceSet, pairs, inter, stream=None):
    """ST_Contains by areas (sccg_contains): uint8 [N], bit 0 = p
    contains q (|p n q| == |q| > 0), bit 1 = q contains p; inter from pixelbox."""
    torch = _torch()
    _require_cuda(pairs, "pairs", torch.int32)
    _require_cuda(inter, "inter", torch.int64)
    n = int(pairs.shape[0])
    out = torch.empty(n, dtype=torch.uint8, device=pairs.device)
    _check(load().sccg_contains(ctypes.byref(P.c), ctypes.byref(Q.c), pairs.data_ptr(), n, inter.data_ptr(),
                                out.data_ptr(), _stream_ptr(stream)), "sccg_contains")
    return out


def tile_report(P: DeviceSet, Q: DeviceSet, pairs, inter, uni, hits, tiling, tiles=None, stream=None):
    """Per-tile report (sccg_report): int64 [ntx * nty, 15]
    device tensor (fields REPORT_FIELDS), accumulated into `tiles` if given.
    tiling = Tiling or (x0, y0, tile_w, tile_h, ntx, nty)."""
    torch = _torch()
    t = tiling if isinstance(tiling, Tiling) else Tiling(*tiling)
    n = int(pairs.shape[0])
    if tiles is None:
        tiles = torch.zeros((t.ntx * t.nty, len(REPORT_FIELDS)), dtype=torch.int64, device=P.xy.device)
    _check(load().sccg_report(ctypes.byref(P.c), ctypes.byref(Q.c), pairs.data_ptr() if n else None, n,
                              inter.data_ptr() if n else None, uni.data_ptr() if n else None, hits[0].data_ptr(),
                              hits[1].data_ptr(), ctypes.byref(t), tiles.data_ptr(), _stream_ptr(stream)),
           "sccg_report")
    return tiles


def similarity_report(P: DeviceSet, Q: DeviceSet, pairs, inter, uni, hits, tiling, stream=None) -> dict:
    """The SimilarityReport of SPEC S:343-346 from one image's pairs: per tile
    {tile_id, pairs, intersecting, jaccard, ratio_limbs, missing_p, missing_q,
    polygons_p, polygons_q}, the image J' (Eq. 1 over all pairs) and the totals."""
    tiles = tile_report(P, Q, pairs, inter, uni, hits, tiling, stream=stream).cpu().tolist()
    per_tile = []
    tot = [0] * 11
    for tid, row in enumerate(tiles):
        s = Sums(*row[:11])
        j, _ = jaccard(s)
        per_tile.append(dict(tile_id=tid, pairs=row[0], intersecting=row[1], jaccard=None if math.isnan(j) else j,
                             ratio_limbs=row[6:10], polygons_p=row[11], polygons_q=row[12], missing_p=row[13],
                             missing_q=row[14]))
        tot = [a + b for a, b in zip(tot, row[:11])]
    j, pooled = jaccard(Sums(*tot))
    return dict(tiles=per_tile, jaccard=None if math.isnan(j) else j, pooled=None if math.isnan(pooled) else pooled,
                pairs=tot[0], intersecting=tot[1], polygons_p=P.n, polygons_q=Q.n,
                missing_p=sum(t["missing_p"] for t in per_tile), missing_q=sum(t["missing_q"] for t in per_tile))


def sums_pack(sums, vec=None, stream=None):
    """sccg_sums_pack: the REDUCE_WORDS int64 all-reduce vector of a device sums vector."""
    torch = _torch()
    if vec is None:
        vec = torch.empty(REDUCE_WORDS, dtype=torch.int64, device=sums.device)
    _check(load().sccg_sums_pack(sums.data_ptr(), vec.data_ptr(), _stream_ptr(stream)), "sccg_sums_pack")
    return vec


def sums_unpack(vec, sums, stream=None):
    """sccg_sums_unpack: sums (device int64 [11]) from a (reduced) vector."""
    _check(load().sccg_sums_unpack(vec.data_ptr(), sums.data_ptr(), _stream_ptr(stream)), "sccg_sums_unpack")
    return sums


def sums_to_host(sums) -> Sums:
    vals = [int(v) for v in (sums.tolist() if hasattr(sums, "tolist") else sums)]
    return Sums(*vals)


def sums_copy(src, dst, stream=None):
    """Enqueue a copy of the sums vector `src` (device int64 [11]) into `dst`
    (device tensor, or a pinned host tensor the GPU writes directly): one
    single-warp kernel instead of a copy-engine transfer (sccg_sums_copy)."""
    _check(load().sccg_sums_copy(src.data_ptr(), dst.data_ptr(), _stream_ptr(stream)), "sccg_sums_copy")
    return dst


def jaccard(sums) -> tuple[float, float]:
    """(J', pooled) from a sums vector (device tensor, list or Sums); NaN if empty."""
    lib = load()
    s = sums if isinstance(sums, Sums) else sums_to_host(sums)
    j, pooled = ctypes.c_double(), ctypes.c_double()
    code = lib.sccg_jaccard(ctypes.byref(s), ctypes.byref(j), ctypes.byref(pooled))
    if code == E_EMPTY:
        return math.nan, math.nan
    _check(code, "sccg_jaccard")  # sums carrying device status bits are rejected
    return j.value, pooled.value


def encode_rect(xy, offsets):
    """Compact rectilinear rings for the host -> device transfer (sccg_decode_rect):
    (start int32 [n, 2], move int16 [V - n], first_vertical uint8 [n]) with
    2 bytes per vertex after each ring's first, or None when some ring is not
    encodable (a zero-length or non-alternating move, a move beyond int16, an
    empty ring).  Host-side numpy; lossless: the device decode is exact."""
    import numpy as np

    xy = np.asarray(xy, np.int64).reshape(-1, 2)
    off = np.asarray(offsets, np.int64)
    n = off.shape[0] - 1
    V = np.diff(off)
    if n == 0:
        return np.zeros((0, 2), np.int32), np.zeros(0, np.int16), np.zeros(0, np.uint8)
    if (V < 1).any():
        return None
    d = np.diff(xy, axis=0)  # d[j] = xy[j + 1] - xy[j]
    first = np.zeros(xy.shape[0], bool)
    first[off[:-1]] = True
    keep = ~first[1:]  # moves within a ring: vertex j + 1 is not a ring start
    mv = d[keep]
    ring = np.repeat(np.arange(n), V - 1)
    k = np.arange(mv.shape[0]) - np.repeat(off[:-1] - np.arange(n), V - 1) + 1  # vertex index in its ring (>= 1)
    vert_move = mv[:, 0] == 0
    if ((mv[:, 0] != 0) == (mv[:, 1] != 0)).any():  # exactly one coordinate changes
        return None
    fv = np.zeros(n, np.uint8)
    has = V > 1
    fv[has] = vert_move[(off[:-1] - np.arange(n))[has]]
    expect_vert = ((k & 1) == 1) == (fv[ring] == 1)
    if (vert_move != expect_vert).any():
        return None
    m = np.where(vert_move, mv[:, 1], mv[:, 0])
    if m.size and (np.abs(m).max() > 32767):
        return None
    start = xy[off[:-1]].astype(np.int32)
    return start, m.astype(np.int16), fv


def decode_rect(start, move, first_vertical, offsets, stream=None):
    """sccg_decode_rect on device tensors: the plain int32 [V, 2] vertices."""
    torch = _torch()
    n = int(offsets.numel()) - 1
    nv = int(offsets[-1].item()) if n > 0 else 0
    xy = torch.empty((max(nv, 1), 2), dtype=torch.int32, device=offsets.device)
    _check(load().sccg_decode_rect(start.data_ptr(), move.data_ptr() if move.numel() else None,
                                   first_vertical.data_ptr(), offsets.data_ptr(), n, xy.data_ptr(), _stream_ptr(stream)),
           "sccg_decode_rect")
    return xy[:nv]


RECTP_BLOCK = 256  # SCCG_RECTP_BLOCK


def encode_rect_packed(xy, offsets, vlc: bool = True):
    """Packed rectilinear rings (sccg_decode_rect_packed, format 2 in
    include/sccg.h): dict of numpy arrays head uint16 [n], vlen uint8 [n],
    start int16 [...], units uint16 [...], block int64 [ceil(n / 256), 4] --
    each ring's moves variable-length coded (class 3: exp-Golomb symbols of
    magnitude and sign flip, ~2.2 bits per move on segmentation contours) or,
    where that cannot hold them, at the narrowest of 4, 8 or 16 bits; starts as
    int16 deltas from the block's first start where they fit; no offsets.
    vlc=False keeps the fixed widths only.  None when some ring is not
    encodable (more than 8191 vertices, a zero-length or non-alternating move,
    a move beyond int16).  Host-side numpy; lossless: the device decode is
    exact.  Rings with 0 vertices are allowed."""
    import numpy as np

    xy = np.asarray(xy, np.int64).reshape(-1, 2)
    off = np.asarray(offsets, np.int64)
    n = off.shape[0] - 1
    V = np.diff(off)
    if n < 0 or (V < 0).any() or (V > 8191).any():
        return None
    m = np.maximum(V - 1, 0)  # moves per ring
    nm = int(m.sum())
    ring = np.repeat(np.arange(n), m)
    # move j of ring i: xy[off[i] + j + 1] - xy[off[i] + j]
    mstart = np.cumsum(m) - m
    j = np.arange(nm) - np.repeat(mstart, m)
    src = np.repeat(off[:-1], m) + j
    d = xy[src + 1] - xy[src] if nm else np.zeros((0, 2), np.int64)
    if ((d[:, 0] != 0) == (d[:, 1] != 0)).any():  # exactly one coordinate changes
        return None
    ymove = d[:, 0] == 0
    fv = np.zeros(n, np.int64)
    has = m > 0
    fv[has] = ymove[mstart[has]]
    if (ymove != (((j & 1) == 0) == (fv[ring] == 1))).any():  # the axes alternate
        return None
    mv = np.where(ymove, d[:, 1], d[:, 0])
    a = np.abs(mv)
    if nm and a.max() > 32767:
        return None
    amax = np.zeros(n, np.int64)
    if nm:
        np.maximum.at(amax, ring, a)
    w = np.where(amax <= 8, 0, np.where(amax <= 128, 1, 2))
    # variable-length class: symbol 2 (|d| - 1) + flip (sign vs the previous move on the same axis, the first
    # one on each axis vs +), exp-Golomb LSB first (2 L + 1 bits, L = floor(log2(symbol + 1)))
    neg = (mv < 0).astype(np.int64)
    prev = np.zeros(nm, np.int64)
    back2 = j >= 2
    prev[back2] = neg[np.nonzero(back2)[0] - 2]
    sym = 2 * (a - 1) + (neg ^ prev)
    v = sym + 1
    L = np.zeros(nm, np.int64)
    if nm:
        L = np.floor(np.log2(v.astype(np.float64))).astype(np.int64)
        L += (np.left_shift(1, L + 1) <= v).astype(np.int64)  # guard float rounding
        L -= (np.left_shift(1, L) > v).astype(np.int64)
    ln = 2 * L + 1
    code = np.left_shift(1, L) | np.left_shift(v & (np.left_shift(1, L) - 1), L + 1)
    rbits = np.bincount(ring, weights=ln, minlength=n).astype(np.int64) if nm else np.zeros(n, np.int64)
    vunits = (rbits + 15) // 16
    if vlc:
        w = np.where((amax <= 127) & (vunits <= 255) & (m > 0), 3, w)
    c = np.array([4, 2, 1, 1])[w]
    nu = np.where(w == 3, vunits, (m + c - 1) // c)
    u0 = np.cumsum(nu) - nu  # global unit offset of each ring
    head = (V | (w << 13) | (fv << 15)).astype(np.uint16)
    vlen = np.where(w == 3, vunits, 0).astype(np.uint8)
    units = np.zeros(int(nu.sum()), np.int64)
    wr = w[ring]
    # fixed classes: 4-bit nibbles of a flat array, 4 per unit
    fx = wr < 3
    nib = np.zeros(4 * units.shape[0], np.int64)
    cr = c[ring]
    pos = 4 * (u0[ring] + j // cr) + (j % cr) * (4 // cr)
    small = fx & (wr < 2)
    bits = np.where(wr == 0, 4, 8)
    fcode = np.where(mv < 0, 1, 0) << (bits - 1) | (a - 1)
    for k in range(2):  # an 8-bit code spans two nibbles
        sel = small & ((wr == 1) | (k == 0))
        nib[pos[sel] + k] = (fcode[sel] >> (4 * k)) & 15
    big = fx & (wr == 2)
    v16 = mv[big] & 0xFFFF
    for k in range(4):
        nib[pos[big] + k] = (v16 >> (4 * k)) & 15
    units |= nib[0::4] | nib[1::4] << 4 | nib[2::4] << 8 | nib[3::4] << 12
    # variable-length class: each code at its ring's bit offset (a code spans at most two units)
    vl = wr == 3
    if vl.any():
        bo = np.cumsum(ln) - ln - np.repeat(np.cumsum(rbits) - rbits, m)  # bit offset of each move in its ring
        bp = 16 * u0[ring] + bo
        sel = np.nonzero(vl)[0]
        ui, sh, cd = bp[sel] >> 4, bp[sel] & 15, code[sel]
        np.bitwise_or.at(units, ui, (cd << sh) & 0xFFFF)
        spill = sh + ln[sel] > 16
        np.bitwise_or.at(units, ui[spill] + 1, cd[spill] >> (16 - sh[spill]))
    units = units.astype(np.uint16)
    # starts: per block of RECTP_BLOCK rings, int16 deltas from its first start or int32 pairs
    nb = (n + RECTP_BLOCK - 1) // RECTP_BLOCK
    block = np.zeros((max(nb, 0), 4), np.int64)
    st = np.zeros((n, 2), np.int64)
    st[V > 0] = xy[off[:-1][V > 0]]
    parts, soff = [], 0
    for b in range(nb):
        lo, hi = b * RECTP_BLOCK, min(n, (b + 1) * RECTP_BLOCK)
        s = st[lo:hi]
        x0, y0 = int(s[0, 0]), int(s[0, 1])
        dd = s - np.array([x0, y0])
        wide = bool((np.abs(dd) > 32767).any())
        if wide:
            p = (s.astype(np.int64) & 0xFFFFFFFF)
            part = np.stack([p[:, 0] & 0xFFFF, p[:, 0] >> 16, p[:, 1] & 0xFFFF, p[:, 1] >> 16], 1).reshape(-1)
        else:
            part = (dd & 0xFFFF).reshape(-1)
        org = (x0 & 0xFFFFFFFF) | ((y0 & 0xFFFFFFFF) << 32)
        block[b] = (off[lo], u0[lo], soff | (int(wide) << 62), org - (1 << 64) if org >= 1 << 63 else org)
        parts.append(part.astype(np.uint16))
        soff += part.shape[0]
    start = (np.concatenate(parts) if parts else np.zeros(0, np.uint16)).view(np.int16)
    return dict(head=head, vlen=vlen, start=start, units=units, block=block)


def decode_rect_packed(enc, n_vertices: int, stream=None, out=None):
    """sccg_decode_rect_packed on device tensors (the dict of encode_rect_packed
    moved to the device): returns (xy int32 [V, 2], offsets int64 [n + 1]).
    out = (xy, offsets) device buffers to fill instead of allocating."""
    torch = _torch()
    head = enc["head"]
    n = int(head.numel())
    dev = head.device
    if out is None:
        xy = torch.empty((max(n_vertices, 1), 2), dtype=torch.int32, device=dev)
        off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    else:
        xy, off = out
    ptr = lambda t: t.data_ptr() if t.numel() else None  # noqa: E731
    vl = enc.get("vlen")
    _check(load().sccg_decode_rect_packed(ptr(head), ptr(vl) if vl is not None else None, ptr(enc["start"]),
                                          ptr(enc["units"]), ptr(enc["block"]), n, off.data_ptr(), xy.data_ptr(),
                                          _stream_ptr(stream)),
           "sccg_decode_rect_packed")
    return xy[:n_vertices], off


def to_device(xy, offsets, device="cuda", non_blocking=True):
    """Copy host numpy / tensor arrays (pinned if possible) to the GPU."""
    torch = _torch()
    xy_t = torch.as_tensor(xy).to(torch.int32)
    off_t = torch.as_tensor(offsets).to(torch.int64)
    return (xy_t.reshape(-1, 2).to(device, non_blocking=non_blocking),
            off_t.to(device, non_blocking=non_blocking))


def compare(xy_p, off_p, xy_q, off_q, threshold: int = 0, device="cuda", stream=None) -> dict:
    """End-to-end cross-comparison of two host polygon sets (the public API):
    H2D copy, prep, MBR join, PixelBox, sums D2H, J'.  Returns a report dict."""
    dxp, dop = to_device(xy_p, off_p, device)
    dxq, doq = to_device(xy_q, off_q, device)
    P = DeviceSet(dxp, dop, stream=stream)
    Q = DeviceSet(dxq, doq, stream=stream)
    pairs = filter_pairs(P, Q, stream=stream)
    _, _, sums = pixelbox(P, Q, pairs, threshold=threshold, want_inter=False, want_union=False, stream=stream,
                          check=False)
    host = sums_to_host(sums.cpu())
    check_status(host, "compare")
    j, pooled = jaccard(host)
    return dict(jprime=j, pooled=pooled, **{f: getattr(host, f) for f in SUMS_FIELDS})
