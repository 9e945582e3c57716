"""Python mirror of the reference's hot-path API, backed by the sm_100a C ABI.

Reference interface (paths under /root/reference/proj)      ->  here
  lamina::parseLayout(text, schema, extents)  layout_spec.hpp:19 ->  parse_layout / Layout
  lamina::View(MappingPtr) / View(m, blobs)   view.hpp:108-111   ->  View(layout) / View(layout, blobs=...)
  lamina::copyView(const View&, View&)        view.hpp:285       ->  copy_view(src, dst)
  FieldAccessCount::counters()/reset()        instrument.hpp:56  ->  View.counters() / View.reset_counters()
  Heatmap::blockCounter / totalTouches        instrument.hpp:112 ->  View.heatmap(nr)
  View::read / View::write                    view.hpp:144-149   ->  View.read_values / View.write_values
  writeFieldAccessCsv / writeHeatmapCsv       instrument.hpp:131 ->  field_access_csv / heatmap_csv

Exceptions mirror the reference's exception types (std::invalid_argument ->
InvalidArgument(ValueError), std::out_of_range -> OutOfRange(IndexError),
std::overflow_error -> IndexTypeOverflow(OverflowError), std::logic_error ->
LogicError(RuntimeError)) with the reference's message text.
"""
from __future__ import annotations

import ctypes as C
from typing import Iterable, Sequence

import numpy as np

from ._lib import lib

# scalar kinds (scalar.hpp:16-29)
I8, I16, I32, I64, U8, U16, U32, U64, F32, F64, BOOL = range(11)
SCALAR_NAMES = ("i8", "i16", "i32", "i64", "u8", "u16", "u32", "u64", "f32", "f64", "bool")
SCALAR_SIZE = (1, 2, 4, 8, 1, 2, 4, 8, 4, 8, 1)

WRAP_FIELD_ACCESS_COUNT = 1
WRAP_HEATMAP = 2
NBODY_EXACT = 0
NBODY_FAST = 1


class LaminaError(Exception):
    pass


class InvalidArgument(LaminaError, ValueError):
    pass


class OutOfRange(LaminaError, IndexError):
    pass


class IndexTypeOverflow(LaminaError, OverflowError):
    pass


class LogicError(LaminaError, RuntimeError):
    pass


class CudaError(LaminaError, RuntimeError):
    pass


class ReferenceRuntimeError(LaminaError, RuntimeError):
    """std::runtime_error in the reference (e.g. readViewDump's "cannot read")."""


_ERR = {1: InvalidArgument, 2: OutOfRange, 3: IndexTypeOverflow, 4: LogicError, 5: ReferenceRuntimeError,
        6: CudaError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().lam_last_error().decode()
        raise _ERR.get(rc, LaminaError)(msg)


def _stream_handle(stream) -> C.c_void_p:
    if stream is None:
        return C.c_void_p(0)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    h = getattr(stream, "cuda_stream", None)  # torch.cuda.Stream
    if h is not None:
        return C.c_void_p(h)
    raise TypeError(f"unsupported stream object {stream!r}")


def _str(fn, handle, *extra) -> str:
    n = fn(handle, *extra, None, 0)
    buf = C.create_string_buffer(n + 1)
    fn(handle, *extra, buf, n + 1)
    return buf.value.decode()


class Layout:
    """A lowered mapping: schema + extents + layout grammar (+ instrumentation wrappers)."""

    def __init__(self, schema: str, extents: str, layout: str, dyn: Sequence[int] = (), wrap: int = 0,
                 granularity: int = 0):
        L = lib()
        arr = (C.c_uint64 * max(1, len(dyn)))(*dyn)
        h = C.c_void_p()
        _check(L.lam_layout_create(schema.encode(), extents.encode(), arr, len(dyn), layout.encode(), wrap,
                                   granularity, C.byref(h)))
        self._h = h
        self.layout_text = layout
        self.dyn = tuple(dyn)

    @classmethod
    def _adopt(cls, handle: C.c_void_p) -> "Layout":
        self = cls.__new__(cls)
        self._h = handle
        self.layout_text = _str(lib().lam_layout_name, handle)
        self.dyn = ()
        return self

    def contiguous_run(self, linear: int, leaf: int, n: int):
        """Mapping::contiguousRun: (nr, offset) when n values of the leaf are contiguous, else None."""
        has, nr, off = C.c_int(), C.c_size_t(), C.c_uint64()
        _check(lib().lam_layout_contiguous_run(self._h, linear, leaf, n, C.byref(has), C.byref(nr), C.byref(off)))
        return (nr.value, off.value) if has.value else None

    def dump_meta(self) -> str:
        """The .meta sidecar text writeViewDump writes for a view of this layout (view_io.cpp:30-44)."""
        return _str(lib().lam_layout_dump_meta, self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().lam_layout_destroy(h)
            except TypeError:  # interpreter shutdown: module globals already torn down
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def name(self) -> str:
        return _str(lib().lam_layout_name, self._h)

    @property
    def schema(self) -> str:
        return _str(lib().lam_layout_schema, self._h)

    @property
    def extents(self) -> str:
        return _str(lib().lam_layout_extents, self._h)

    @property
    def blob_count(self) -> int:
        return lib().lam_layout_blob_count(self._h)

    def blob_size(self, nr: int) -> int:
        return lib().lam_layout_blob_size(self._h, nr)

    @property
    def blob_sizes(self) -> list[int]:
        return [self.blob_size(k) for k in range(self.blob_count)]

    @property
    def element_count(self) -> int:
        return lib().lam_layout_element_count(self._h)

    @property
    def leaf_count(self) -> int:
        return lib().lam_layout_leaf_count(self._h)

    def leaf(self, f: int) -> tuple[int, int, int]:
        k, s, o = C.c_int(), C.c_size_t(), C.c_size_t()
        _check(lib().lam_layout_leaf(self._h, f, C.byref(k), C.byref(s), C.byref(o)))
        return k.value, s.value, o.value

    def leaf_path(self, f: int) -> str:
        return _str(lib().lam_layout_leaf_path, self._h, f)

    @property
    def leaf_types(self) -> list[int]:
        return [self.leaf(f)[0] for f in range(self.leaf_count)]

    def is_computed(self, f: int) -> bool:
        return bool(lib().lam_layout_is_computed(self._h, f))

    @property
    def is_fully_physical(self) -> bool:
        return bool(lib().lam_layout_is_fully_physical(self._h))

    @property
    def has_mutable_state(self) -> bool:
        return bool(lib().lam_layout_has_mutable_state(self._h))

    @property
    def is_fully_static(self) -> bool:
        return bool(lib().lam_layout_is_fully_static(self._h))

    @property
    def runtime_state_bytes(self) -> int:
        return int(lib().lam_layout_runtime_state_bytes(self._h))

    def physical_offset(self, linear: int, f: int) -> tuple[int, int]:
        nr, off = C.c_size_t(), C.c_uint64()
        _check(lib().lam_layout_physical_offset(self._h, linear, f, C.byref(nr), C.byref(off)))
        return nr.value, off.value

    def heatmap_blocks(self, nr: int) -> int:
        return lib().lam_layout_heatmap_blocks(self._h, nr)

    @property
    def shard_unit(self) -> int:
        return lib().lam_layout_shard_unit(self._h)

    @property
    def stream_count(self) -> int:
        return lib().lam_layout_stream_count(self._h)

    def stream_region(self, stream: int, begin: int, end: int) -> tuple[int, int, int]:
        """(blob nr, lo, hi): bytes of blob nr that elements [begin, end) occupy in `stream`."""
        nr, lo, hi = C.c_size_t(), C.c_uint64(), C.c_uint64()
        _check(lib().lam_layout_stream_region(self._h, stream, begin, end, C.byref(nr), C.byref(lo), C.byref(hi)))
        return nr.value, lo.value, hi.value

    def __repr__(self):
        return f"Layout({self.name!r}, {self.schema!r}, {self.extents!r})"


def parse_layout(text: str, schema: str, extents: str, dyn: Sequence[int] = ()) -> Layout:
    """lamina::parseLayout (layout_spec.cpp:164-167)."""
    return Layout(schema, extents, text, dyn)


class View:
    """Device view: blobs in HBM on `device` + the device plan + device counters.

    ``View(layout)`` allocates zero-filled blobs (Blob, blob.hpp:22-29).
    ``View(layout, blobs=[ptr, ...])`` adopts caller-owned device pointers (e.g.
    ``torch.Tensor.data_ptr()``), checking count/size like view.cpp:105-118.
    """

    def __init__(self, layout: Layout, device: int = 0, stream=None, blobs: Sequence[int] | None = None,
                 blob_bytes: Sequence[int] | None = None):
        L = lib()
        self.layout = layout
        self.device = device
        h = C.c_void_p()
        if blobs is None:
            _check(L.lam_view_alloc(layout.handle, device, _stream_handle(stream), C.byref(h)))
        else:
            n = len(blobs)
            if blob_bytes is None or len(blob_bytes) != n:
                raise InvalidArgument("blob size mismatch: pass blob_bytes (one size per adopted blob)")
            ptrs = (C.c_void_p * max(1, n))(*[C.c_void_p(int(p)) for p in blobs])
            sizes = (C.c_uint64 * max(1, n))(*blob_bytes)
            _check(L.lam_view_wrap(layout.handle, device, ptrs, sizes, n, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().lam_view_free(h)
            except TypeError:  # interpreter shutdown: module globals already torn down
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def device_plan(self) -> int:
        """Device pointer of the lowered plan, for user kernels on include/lamina_b200_device.cuh."""
        return lib().lam_view_device_plan(self._h) or 0

    def dump(self, stem: str) -> None:
        """lamina::writeViewDump (view_io.cpp:28-59): <stem>.meta + <stem>.blob<nr>.bin."""
        _check(lib().lam_view_dump(self._h, str(stem).encode()))

    def is_trivially_relocatable(self) -> bool:
        return bool(lib().lam_view_is_trivially_relocatable(self._h))

    def blob_bytes(self) -> int:
        return int(lib().lam_view_blob_bytes(self._h))

    def state_bytes(self) -> int:
        return int(lib().lam_view_state_bytes(self._h))

    def blob_ptr(self, nr: int) -> int:
        return lib().lam_view_blob(self._h, nr) or 0

    def upload(self, nr: int, host: np.ndarray, stream=None) -> None:
        host = np.ascontiguousarray(host)
        if host.nbytes != self.layout.blob_size(nr):
            raise InvalidArgument(f"blob size mismatch: blob {nr} declares {self.layout.blob_size(nr)}, "
                                  f"got {host.nbytes}")
        _check(lib().lam_view_upload(self._h, nr, host.ctypes.data_as(C.c_void_p), _stream_handle(stream)))
        if stream is None:
            self.sync()

    def download(self, nr: int, out: np.ndarray | None = None, stream=None) -> np.ndarray:
        if out is None:
            out = np.empty(self.layout.blob_size(nr), dtype=np.uint8)
        _check(lib().lam_view_download(self._h, nr, out.ctypes.data_as(C.c_void_p), _stream_handle(stream)))
        if stream is None:
            self.sync()
        return out

    def upload_range(self, nr: int, offset: int, host: np.ndarray, stream=None) -> None:
        host = np.ascontiguousarray(host)
        _check(lib().lam_view_upload_range(self._h, nr, offset, host.nbytes, host.ctypes.data_as(C.c_void_p),
                                           _stream_handle(stream)))
        if stream is None:
            self.sync()

    def download_range(self, nr: int, offset: int, nbytes: int, stream=None) -> np.ndarray:
        out = np.empty(nbytes, dtype=np.uint8)
        _check(lib().lam_view_download_range(self._h, nr, offset, nbytes, out.ctypes.data_as(C.c_void_p),
                                             _stream_handle(stream)))
        if stream is None:
            self.sync()
        return out

    def upload_all(self, blobs: Sequence[np.ndarray]) -> None:
        for nr, b in enumerate(blobs):
            if self.layout.blob_size(nr):
                self.upload(nr, b)

    def download_all(self) -> list[np.ndarray]:
        return [self.download(nr) for nr in range(self.layout.blob_count)]

    def sync(self) -> None:
        _check(lib().lam_device_sync(self.device))

    def read_values(self, linear: Iterable[int], leaf: Iterable[int], stream=None) -> np.ndarray:
        lin = np.ascontiguousarray(np.asarray(linear, dtype=np.uint64))
        lf = np.ascontiguousarray(np.asarray(leaf, dtype=np.uint32))
        out = np.empty(lin.size, dtype=np.uint64)
        _check(lib().lam_view_read_values(self._h, lin.ctypes.data_as(C.POINTER(C.c_uint64)),
                                          lf.ctypes.data_as(C.POINTER(C.c_uint32)),
                                          out.ctypes.data_as(C.POINTER(C.c_uint64)), lin.size,
                                          _stream_handle(stream)))
        return out

    def write_values(self, linear: Iterable[int], leaf: Iterable[int], bits: Iterable[int], stream=None) -> None:
        lin = np.ascontiguousarray(np.asarray(linear, dtype=np.uint64))
        lf = np.ascontiguousarray(np.asarray(leaf, dtype=np.uint32))
        b = np.ascontiguousarray(np.asarray(bits, dtype=np.uint64))
        _check(lib().lam_view_write_values(self._h, lin.ctypes.data_as(C.POINTER(C.c_uint64)),
                                           lf.ctypes.data_as(C.POINTER(C.c_uint32)),
                                           b.ctypes.data_as(C.POINTER(C.c_uint64)), lin.size,
                                           _stream_handle(stream)))

    def counters(self) -> tuple[np.ndarray, np.ndarray]:
        n = self.layout.leaf_count
        r = np.zeros(max(1, n), dtype=np.uint64)
        w = np.zeros(max(1, n), dtype=np.uint64)
        _check(lib().lam_counters_read(self._h, r.ctypes.data_as(C.POINTER(C.c_uint64)),
                                       w.ctypes.data_as(C.POINTER(C.c_uint64))))
        return r[:n], w[:n]

    def reset_counters(self, stream=None) -> None:
        _check(lib().lam_counters_reset(self._h, _stream_handle(stream)))

    def heatmap(self, nr: int) -> np.ndarray:
        out = np.zeros(max(1, self.layout.heatmap_blocks(nr)), dtype=np.uint64)
        _check(lib().lam_heatmap_read(self._h, nr, out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return out[: self.layout.heatmap_blocks(nr)]

    # ---- n-body (tools/nbody) ---------------------------------------------------------------
    def nbody_init(self, seed: int = 42, stream=None) -> None:
        _check(lib().lam_nbody_init(self._h, seed, _stream_handle(stream)))

    def nbody_update(self, mode: int = NBODY_EXACT, begin: int = 0, end: int | None = None, stream=None) -> None:
        end = self.layout.element_count if end is None else end
        _check(lib().lam_nbody_update(self._h, mode, begin, end, _stream_handle(stream)))

    def nbody_move(self, begin: int = 0, end: int | None = None, stream=None) -> None:
        end = self.layout.element_count if end is None else end
        _check(lib().lam_nbody_move(self._h, begin, end, _stream_handle(stream)))

    def nbody_step(self, mode: int = NBODY_EXACT, begin: int = 0, end: int | None = None, stream=None) -> None:
        end = self.layout.element_count if end is None else end
        _check(lib().lam_nbody_step(self._h, mode, begin, end, _stream_handle(stream)))

    def nbody_update_from(self, sources, mode: int = NBODY_EXACT, begin: int = 0, end: int | None = None,
                          stream=None) -> None:
        """Fused update: j-particles read from other views, sources = [(view, j_begin, j_end), ...]."""
        end = self.layout.element_count if end is None else end
        k = len(sources)
        hv = (C.c_void_p * k)(*[v.handle for v, _, _ in sources])
        jb = (C.c_uint64 * k)(*[int(b) for _, b, _ in sources])
        je = (C.c_uint64 * k)(*[int(e) for _, _, e in sources])
        _check(lib().lam_nbody_update_multi(self._h, hv, jb, je, k, mode, begin, end, _stream_handle(stream)))

    def nbody_pack_positions(self, begin: int, end: int, out_ptr: int, with_mass: bool = False, stream=None) -> None:
        """SoA x, y, z (, m) of particles [begin, end) into the device buffer at out_ptr."""
        _check(lib().lam_nbody_pack_positions(self._h, begin, end, 1 if with_mass else 0, C.c_void_p(out_ptr),
                                              _stream_handle(stream)))

    def nbody_checksum(self) -> float:
        out = C.c_double()
        _check(lib().lam_nbody_checksum(self._h, C.byref(out)))
        return out.value


class ManualNbody:
    """The reference's hand-written n-body baselines (steps.hpp:124-230) on the device:
    kind "manual-aos" (ManualParticle[]) or "manual-soa" (ManualSoA), no mapping involved."""

    def __init__(self, kind: str, n: int, f64: bool = False, seed: int = 42, device: int = 0, stream=None):
        h = C.c_void_p()
        _check(lib().lam_nbody_manual_create(kind.encode(), n, 1 if f64 else 0, seed, device, _stream_handle(stream),
                                             C.byref(h)))
        self._h, self.kind, self.n = h, kind, n

    def update(self, mode: int = NBODY_EXACT, stream=None) -> None:
        _check(lib().lam_nbody_manual_update(self._h, mode, _stream_handle(stream)))

    def move(self, stream=None) -> None:
        _check(lib().lam_nbody_manual_move(self._h, _stream_handle(stream)))

    def checksum(self) -> float:
        out = C.c_double()
        _check(lib().lam_nbody_manual_checksum(self._h, C.byref(out)))
        return out.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().lam_nbody_manual_free(h)
            except TypeError:
                pass
            self._h = None


def write_view_dump(view: View, stem: str) -> None:
    """lamina::writeViewDump (core/src/view_io.cpp:28-59)."""
    view.dump(stem)


def read_view_dump(stem: str, device: int = 0, stream=None) -> View:
    """lamina::readViewDump (core/src/view_io.cpp:61-129): a new device view from a dump."""
    lh, vh = C.c_void_p(), C.c_void_p()
    _check(lib().lam_view_restore(str(stem).encode(), device, _stream_handle(stream), C.byref(lh), C.byref(vh)))
    v = View.__new__(View)
    v.layout = Layout._adopt(lh)
    v.device = device
    v._h = vh
    return v


def copy_sharded(pairs) -> None:
    """lam_copy_sharded: copyView for every (src, dst) pair, each on its own device, all in flight."""
    k = len(pairs)
    s = (C.c_void_p * max(1, k))(*[a.handle for a, _ in pairs])
    d = (C.c_void_p * max(1, k))(*[b.handle for _, b in pairs])
    _check(lib().lam_copy_sharded(s, d, k))


def ipc_handle(device_ptr: int) -> bytes:
    """cudaIpcGetMemHandle of a device allocation (64 bytes)."""
    buf = C.create_string_buffer(64)
    _check(lib().lam_ipc_get_handle(C.c_void_p(device_ptr), buf))
    return buf.raw


def ipc_open(handle: bytes, device: int) -> int:
    """Map a peer allocation into this process (cudaIpcOpenMemHandle, lazy peer access)."""
    p = C.c_void_p()
    _check(lib().lam_ipc_open(C.create_string_buffer(handle, 64), device, C.byref(p)))
    return p.value or 0


def ipc_close(device_ptr: int) -> None:
    _check(lib().lam_ipc_close(C.c_void_p(device_ptr)))


def copy_view(src: View, dst: View, stream=None) -> None:
    """lamina::copyView (view.cpp:168-189) on device views; stream-ordered."""
    _check(lib().lam_copy(src.handle, dst.handle, _stream_handle(stream)))


def copy_view_range(src: View, dst: View, begin: int, end: int, stream=None) -> None:
    """copyView restricted to elements [begin, end) (one shard of a multi-GPU copy)."""
    _check(lib().lam_copy_range(src.handle, dst.handle, begin, end, _stream_handle(stream)))


def copy_view_host(src: Layout, src_blobs: Sequence[np.ndarray], dst: Layout, dst_blobs: Sequence[np.ndarray],
                   device: int = 0):
    """copyView over HOST blobs through the GPU (H2D, copy, D2H inside).

    dst_blobs are updated in place.  Returns (src_counters, dst_counters): [reads..., writes...]
    for a FieldAccessCount view, followed by the heatmap blocks of a Heatmap view, else None.
    """
    def ptrs(bl):
        arr = (C.c_void_p * max(1, len(bl)))()
        for k, b in enumerate(bl):
            if not isinstance(b, np.ndarray):
                raise TypeError("host blobs must be numpy arrays")
            if not b.flags.c_contiguous:
                raise InvalidArgument("host blobs must be contiguous")
            arr[k] = b.ctypes.data
        return arr

    def counters(lay: Layout):
        # [reads, writes] when FieldAccessCount wraps the mapping, then the heatmap blocks
        n = 2 * lay.leaf_count if "field-access-count(" in lay.name else 0
        n += sum(lay.heatmap_blocks(k) for k in range(lay.blob_count))
        return np.zeros(max(1, n), dtype=np.uint64), n

    if len(src_blobs) != src.blob_count or len(dst_blobs) != dst.blob_count:
        raise InvalidArgument("blob count mismatch")
    for lay, bl in ((src, src_blobs), (dst, dst_blobs)):
        for k, b in enumerate(bl):
            if b.nbytes != lay.blob_size(k):
                raise InvalidArgument(f"blob size mismatch: blob {k} declares {lay.blob_size(k)}, got {b.nbytes}")
    sc, sn = counters(src)
    dc, dn = counters(dst)
    _check(lib().lam_copy_host(src.handle, ptrs(src_blobs), dst.handle, ptrs(dst_blobs), device,
                               sc.ctypes.data_as(C.POINTER(C.c_uint64)), dc.ctypes.data_as(C.POINTER(C.c_uint64))))
    return (sc[:sn] if sn else None), (dc[:dn] if dn else None)


def launch_count() -> int:
    return lib().lam_launch_count()


def fp32_peak_tflops(device: int = 0, seconds: float = 1.0) -> float:
    """Measured sustained FP32 FFMA throughput (the n-body roofline denominator)."""
    out = C.c_double()
    _check(lib().lam_bench_fma_peak(device, seconds, C.byref(out)))
    return out.value


# ---- reports (instrument.cpp:235-257) ------------------------------------------------------------
def field_access_csv(layout: Layout, reads, writes) -> str:
    rows = ["field,reads,writes,total"]
    for f in range(layout.leaf_count):
        r, w = int(reads[f]), int(writes[f])
        rows.append(f"{layout.leaf_path(f)},{r},{w},{r + w}")
    tr, tw = int(sum(int(x) for x in reads)), int(sum(int(x) for x in writes))
    rows.append(f"TOTAL,{tr},{tw},{tr + tw}")
    return "\n".join(rows) + "\n"


def heatmap_csv(granularity: int, blocks_per_blob: Sequence[np.ndarray]) -> str:
    rows = []
    for nr, blocks in enumerate(blocks_per_blob):
        rows.append(f"# blob {nr}")
        rows.append("blockIndex,byteStart,count")
        for b, c in enumerate(blocks):
            rows.append(f"{b},{b * granularity},{int(c)}")
    return "\n".join(rows) + ("\n" if rows else "")
