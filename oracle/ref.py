"""TEST INFRASTRUCTURE ONLY: ctypes access to the reference itself.

``oracle/_ref/libref.so`` is the unmodified reference library (lamina) compiled by
``oracle/Makefile`` from /root/reference/proj, plus ``oracle/ref_shim.cpp``.  Used
by tests (as the checker), by tests/golden/make_golden.py and by bench.py's
``cpu_baseline`` / ``--impl reference`` arms.  Never imported by the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libref.so")
REF_SRC = "/root/reference/proj"

_lib = None


def build(force: bool = False) -> bool:
    """Compile the reference (only where /root/reference exists)."""
    if os.path.exists(REF_SO) and not force:
        return True
    if not os.path.isdir(REF_SRC):
        return False
    subprocess.run(["make", "-j8", "-C", HERE, f"REF={REF_SRC}"], check=True, stdout=subprocess.DEVNULL)
    return os.path.exists(REF_SO)


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(REF_SO):
            raise ImportError(f"reference oracle not built at {REF_SO}")
        L = C.CDLL(REF_SO)
        u64, sz, vp, cp, i32, dbl = C.c_uint64, C.c_size_t, C.c_void_p, C.c_char_p, C.c_int, C.c_double
        P = C.POINTER
        L.ref_last_error.restype = cp
        L.ref_last_kind.restype = i32
        L.ref_layout_info.argtypes = [cp, cp, P(u64), sz, cp, i32, u64, cp, sz, P(u64), sz, P(sz), P(sz), P(sz)]
        L.ref_copy.argtypes = [cp, cp, P(u64), sz, cp, i32, u64, cp, i32, u64, P(vp), P(vp), i32, i32, P(u64), P(u64),
                               P(u64), P(u64), P(dbl)]
        L.ref_write_values.argtypes = [cp, cp, P(u64), sz, cp, P(u64), P(vp)]
        L.ref_read_values.argtypes = [cp, cp, P(u64), sz, cp, P(vp), P(u64)]
        L.ref_scalar_sample.restype = u64
        L.ref_scalar_sample.argtypes = [i32, u64]
        L.ref_float_encode.restype = u64
        L.ref_float_encode.argtypes = [dbl, C.c_uint, C.c_uint]
        L.ref_float_decode.restype = dbl
        L.ref_float_decode.argtypes = [u64, C.c_uint, C.c_uint]
        L.ref_float_encode_f32_array.argtypes = [P(C.c_uint32), P(u64), sz, C.c_uint, C.c_uint]
        L.ref_f64_to_f32_array.argtypes = [P(u64), P(C.c_uint32), sz]
        L.ref_f32_to_f64_array.argtypes = [P(C.c_uint32), P(u64), sz]
        L.ref_nbody.argtypes = [cp, u64, u64, i32, u64, i32, i32, P(vp), P(dbl), P(dbl), P(dbl)]
        L.ref_nbody_cli.argtypes = [cp, u64, u64, i32, u64, i32]
        L.ref_nbody_trace.argtypes = [cp, u64, u64, i32, u64, i32, u64, cp, cp]
        L.ref_view_new.restype = vp
        L.ref_view_new.argtypes = [cp, cp, P(u64), sz, cp, i32, u64]
        L.ref_view_free.argtypes = [vp]
        L.ref_view_blob_count.restype = sz
        L.ref_view_blob_count.argtypes = [vp]
        L.ref_view_blob.restype = vp
        L.ref_view_blob.argtypes = [vp, sz, P(u64)]
        L.ref_view_copy.argtypes = [vp, vp, i32, P(dbl), P(u64)]
        L.ref_state_info.argtypes = [cp, cp, P(u64), sz, cp, i32, u64, P(i32), P(u64), P(i32), P(u64), P(u64)]
        L.ref_contiguous_run.argtypes = [cp, cp, P(u64), C.c_size_t, cp, i32, u64, u64, C.c_size_t, u64, P(C.c_int),
                                         P(C.c_size_t), P(u64)]
        _lib = L
    return _lib


class RefError(Exception):
    def __init__(self, kind: int, msg: str):
        super().__init__(msg)
        self.kind = kind  # 1 invalid_argument 2 out_of_range 3 overflow_error 4 logic_error 5 other


def _check(rc):
    if rc != 0:
        L = lib()
        raise RefError(L.ref_last_kind(), L.ref_last_error().decode())


def _dyn(dyn):
    return (C.c_uint64 * max(1, len(dyn)))(*dyn), len(dyn)


def _ptrs(blobs):
    arr = (C.c_void_p * max(1, len(blobs)))()
    for k, b in enumerate(blobs):
        arr[k] = b.ctypes.data if b.nbytes else None
    return arr


def layout_info(schema, extents, layout, dyn=(), wrap=0, gran=0):
    L = lib()
    name = C.create_string_buffer(4096)
    sizes = (C.c_uint64 * 4096)()
    nb, nl, hb = C.c_size_t(), C.c_size_t(), C.c_size_t()
    d, nd = _dyn(dyn)
    _check(L.ref_layout_info(schema.encode(), extents.encode(), d, nd, layout.encode(), wrap, gran, name, 4096,
                             sizes, 4096, C.byref(nb), C.byref(nl), C.byref(hb)))
    return {"name": name.value.decode(), "blob_sizes": [sizes[k] for k in range(nb.value)], "leaves": nl.value,
            "heat_blocks": hb.value}


def copy(schema, extents, src_layout, src_blobs, dst_layout, dst_blobs, dyn=(), src_wrap=0, src_gran=0, dst_wrap=0,
         dst_gran=0, nthreads=1, repeats=1):
    """Reference copyView; dst_blobs updated in place. Returns dict with counters and seconds."""
    L = lib()
    info_s = layout_info(schema, extents, src_layout, dyn, src_wrap, src_gran)
    info_d = layout_info(schema, extents, dst_layout, dyn, dst_wrap, dst_gran)
    nl = info_s["leaves"]
    sf = np.zeros(max(1, 2 * nl), np.uint64)
    df = np.zeros(max(1, 2 * nl), np.uint64)
    sh = np.zeros(max(1, info_s["heat_blocks"]), np.uint64)
    dh = np.zeros(max(1, info_d["heat_blocks"]), np.uint64)
    secs = C.c_double()
    d, nd = _dyn(dyn)
    P = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint64))  # noqa: E731
    _check(L.ref_copy(schema.encode(), extents.encode(), d, nd, src_layout.encode(), src_wrap, src_gran,
                      dst_layout.encode(), dst_wrap, dst_gran, _ptrs(src_blobs), _ptrs(dst_blobs), nthreads, repeats,
                      P(sf), P(df), P(sh), P(dh), C.byref(secs)))
    return {"src_fac": sf[: 2 * nl], "dst_fac": df[: 2 * nl], "src_heat": sh[: info_s["heat_blocks"]],
            "dst_heat": dh[: info_d["heat_blocks"]], "seconds": secs.value}


def zero_blobs(schema, extents, layout, dyn=()):
    return [np.zeros(s, np.uint8) for s in layout_info(schema, extents, layout, dyn)["blob_sizes"]]


def write_values(schema, extents, layout, values, dyn=()):
    """Blobs of a fresh view after View::write of every (i, f) (values: [N, leaves] u64 storage bits)."""
    blobs = zero_blobs(schema, extents, layout, dyn)
    v = np.ascontiguousarray(values, dtype=np.uint64)
    d, nd = _dyn(dyn)
    _check(lib().ref_write_values(schema.encode(), extents.encode(), d, nd, layout.encode(),
                                  v.ctypes.data_as(C.POINTER(C.c_uint64)), _ptrs(blobs)))
    return blobs


def read_values(schema, extents, layout, blobs, n, leaves, dyn=()):
    out = np.zeros((max(1, n), max(1, leaves)), np.uint64)
    d, nd = _dyn(dyn)
    _check(lib().ref_read_values(schema.encode(), extents.encode(), d, nd, layout.encode(), _ptrs(blobs),
                                 out.ctypes.data_as(C.POINTER(C.c_uint64))))
    return out[:n, :leaves]


def scalar_sample(kind, salt):
    return lib().ref_scalar_sample(kind, salt)


def float_encode(v, e, m):
    return lib().ref_float_encode(v, e, m)


def float_decode(p, e, m):
    return lib().ref_float_decode(p, e, m)


def float_encode_f32(bits32: np.ndarray, e, m):
    b = np.ascontiguousarray(bits32, dtype=np.uint32)
    out = np.empty(b.size, np.uint64)
    lib().ref_float_encode_f32_array(b.ctypes.data_as(C.POINTER(C.c_uint32)), out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                     b.size, e, m)
    return out


def f64_to_f32(bits64: np.ndarray):
    b = np.ascontiguousarray(bits64, dtype=np.uint64)
    out = np.empty(b.size, np.uint32)
    lib().ref_f64_to_f32_array(b.ctypes.data_as(C.POINTER(C.c_uint64)), out.ctypes.data_as(C.POINTER(C.c_uint32)), b.size)
    return out


def f32_to_f64(bits32: np.ndarray):
    b = np.ascontiguousarray(bits32, dtype=np.uint32)
    out = np.empty(b.size, np.uint64)
    lib().ref_f32_to_f64_array(b.ctypes.data_as(C.POINTER(C.c_uint32)), out.ctypes.data_as(C.POINTER(C.c_uint64)), b.size)
    return out


def nbody(layout, n, steps, f64=False, seed=42, width=1, nthreads=1, with_blobs=True):
    """Reference n-body run; returns (checksum, blobs, update_s, move_s)."""
    L = lib()
    prec = "f64" if f64 else "f32"
    t = prec
    schema = f"Record{{Pos:Record{{x:{t},y:{t},z:{t}}},Vel:Record{{x:{t},y:{t},z:{t}}},Mass:{t}}}"
    blobs = zero_blobs(schema, f"i64:[{n}]", layout) if with_blobs else []
    cs, us, ms = C.c_double(), C.c_double(), C.c_double()
    _check(L.ref_nbody(layout.encode(), n, steps, 1 if f64 else 0, seed, width, nthreads,
                       _ptrs(blobs) if with_blobs else None, C.byref(cs), C.byref(us), C.byref(ms)))
    return cs.value, blobs, us.value, ms.value


def nbody_trace(layout, n, steps, report_dir, trace=True, heat_gran=0, f64=False, seed=42, csv_path=None):
    """The reference runner with field tracing / heatmap: report CSVs land in report_dir."""
    import os
    os.makedirs(report_dir, exist_ok=True)
    rc = lib().ref_nbody_trace(layout.encode(), n, steps, 1 if f64 else 0, seed, 1 if trace else 0, heat_gran,
                               str(report_dir).encode(), csv_path.encode() if csv_path else None)
    if rc != 0:
        raise RefError(5, f"ref_nbody_trace exit code {rc}")


def state_info(schema, extents, layout, dyn=(), wrap=0, gran=1):
    """(isFullyStatic, runtimeStateBytes, isTriviallyRelocatable, stateBytes, blobBytes)."""
    d, nd = _dyn(dyn)
    fs, rs, tr, sb, bb = C.c_int(), C.c_uint64(), C.c_int(), C.c_uint64(), C.c_uint64()
    _check(lib().ref_state_info(schema.encode(), extents.encode(), d, nd, layout.encode(), wrap, gran, C.byref(fs),
                                C.byref(rs), C.byref(tr), C.byref(sb), C.byref(bb)))
    return bool(fs.value), rs.value, bool(tr.value), sb.value, bb.value


def contiguous_run(schema, extents, layout, linear, leaf, n, dyn=(), wrap=0, gran=1):
    """Mapping::contiguousRun of the reference: (nr, offset) or None."""
    d, nd = _dyn(dyn)
    has, nr, off = C.c_int(), C.c_size_t(), C.c_uint64()
    _check(lib().ref_contiguous_run(schema.encode(), extents.encode(), d, nd, layout.encode(), wrap, gran, linear, leaf,
                                    n, C.byref(has), C.byref(nr), C.byref(off)))
    return (nr.value, off.value) if has.value else None


class RefView:
    """A resident lamina::View (zeroed Blobs owned by the reference) whose blobs are exposed
    as writable numpy arrays; copy_from runs the reference copyView into it."""

    def __init__(self, schema, extents, layout, dyn=(), wrap=0, gran=0):
        d, nd = _dyn(dyn)
        self._h = lib().ref_view_new(schema.encode(), extents.encode(), d, nd, layout.encode(), wrap, gran)
        if not self._h:
            _check(lib().ref_last_kind() or 5)
        self.leaves = layout_info(schema, extents, layout, dyn, wrap, gran)["leaves"]
        self.blobs = []
        for nr in range(lib().ref_view_blob_count(self._h)):
            size = C.c_uint64()
            ptr = lib().ref_view_blob(self._h, nr, C.byref(size))
            if size.value == 0:
                self.blobs.append(np.zeros(0, np.uint8))
            else:
                self.blobs.append(np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(size.value,)))

    def copy_from(self, src: "RefView", nthreads=1):
        """copyView(src, self); returns (seconds, dst FieldAccessCount [reads..., writes...])."""
        secs = C.c_double()
        fac = np.zeros(max(1, 2 * self.leaves), np.uint64)
        _check(lib().ref_view_copy(src._h, self._h, nthreads, C.byref(secs),
                                   fac.ctypes.data_as(C.POINTER(C.c_uint64))))
        return secs.value, fac[: 2 * self.leaves]

    def __del__(self):
        if getattr(self, "_h", None):
            self.blobs = []
            lib().ref_view_free(self._h)
            self._h = None
