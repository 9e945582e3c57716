"""Loader for the in-tree C ABI library (include/lamina_b200.h).

The product path has exactly one implementation: the sm_100a kernels in
``_lib/liblamina_b200.so``.  There is no CPU fallback; a missing library raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "liblamina_b200.so")

_lib = None

u64 = C.c_uint64
sz = C.c_size_t
vp = C.c_void_p
cp = C.c_char_p
i32 = C.c_int

_SIGS = {
    "lam_last_error": (cp, []),
    "lam_version": (cp, []),
    "lam_layout_create": (i32, [cp, cp, C.POINTER(u64), sz, cp, i32, u64, C.POINTER(vp)]),
    "lam_layout_destroy": (None, [vp]),
    "lam_layout_name": (sz, [vp, cp, sz]),
    "lam_layout_schema": (sz, [vp, cp, sz]),
    "lam_layout_extents": (sz, [vp, cp, sz]),
    "lam_layout_blob_count": (sz, [vp]),
    "lam_layout_blob_size": (u64, [vp, sz]),
    "lam_layout_element_count": (u64, [vp]),
    "lam_layout_leaf_count": (sz, [vp]),
    "lam_layout_leaf": (i32, [vp, sz, C.POINTER(i32), C.POINTER(sz), C.POINTER(sz)]),
    "lam_layout_leaf_path": (sz, [vp, sz, cp, sz]),
    "lam_layout_is_computed": (i32, [vp, sz]),
    "lam_layout_is_fully_physical": (i32, [vp]),
    "lam_layout_has_mutable_state": (i32, [vp]),
    "lam_layout_physical_offset": (i32, [vp, u64, sz, C.POINTER(sz), C.POINTER(u64)]),
    "lam_layout_heatmap_blocks": (u64, [vp, sz]),
    "lam_layout_shard_unit": (u64, [vp]),
    "lam_layout_stream_count": (sz, [vp]),
    "lam_layout_stream_region": (i32, [vp, sz, u64, u64, C.POINTER(sz), C.POINTER(u64), C.POINTER(u64)]),
    "lam_view_alloc": (i32, [vp, i32, vp, C.POINTER(vp)]),
    "lam_view_wrap": (i32, [vp, i32, C.POINTER(vp), C.POINTER(u64), sz, C.POINTER(vp)]),
    "lam_view_free": (None, [vp]),
    "lam_view_layout": (vp, [vp]),
    "lam_view_blob": (vp, [vp, sz]),
    "lam_view_upload": (i32, [vp, sz, vp, vp]),
    "lam_view_download": (i32, [vp, sz, vp, vp]),
    "lam_layout_is_fully_static": (i32, [vp]),
    "lam_layout_runtime_state_bytes": (u64, [vp]),
    "lam_view_is_trivially_relocatable": (i32, [vp]),
    "lam_view_blob_bytes": (u64, [vp]),
    "lam_view_state_bytes": (u64, [vp]),
    "lam_view_upload_range": (i32, [vp, sz, u64, u64, vp, vp]),
    "lam_view_download_range": (i32, [vp, sz, u64, u64, vp, vp]),
    "lam_view_device_plan": (vp, [vp]),
    "lam_copy_sharded": (i32, [C.POINTER(vp), C.POINTER(vp), sz]),
    "lam_nbody_step": (i32, [vp, i32, u64, u64, vp]),
    "lam_nbody_update_multi": (i32, [vp, C.POINTER(vp), C.POINTER(u64), C.POINTER(u64), sz, i32, u64, u64, vp]),
    "lam_ipc_get_handle": (i32, [vp, vp]),
    "lam_ipc_open": (i32, [vp, i32, C.POINTER(vp)]),
    "lam_ipc_close": (i32, [vp]),
    "lam_layout_contiguous_run": (i32, [vp, u64, sz, u64, C.POINTER(C.c_int), C.POINTER(sz), C.POINTER(u64)]),
    "lam_layout_dump_meta": (sz, [vp, cp, sz]),
    "lam_view_dump": (i32, [vp, cp]),
    "lam_view_restore": (i32, [cp, i32, vp, C.POINTER(vp), C.POINTER(vp)]),
    "lam_copy": (i32, [vp, vp, vp]),
    "lam_copy_range": (i32, [vp, vp, u64, u64, vp]),
    "lam_copy_host": (i32, [vp, C.POINTER(vp), vp, C.POINTER(vp), i32, C.POINTER(u64), C.POINTER(u64)]),
    "lam_counters_read": (i32, [vp, C.POINTER(u64), C.POINTER(u64)]),
    "lam_counters_reset": (i32, [vp, vp]),
    "lam_heatmap_read": (i32, [vp, sz, C.POINTER(u64)]),
    "lam_view_read_values": (i32, [vp, C.POINTER(u64), C.POINTER(C.c_uint32), C.POINTER(u64), sz, vp]),
    "lam_view_write_values": (i32, [vp, C.POINTER(u64), C.POINTER(C.c_uint32), C.POINTER(u64), sz, vp]),
    "lam_nbody_init": (i32, [vp, u64, vp]),
    "lam_nbody_update": (i32, [vp, i32, u64, u64, vp]),
    "lam_nbody_move": (i32, [vp, u64, u64, vp]),
    "lam_nbody_checksum": (i32, [vp, C.POINTER(C.c_double)]),
    "lam_nbody_pack_positions": (i32, [vp, u64, u64, i32, vp, vp]),
    "lam_nbody_manual_create": (i32, [cp, u64, i32, u64, i32, vp, C.POINTER(vp)]),
    "lam_nbody_manual_update": (i32, [vp, i32, vp]),
    "lam_nbody_manual_move": (i32, [vp, vp]),
    "lam_nbody_manual_checksum": (i32, [vp, C.POINTER(C.c_double)]),
    "lam_nbody_manual_free": (None, [vp]),
    "lam_launch_count": (u64, []),
    "lam_bench_fma_peak": (i32, [i32, C.c_double, C.POINTER(C.c_double)]),
    "lam_device_sync": (i32, [i32]),
}

EXPORTED = tuple(_SIGS)


def lib():
    """The loaded C ABI library; raises ImportError if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"lamina_b200 native library missing at {LIB_PATH}; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
