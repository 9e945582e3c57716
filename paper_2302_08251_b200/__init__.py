"""lamina_b200: B200-native (sm_100a) layout copy / bit packing / instrumentation / n-body
hot path of the LLAMA-paper reference library (arXiv 2302.08251), behind its C ABI."""
from .lamina import (  # noqa: F401
    BOOL, F32, F64, I8, I16, I32, I64, U8, U16, U32, U64, NBODY_EXACT, NBODY_FAST, SCALAR_NAMES, SCALAR_SIZE,
    WRAP_FIELD_ACCESS_COUNT, WRAP_HEATMAP, CudaError, IndexTypeOverflow, InvalidArgument, LaminaError, Layout,
    LogicError, OutOfRange, ReferenceRuntimeError, View, copy_view, copy_view_host, copy_view_range,
    field_access_csv, heatmap_csv, launch_count, parse_layout, read_view_dump, write_view_dump, copy_sharded,
    ipc_handle, ipc_open, ipc_close)
