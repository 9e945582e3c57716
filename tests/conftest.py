import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")


R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"
R64 = "Record{Pos:Record{x:f64,y:f64,z:f64},Vel:Record{x:f64,y:f64,z:f64},Mass:f64}"
MIXED = "Record{a:i8,b:u16,c:i32,d:u64,e:f32,f:f64,g:bool,h:Record{x:i16,y:f32[3]}}"

SPECIAL_F32 = np.array([0x7FC00000, 0xFFC00000, 0x7F800001, 0xFFA00001, 0x7F800000, 0xFF800000, 0x00000001,
                        0x80000001, 0x007FFFFF, 0x80000000, 0x00000000, 0x7F7FFFFF, 0x477FF000, 0x477FEFFF,
                        0x33800000, 0x33000000, 0x38800000, 0x387FFFFF], dtype=np.uint64)
SPECIAL_F64 = np.array([0x7FF8000000000000, 0xFFF8000000000000, 0x7FF0000000000001, 0xFFF4000000000123,
                        0x7FF0000000000000, 0xFFF0000000000000, 0x0000000000000001, 0x8000000000000001,
                        0x000FFFFFFFFFFFFF, 0x8000000000000000, 0x0000000000000000, 0x7FEFFFFFFFFFFFFF,
                        0x47EFFFFFE0000000, 0x47EFFFFFF0000000, 0x3690000000000000, 0x36A0000000000000,
                        0x3810000000000000, 0xC7EFFFFFE0000001, 0x3FB999999999999A], dtype=np.uint64)

SIZES = (1, 2, 4, 8, 1, 2, 4, 8, 4, 8, 1)


def random_values(rng: np.random.Generator, types, n, specials=True):
    """[n, leaves] u64 storage bits per leaf type; floats mix finite values, NaN payloads,
    sNaN, infinities, subnormals and signed zeros."""
    out = np.zeros((n, len(types)), np.uint64)
    for f, t in enumerate(types):
        if t == 10:  # bool
            col = rng.integers(0, 2, n, dtype=np.uint64)
        elif t == 8:
            col = rng.standard_normal(n).astype(np.float32) * np.float32(10.0) ** rng.integers(-6, 7, n).astype(np.float32)
            col = col.view(np.uint32).astype(np.uint64)
            raw = rng.integers(0, 2**32, n, dtype=np.uint64)
            col = np.where(rng.random(n) < 0.1, raw, col)
            if specials:
                k = min(n, len(SPECIAL_F32))
                col[:k] = SPECIAL_F32[:k]
        elif t == 9:
            col = (rng.standard_normal(n) * 10.0 ** rng.integers(-30, 31, n)).view(np.uint64)
            raw = rng.integers(0, 2**63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
            col = np.where(rng.random(n) < 0.1, raw, col)
            if specials:
                k = min(n, len(SPECIAL_F64))
                col[:k] = SPECIAL_F64[:k]
        else:
            bits = 8 * SIZES[t]
            col = rng.integers(0, 2**63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
            if bits < 64:
                col &= np.uint64((1 << bits) - 1)
        out[:, f] = col
    return out


def leaf_types(schema: str):
    from oracle.lamina_oracle import Schema
    return [l.type for l in Schema.parse(schema).leaves]


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as R
    if not R.available():
        R.build()
    if not R.available():
        pytest.skip("reference oracle (oracle/_ref) not built")
    return R
