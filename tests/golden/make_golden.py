"""Generates tests/golden/*.npz from the reference itself (oracle/_ref, compiled from
/root/reference/proj).  Run in the build container:  python tests/golden/make_golden.py

The fixtures let the oracle and the GPU path be checked against reference outputs on
machines where /root/reference is absent.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import MIXED, R32, R64, random_values  # noqa: E402
from oracle import ref  # noqa: E402
from oracle.lamina_oracle import Schema  # noqa: E402

COPY_CASES = [
    (R32, 37, "aos-packed", "soa-mb", 0),
    (R32, 37, "aos-packed", "aosoa:8", 0),
    (R32, 37, "soa-sb", "aosoa:32", 0),
    (R32, 37, "aosoa:8", "aos-packed", 0),
    (R32, 37, "aos-packed", "bytesplit:soa-mb", 1),
    (R32, 37, "soa-mb", "bitpack-float:8,10", 0),
    (R32, 37, "soa-mb", "bitpack-float:5,10", 2),
    (R32, 37, "aos-packed", "split:Pos:soa-mb:aos-packed", 0),
    (R64, 29, "aos-packed", "changetype:f64=f32:bytesplit:soa-mb", 1),
    (MIXED, 23, "aos-packed", "aos-aligned", 0),
    (MIXED, 23, "soa-mb", "changetype:f64=f32,i8=i64,u16=u8:aosoa:2", 0),
    (MIXED, 23, "aosoa:4", "bytesplit:soa-sb", 2),
    ("Record{v:u32,w:i32}", 100, "soa-mb", "bitpack-int:3", 0),
    ("Record{v:u32,w:i32}", 100, "soa-mb", "bitpack-int:31", 1),
    ("Record{v:u32,w:i32}", 100, "aos-packed", "bitpack-int:12", 2),
]


def main():
    ref.build()
    rng = np.random.default_rng(20261018)
    index = []
    for k, (schema, n, a, b, wrap) in enumerate(COPY_CASES):
        types = [l.type for l in Schema.parse(schema).leaves]
        vals = random_values(rng, types, n)
        ext = f"i32:[{n}]"
        sb = ref.write_values(schema, ext, a, vals)
        db = ref.zero_blobs(schema, ext, b)
        r = ref.copy(schema, ext, a, sb, b, db, dst_wrap=wrap, dst_gran=3)
        arrays = {"values": vals}
        for nr, x in enumerate(sb):
            arrays[f"src{nr}"] = x
        for nr, x in enumerate(db):
            arrays[f"dst{nr}"] = x
        arrays["dst_fac"] = r["dst_fac"]
        arrays["dst_heat"] = r["dst_heat"]
        name = f"copy_{k:02d}.npz"
        np.savez_compressed(os.path.join(HERE, name), **arrays)
        index.append({"file": name, "schema": schema, "n": n, "src": a, "dst": b, "dst_wrap": wrap, "gran": 3,
                      "src_blobs": len(sb), "dst_blobs": len(db),
                      "dst_name": ref.layout_info(schema, ext, b, wrap=wrap, gran=3)["name"]})
    # floatEncode / floatDecode vectors (bitpack.cpp:96-188)
    fmts = [(5, 10), (8, 10), (8, 23), (11, 52), (4, 3), (2, 1), (6, 0), (11, 30), (15, 40)]
    d = np.concatenate([random_values(rng, [9], 4000)[:, 0], random_values(rng, [8], 4000)[:, 0]])
    f32 = random_values(rng, [8], 4000)[:, 0].astype(np.uint32)
    enc = {}
    for e, m in fmts:
        enc[f"enc_{e}_{m}"] = np.array([ref.float_encode(float(np.uint64(x).view(np.float64)), e, m) for x in d],
                                       dtype=np.uint64)
        pats = rng.integers(0, 2 ** min(63, 1 + e + m), 2000, dtype=np.uint64)
        enc[f"pat_{e}_{m}"] = pats
        enc[f"dec_{e}_{m}"] = np.array([np.float64(ref.float_decode(int(p), e, m)).view(np.uint64) for p in pats],
                                       dtype=np.uint64)
        enc[f"enc32_{e}_{m}"] = ref.float_encode_f32(f32, e, m)
    np.savez_compressed(os.path.join(HERE, "minifloat.npz"), doubles=d, f32=f32, **enc)
    index.append({"file": "minifloat.npz", "formats": fmts})
    # conversions (ScalarValue::convertTo)
    np.savez_compressed(os.path.join(HERE, "convert.npz"), f64=d, f64_to_f32=ref.f64_to_f32(d), f32=f32,
                        f32_to_f64=ref.f32_to_f64(f32))
    # n-body (tools/nbody): checksum and final state
    nb = []
    for layout, n, steps, f64 in [("aos-packed", 64, 2, False), ("soa-mb", 256, 5, False), ("aosoa:8", 128, 3, True),
                                  ("aos-packed", 1024, 5, False)]:
        cs, blobs, _, _ = ref.nbody(layout, n, steps, f64=f64, seed=42)
        name = f"nbody_{layout.replace(':', '')}_{n}_{steps}_{'f64' if f64 else 'f32'}.npz"
        np.savez_compressed(os.path.join(HERE, name), checksum=np.float64(cs), **{f"b{k}": b for k, b in enumerate(blobs)})
        nb.append({"file": name, "layout": layout, "n": n, "steps": steps, "f64": f64, "checksum": repr(cs)})
    index += nb
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump(index, f, indent=1)
    print(f"wrote {len(index)} fixtures")


if __name__ == "__main__":
    main()
