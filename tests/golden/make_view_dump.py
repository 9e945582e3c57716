"""Generates tests/golden/view_dump/*: views written by the reference's writeViewDump
(core/src/view_io.cpp:28-59) through oracle/_ref/ref_tool, filled like
test_view_io.cpp:37-48.  Run in the build container:  python tests/golden/make_view_dump.py
"""
import json
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "view_dump")
S_IO = "Record{Pos: Record{x: f64, y: f64}, Flags: u8, Count: i32}"
R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"

# (name, schema, extents, dyn, layout, salt)
CASES = [
    ("io_aos", S_IO, "i32:[6]", [], "aos-packed", 50),
    ("io_soamb", S_IO, "i32:[6]", [], "soa-mb", 50),
    ("io_aosoa4", S_IO, "i32:[6]", [], "aosoa:4", 50),
    ("io_bytesplit", S_IO, "i32:[6]", [], "bytesplit:soa-sb", 50),
    ("io_split", S_IO, "i32:[6]", [], "split:Pos:soa-mb:aos-packed", 50),
    ("io_dyn", "Record{x: f64, n: u16}", "u32:[2,dyn,3]", [5], "soa-sb", 7),
    ("r32_aosoa8", R32, "i64:[37]", [], "aosoa:8", 3),
    ("bits_int5", "Record{v:u32,w:i32}", "i32:[41]", [], "bitpack-int:5", 11),
    ("bits_e5m10", "Record{v:f32}", "i16:[29]", [], "bitpack-float:5,10", 13),
    ("changetype", "Record{a:f64,b:i64}", "i32:[9]", [], "changetype:f64=f32,i64=i16:aos-aligned", 17),
]


def main():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    index = []
    for name, schema, ext, dyn, layout, salt in CASES:
        stem = os.path.join(OUT, name)
        subprocess.run([exe, "dump", schema, ext, ",".join(map(str, dyn)) if dyn else "-", layout, str(salt), stem],
                       check=True)
        index.append({"name": name, "schema": schema, "extents": ext, "dyn": dyn, "layout": layout, "salt": salt})
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump(index, f, indent=1)
    print(f"wrote {len(index)} view dumps")


if __name__ == "__main__":
    sys.exit(main())
