"""The C++ mirror on a GPU: readViewDump of a reference-written dump, copyView on the device,
writeViewDump, and the result read back by the oracle."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from oracle import lamina_oracle as O

pytestmark = pytest.mark.gpu

SRC = r"""
#include "lamina_b200.hpp"
#include <cstdio>
int main(int argc, char** argv)
{
    auto v = lamina_b200::readViewDump(argv[1]);
    const std::string S = "Record{Pos: Record{x: f64, y: f64}, Flags: u8, Count: i32}";
    lamina_b200::View out(lamina_b200::parseLayout("aosoa:4", S, "i32:[6]"));
    lamina_b200::copyView(v, out);
    lamina_b200::writeViewDump(out, argv[2]);
    std::printf("%s\n", v.mapping().name().c_str());
    return 0;
}
"""


def test_cpp_mirror_dump_roundtrip_on_device(tmp_path):
    lib = os.path.join(ROOT, "paper_2302_08251_b200", "_lib")
    src = tmp_path / "t.cpp"
    src.write_text(SRC)
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", str(src), f"-L{lib}", "-llamina_b200",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    stem_in = os.path.join(ROOT, "tests", "golden", "view_dump", "io_split")
    stem_out = str(tmp_path / "out")
    r = subprocess.run([str(exe), stem_in, stem_out], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip() == "split:Pos:soa-mb:aos-packed"
    S = "Record{Pos: Record{x: f64, y: f64}, Flags: u8, Count: i32}"
    src_m = O.make(S, "i32:[6]", "split:Pos:soa-mb:aos-packed")
    src_b = [np.fromfile(f"{stem_in}.blob{k}.bin", np.uint8) for k in range(3)]
    out_m = O.make(S, "i32:[6]", "aosoa:4")
    out_b = [np.fromfile(f"{stem_out}.blob0.bin", np.uint8)]
    assert np.array_equal(O.read_all(out_m, out_b), O.read_all(src_m, src_b))
