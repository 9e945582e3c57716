"""The header-only C++ mirror (include/lamina_b200.hpp) compiles against the C ABI library
and maps errors onto the reference's exception types.  Host-only calls: runs on CPU."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = r"""
#include "lamina_b200.hpp"
#include <cstdio>
int main()
{
    const std::string R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}";
    auto m = lamina_b200::parseLayout("changetype:f32=f64:bytesplit:soa-mb", R32, "i32:[1000]");
    std::printf("%s %zu %llu\n", m->name().c_str(), m->blobCount(), (unsigned long long)m->blobSize(0));
    int caught = 0;
    try { lamina_b200::parseLayout("bogus", R32, "i32:[4]"); }
    catch(const std::invalid_argument& e) { caught += std::string(e.what()).find("unknown layout") != std::string::npos; }
    try { lamina_b200::parseLayout("aos-packed", R32, "i16:[40000]"); }
    catch(const std::overflow_error& e) { caught += 1; }
    std::printf("caught %d\n", caught);
    // Mapping::contiguousRun: SoA always, AoS never for n > 1, AoSoA inside a block
    auto soa = lamina_b200::parseLayout("soa-mb", R32, "i32:[100]");
    auto aos = lamina_b200::parseLayout("aos-packed", R32, "i32:[100]");
    auto aosoa = lamina_b200::parseLayout("aosoa:8", R32, "i32:[100]");
    const bool runs = soa->contiguousRun(5, 1, 50).has_value() && !aos->contiguousRun(5, 1, 2).has_value()
        && aosoa->contiguousRun(8, 2, 8).has_value() && !aosoa->contiguousRun(7, 2, 2).has_value();
    std::printf("runs %d\n", runs ? 1 : 0);
    std::printf("%s", soa->dumpMeta().c_str());
    return caught == 2 && runs ? 0 : 1;
}
"""


def test_cpp_mirror_compiles_and_maps_errors(tmp_path):
    lib = os.path.join(ROOT, "paper_2302_08251_b200", "_lib")
    if not os.path.exists(os.path.join(lib, "liblamina_b200.so")):
        pytest.skip("library not built")
    src = tmp_path / "t.cpp"
    src.write_text(SRC)
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", str(src), f"-L{lib}", "-llamina_b200",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    # f32 -> f64 storage, split into 8 one-byte planes per leaf: 7 x 8 = 56 blobs of n bytes
    assert out.stdout.splitlines()[0] == "changetype:f32=f64:bytesplit:soa-mb 56 1000"
    assert "runs 1" in out.stdout
    assert "mapping=soa-mb\nblobs=7\nblob0-size=400\n" in out.stdout


SRC2 = r"""
#include "lamina_b200.hpp"
#include <cstdio>
int main()
{
    // the reference's signature: parseLayout(text, const RecordSchema&, const ArrayExtents&)
    const auto schema = lamina_b200::RecordSchema::parse("Record{ a : f32 , b : Record{c:u8} }");
    const auto ext = lamina_b200::ArrayExtents::parse("i64:[dyn,3]", {5});
    auto m = lamina_b200::parseLayout("soa-sb", schema, ext);
    std::printf("%s|%s|%llu|%d|%s\n", schema.toString().c_str(), ext.toString().c_str(),
                (unsigned long long)ext.elementCount(), ext.isFullyStatic() ? 1 : 0, m->name().c_str());
    int caught = 0;
    try { lamina_b200::ArrayExtents::parse("i16:[40000]", {}); }
    catch(const std::overflow_error&) { caught += 1; }
    try { lamina_b200::RecordSchema::parse("Record{a:f33}"); }
    catch(const std::invalid_argument&) { caught += 1; }
    std::printf("caught %d\n", caught);
    return caught == 2 ? 0 : 1;
}
"""


def test_cpp_mirror_reference_signature(tmp_path, ref):
    lib = os.path.join(ROOT, "paper_2302_08251_b200", "_lib")
    src = tmp_path / "t2.cpp"
    src.write_text(SRC2)
    exe = tmp_path / "t2"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", str(src), f"-L{lib}", "-llamina_b200",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    schema_txt, ext_txt, count, static, name = out.stdout.splitlines()[0].split("|")
    info = ref.layout_info("Record{a:f32,b:Record{c:u8}}", "i64:[dyn,3]", "soa-sb", dyn=(5,))
    assert (count, static, name) == ("15", "0", info["name"])
    assert schema_txt.replace(" ", "") == "Record{a:f32,b:Record{c:u8}}"
    assert ext_txt.replace(" ", "") == "i64:[dyn,3]"
