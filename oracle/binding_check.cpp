// TEST INFRASTRUCTURE: compiles INTEGRATION.md §1's maintainer-side binding
// (include/lamina_b200_binding.hpp) against the reference's own headers and library, and
// runs lamina::copyViewB200 (this repo's GPU path through the C ABI) next to
// lamina::copyView (the reference, view.cpp:168-189) on the same lamina::View objects.
// Built by oracle/Makefile into oracle/_ref/binding_check (linked with the reference objects
// and paper_2302_08251_b200/_lib/liblamina_b200.so); run by tests/test_gpu_binding.py.
// Prints one line per case and "binding_check: OK <n> cases" (exit 0) or the first failure.
#include <lamina/lamina.hpp>

#include "lamina_b200_binding.hpp"
#include "support/oracles.hpp"

#include <cstdio>
#include <cstring>
#include <iostream>
#include <memory>
#include <string>
#include <vector>

using namespace lamina;

namespace
{
    int g_fail = 0;

    void fail(const std::string& what)
    {
        std::cout << "FAIL " << what << std::endl;
        ++g_fail;
    }

    MappingPtr wrapped(MappingPtr m, int wrap, std::size_t gran)
    {
        if(wrap & 1)
            m = std::make_shared<const FieldAccessCount>(m);
        if(wrap & 2)
            m = std::make_shared<const Heatmap>(m, gran);
        return m;
    }

    const FieldAccessCount* facOf(const Mapping* m)
    {
        for(; m; m = m->inner())
            if(auto* f = dynamic_cast<const FieldAccessCount*>(m))
                return f;
        return nullptr;
    }

    const Heatmap* heatOf(const Mapping* m)
    {
        for(; m; m = m->inner())
            if(auto* h = dynamic_cast<const Heatmap*>(m))
                return h;
        return nullptr;
    }

    // dst side counters of the reference after copyView vs the binding's deltas
    bool countersMatch(const Mapping& ref, const std::vector<std::uint64_t>& reads,
                       const std::vector<std::uint64_t>& writes, const std::vector<std::vector<std::uint64_t>>& heat)
    {
        if(auto* f = facOf(&ref))
        {
            const auto c = f->counters();
            if(c.reads != reads || c.writes != writes)
                return false;
        }
        if(auto* h = heatOf(&ref))
        {
            if(heat.size() != h->blobCount())
                return false;
            for(std::size_t nr = 0; nr < h->blobCount(); ++nr)
                for(std::size_t b = 0; b < h->blockCount(nr); ++b)
                    if(heat[nr][b] != h->blockCounter(nr, b))
                        return false;
        }
        return true;
    }

    void runCase(const std::string& schemaText, std::uint64_t n, const std::string& a, int wa, const std::string& b,
                 int wb, std::size_t gran)
    {
        const RecordSchema schema = RecordSchema::parse(schemaText);
        const ArrayExtents ext(IndexType::I32, {n}, {});
        // the source: every (i, f) written through the reference's View::write
        View src(wrapped(parseLayout(a, schema, ext), wa, gran));
        for(std::uint64_t i = 0; i < n; ++i)
            for(std::size_t f = 0; f < schema.leafCount(); ++f)
                src.write(i, f, oracle::scalarSample(schema.leaf(f).type, i * 131 + f));
        if(auto* fc = facOf(&src.mapping()))
            fc->reset();
        if(auto* h = heatOf(&src.mapping()))
            h->reset();
        View ref(wrapped(parseLayout(b, schema, ext), wb, gran));
        View gpu(wrapped(parseLayout(b, schema, ext), wb, gran));
        copyView(src, ref);
        B200CopyCounters d;
        // the source's counters must not change through the binding: snapshot, then compare
        copyViewB200(src, gpu, 0, &d);
        const std::string tag = schemaText.substr(0, 24) + " n=" + std::to_string(n) + " " + src.mapping().name()
            + " -> " + gpu.mapping().name();
        for(std::size_t nr = 0; nr < ref.blobs().size(); ++nr)
            if(ref.blobs()[nr].size() != gpu.blobs()[nr].size()
               || std::memcmp(ref.blobs()[nr].data(), gpu.blobs()[nr].data(), ref.blobs()[nr].size()) != 0)
            {
                fail(tag + ": blob " + std::to_string(nr) + " differs");
                return;
            }
        if(!countersMatch(ref.mapping(), d.dstReads, d.dstWrites, d.dstHeat))
        {
            fail(tag + ": destination counters differ");
            return;
        }
        // source-side deltas: the reference's src counters after its copyView equal the
        // binding's src deltas (src was reset before the reference copy ran)
        if(!countersMatch(src.mapping(), d.srcReads, d.srcWrites, d.srcHeat))
        {
            fail(tag + ": source counter deltas differ");
            return;
        }
        std::cout << "ok " << tag << std::endl;
    }

    // a user-defined Mapping (mapping.hpp:44-155): reversed AoS, unknown to the grammar
    class ReversedAoS final : public Mapping
    {
    public:
        ReversedAoS(RecordSchema s, ArrayExtents e) : Mapping(std::move(s), std::move(e))
        {
        }
        std::string name() const override
        {
            return "user-reversed-aos";
        }
        std::size_t blobCount() const override
        {
            return 1;
        }
        std::size_t blobSize(std::size_t) const override
        {
            return elementCount() * schema().sizePacked();
        }
        NrAndOffset physicalOffset(std::uint64_t linear, std::size_t flatLeaf) const override
        {
            return {0, (elementCount() - 1 - linear) * schema().sizePacked() + schema().leaf(flatLeaf).offsetPacked};
        }
    };
} // namespace

int main()
{
    const std::string R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}";
    const std::string R64 = "Record{Pos:Record{x:f64,y:f64,z:f64},Vel:Record{x:f64,y:f64,z:f64},Mass:f64}";
    const std::string MIX = "Record{a:i8,b:u16,c:i32,d:u64,e:f32,f:f64,g:bool,h:Record{x:i16,y:f32[3]}}";
    const std::vector<std::string> r32 = {"aos-packed", "soa-sb", "soa-mb", "aosoa:8", "aosoa:32", "aosoa:3",
                                          "bytesplit:soa-mb", "bitpack-float:5,10", "split:Pos:soa-mb:aos-packed",
                                          "changetype:f32=f64:soa-mb"};
    int cases = 0;
    for(const auto& a : r32)
        for(const auto& b : r32)
        {
            runCase(R32, 4099, a, 0, b, 0, 1);
            ++cases;
        }
    for(int w : {1, 2, 3})
        for(std::size_t g : {1, 5, 64})
        {
            runCase(R32, 1000, "aos-packed", 0, "soa-mb", w, g);
            runCase(R32, 1000, "soa-mb", w, "bytesplit:aosoa:4", 0, g);
            cases += 2;
        }
    runCase(R64, 10007, "aos-packed", 0, "changetype:f64=f32:bytesplit:soa-mb", 1, 1); // the C5 shape
    runCase(MIX, 777, "aos-packed", 0, "soa-mb", 0, 1);
    runCase(MIX, 777, "aosoa:4", 0, "changetype:f64=f32,i8=i64,u16=u8:aosoa:2", 1, 1);
    runCase("Record{v:u32,w:i32}", 5003, "soa-mb", 0, "bitpack-int:11", 0, 1);
    cases += 4;

    // errors: the reference's exception and message through the binding
    {
        const RecordSchema s = RecordSchema::parse(R32);
        View x(parseLayout("aos-packed", s, ArrayExtents(IndexType::I32, {8}, {})));
        View y(parseLayout("soa-mb", s, ArrayExtents(IndexType::I32, {9}, {})));
        try
        {
            copyViewB200(x, y);
            fail("incompatible views not rejected");
        }
        catch(const std::invalid_argument& e)
        {
            if(std::string(e.what()).find("incompatible views") == std::string::npos)
                fail(std::string("incompatible views message: ") + e.what());
        }
        View u(std::make_shared<const ReversedAoS>(s, ArrayExtents(IndexType::I32, {8}, {})));
        try
        {
            copyViewB200(u, x);
            fail("user-defined mapping not rejected");
        }
        catch(const std::invalid_argument& e)
        {
            if(std::string(e.what()).find("cannot be lowered") == std::string::npos)
                fail(std::string("user mapping message: ") + e.what());
        }
        copyView(u, x); // the reference path still serves it
        cases += 2;
    }
    if(g_fail)
    {
        std::cout << "binding_check: " << g_fail << " FAILED of " << cases << " cases" << std::endl;
        return 1;
    }
    std::cout << "binding_check: OK " << cases << " cases" << std::endl;
    return 0;
}
