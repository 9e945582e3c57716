// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// extern "C" shim over the *unmodified* reference library (lamina, compiled from
// /root/reference/proj by oracle/Makefile into oracle/_ref/libref.so).  It lets the
// Python test-suite, the golden-fixture generator and bench.py's CPU arms drive the
// reference's own public API:
//   parseLayout            proj/core/src/layout_spec.cpp:164
//   View(MappingPtr, blobs) proj/core/src/view.cpp:105-118
//   copyView               proj/core/src/view.cpp:168-189
//   FieldAccessCount/Heatmap proj/core/include/lamina/instrument.hpp:27-127
//   floatEncode/floatDecode proj/core/src/bitpack.cpp:96-188
//   nbody::updateStep/moveStep proj/tools/nbody/steps.hpp:13-118
// Only this file is ours; the reference sources are compiled where they lie.
#include <lamina/lamina.hpp>

#include "accessors.hpp"
#include "kernel.hpp"
#include "runner.hpp"
#include "steps.hpp"
#include "support/oracles.hpp"

#include <chrono>
#include <iostream>
#include <cstring>
#include <memory>
#include <random>

// this toolchain links libstdc++ statically into the .so; make sure the standard streams
// the reference runner writes to are constructed before it runs
static std::ios_base::Init g_iosInit;
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

using namespace lamina;

namespace
{
    thread_local std::string g_err;
    thread_local int g_kind = 0;

    // 1 invalid_argument, 2 out_of_range, 3 overflow_error, 4 logic_error, 5 other
    template<typename F>
    int guarded(F&& f)
    {
        try
        {
            f();
            g_err.clear();
            g_kind = 0;
            return 0;
        }
        catch(const std::invalid_argument& e)
        {
            g_err = e.what();
            g_kind = 1;
        }
        catch(const std::out_of_range& e)
        {
            g_err = e.what();
            g_kind = 2;
        }
        catch(const std::overflow_error& e)
        {
            g_err = e.what();
            g_kind = 3;
        }
        catch(const std::logic_error& e)
        {
            g_err = e.what();
            g_kind = 4;
        }
        catch(const std::exception& e)
        {
            g_err = e.what();
            g_kind = 5;
        }
        return g_kind;
    }

    /// wrap bit0: FieldAccessCount, bit1: Heatmap(granularity) — Heatmap outermost.
    MappingPtr makeMapping(
        const char* schemaText,
        const char* extentsText,
        const std::uint64_t* dyn,
        std::size_t ndyn,
        const char* layout,
        int wrap,
        std::uint64_t gran)
    {
        const RecordSchema schema = RecordSchema::parse(schemaText);
        const ArrayExtents ext = ArrayExtents::parse(extentsText, std::span<const std::uint64_t>(dyn, ndyn));
        MappingPtr m = parseLayout(layout, schema, ext);
        if(wrap & 1)
            m = std::make_shared<const FieldAccessCount>(m);
        if(wrap & 2)
            m = std::make_shared<const Heatmap>(m, static_cast<std::size_t>(gran));
        return m;
    }

    const FieldAccessCount* facOf(const Mapping* m)
    {
        while(m != nullptr)
        {
            if(auto f = dynamic_cast<const FieldAccessCount*>(m))
                return f;
            m = m->inner();
        }
        return nullptr;
    }

    const Heatmap* heatOf(const Mapping* m)
    {
        while(m != nullptr)
        {
            if(auto h = dynamic_cast<const Heatmap*>(m))
                return h;
            m = m->inner();
        }
        return nullptr;
    }

    View adopt(MappingPtr m, void* const* blobs)
    {
        std::vector<Blob> bl;
        for(std::size_t nr = 0; nr < m->blobCount(); ++nr)
        {
            Blob b(m->blobSize(nr));
            if(b.size() > 0)
                std::memcpy(b.data(), blobs[nr], b.size());
            bl.push_back(std::move(b));
        }
        return View(std::move(m), std::move(bl));
    }

    void giveBack(const View& v, void* const* blobs)
    {
        for(std::size_t nr = 0; nr < v.blobs().size(); ++nr)
            if(v.blobs()[nr].size() > 0)
                std::memcpy(blobs[nr], v.blobs()[nr].data(), v.blobs()[nr].size());
    }

    void exportCounters(const Mapping& m, std::uint64_t* fac, std::uint64_t* heat)
    {
        if(fac != nullptr)
            if(auto f = facOf(&m))
            {
                const auto c = f->counters();
                const std::size_t L = c.reads.size();
                for(std::size_t i = 0; i < L; ++i)
                {
                    fac[i] = c.reads[i];
                    fac[L + i] = c.writes[i];
                }
            }
        if(heat != nullptr)
            if(auto h = heatOf(&m))
            {
                std::size_t k = 0;
                for(std::size_t nr = 0; nr < h->blobCount(); ++nr)
                    for(std::size_t b = 0; b < h->blockCount(nr); ++b)
                        heat[k++] = h->blockCounter(nr, b);
            }
    }

    double now()
    {
        return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    }

    /// lamina::copyView(src, dst) (view.cpp:168-189) for nthreads <= 1; otherwise the same
    /// dispatch with the fieldwise loop body dst.write(i,f,src.read(i,f)) (view.cpp:186-188)
    /// over disjoint 64-element-aligned index ranges, and the blob memcpy path split by bytes.
    void copyThreaded(const View& src, View& dst, int nthreads)
    {
        if(nthreads <= 1)
            copyView(src, dst);
        else
        {
            const Mapping& a = src.mapping();
            const Mapping& b = dst.mapping();
            if(!(a.schema() == b.schema()) || !(a.extents() == b.extents()))
                throw std::invalid_argument("incompatible views");
            const bool sameLayout = a.name() == b.name() && !a.hasMutableState()
                && !b.hasMutableState() && a.isFullyPhysical() && b.isFullyPhysical();
            std::vector<std::thread> pool;
            if(sameLayout)
            {
                for(int t = 0; t < nthreads; ++t)
                    pool.emplace_back(
                        [&, t]
                        {
                            for(std::size_t nr = 0; nr < a.blobCount(); ++nr)
                            {
                                const std::size_t sz = a.blobSize(nr);
                                const std::size_t lo = sz * t / nthreads;
                                const std::size_t hi = sz * (t + 1) / nthreads;
                                std::memcpy(
                                    dst.blobs()[nr].data() + lo,
                                    src.blobs()[nr].data() + lo,
                                    hi - lo);
                            }
                        });
            }
            else
            {
                const std::uint64_t n = a.elementCount();
                const std::size_t leaves = a.schema().leafCount();
                const std::uint64_t units = (n + 63) / 64;
                for(int t = 0; t < nthreads; ++t)
                    pool.emplace_back(
                        [&, t]
                        {
                            const std::uint64_t lo = std::min(n, units * t / nthreads * 64);
                            const std::uint64_t hi = std::min(n, units * (t + 1) / nthreads * 64);
                            for(std::uint64_t i = lo; i < hi; ++i)
                                for(std::size_t f = 0; f < leaves; ++f)
                                    dst.write(i, f, src.read(i, f));
                        });
            }
            for(auto& th : pool)
                th.join();
        }
    }
} // namespace

extern "C"
{
    const char* ref_last_error()
    {
        return g_err.c_str();
    }

    int ref_last_kind()
    {
        return g_kind;
    }

    /// Mapping metadata: canonical name, blob sizes, leaf count, heatmap block count.
    int ref_layout_info(
        const char* schema,
        const char* extents,
        const std::uint64_t* dyn,
        std::size_t ndyn,
        const char* layout,
        int wrap,
        std::uint64_t gran,
        char* nameOut,
        std::size_t nameCap,
        std::uint64_t* blobSizes,
        std::size_t cap,
        std::size_t* nblobs,
        std::size_t* nleaves,
        std::size_t* heatBlocks)
    {
        return guarded(
            [&]
            {
                const MappingPtr m = makeMapping(schema, extents, dyn, ndyn, layout, wrap, gran);
                const std::string n = m->name();
                if(nameOut != nullptr && nameCap > 0)
                {
                    std::strncpy(nameOut, n.c_str(), nameCap - 1);
                    nameOut[nameCap - 1] = '\0';
                }
                *nblobs = m->blobCount();
                for(std::size_t i = 0; i < m->blobCount() && i < cap; ++i)
                    blobSizes[i] = m->blobSize(i);
                *nleaves = m->schema().leafCount();
                std::size_t hb = 0;
                if(auto h = heatOf(m.get()))
                    for(std::size_t nr = 0; nr < h->blobCount(); ++nr)
                        hb += h->blockCount(nr);
                *heatBlocks = hb;
            });
    }

    /// lamina::copyView(src, dst) on views adopting the given blob bytes; dst blobs
    /// (in/out) carry the destination's prior bytes in and the result out.
    /// nthreads > 1 runs the reference loop body dst.write(i,f,src.read(i,f))
    /// (view.cpp:186-188) over disjoint, 64-element-aligned index ranges.
    int ref_copy(
        const char* schema,
        const char* extents,
        const std::uint64_t* dyn,
        std::size_t ndyn,
        const char* srcLayout,
        int srcWrap,
        std::uint64_t srcGran,
        const char* dstLayout,
        int dstWrap,
        std::uint64_t dstGran,
        void* const* srcBlobs,
        void* const* dstBlobs,
        int nthreads,
        int repeats,
        std::uint64_t* srcFac,
        std::uint64_t* dstFac,
        std::uint64_t* srcHeat,
        std::uint64_t* dstHeat,
        double* seconds)
    {
        return guarded(
            [&]
            {
                View src = adopt(makeMapping(schema, extents, dyn, ndyn, srcLayout, srcWrap, srcGran), srcBlobs);
                View dst = adopt(makeMapping(schema, extents, dyn, ndyn, dstLayout, dstWrap, dstGran), dstBlobs);
                double best = 1e300;
                for(int r = 0; r < (repeats < 1 ? 1 : repeats); ++r)
                {
                    if(auto f = facOf(&src.mapping()))
                        f->reset();
                    if(auto f = facOf(&dst.mapping()))
                        f->reset();
                    if(auto h = heatOf(&src.mapping()))
                        h->reset();
                    if(auto h = heatOf(&dst.mapping()))
                        h->reset();
                    const double t0 = now();
                    copyThreaded(src, dst, nthreads);
                    best = std::min(best, now() - t0);
                }
                if(seconds != nullptr)
                    *seconds = best;
                giveBack(dst, dstBlobs);
                exportCounters(src.mapping(), srcFac, srcHeat);
                exportCounters(dst.mapping(), dstFac, dstHeat);
            });
    }

    /// Resident reference views (for timing loops and chunked checks without the per-call
    /// blob adoption copies of ref_copy): a lamina::View owning zeroed Blobs
    /// (view.hpp:108-111, blob.hpp:18-29), its blob pointers, copyView between two of them.
    void* ref_view_new(const char* schema, const char* extents, const std::uint64_t* dyn, std::size_t ndyn,
                       const char* layout, int wrap, std::uint64_t gran)
    {
        View* out = nullptr;
        guarded([&] { out = new View(makeMapping(schema, extents, dyn, ndyn, layout, wrap, gran)); });
        return out;
    }

    void ref_view_free(void* h)
    {
        delete static_cast<View*>(h);
    }

    std::size_t ref_view_blob_count(void* h)
    {
        return static_cast<View*>(h)->blobs().size();
    }

    void* ref_view_blob(void* h, std::size_t nr, std::uint64_t* size)
    {
        auto& b = static_cast<View*>(h)->blobs()[nr];
        *size = b.size();
        return b.data();
    }

    int ref_view_copy(void* src, void* dst, int nthreads, double* seconds, std::uint64_t* dstFac)
    {
        return guarded(
            [&]
            {
                View& s = *static_cast<View*>(src);
                View& d = *static_cast<View*>(dst);
                if(auto f = facOf(&d.mapping()))
                    f->reset();
                const double t0 = now();
                copyThreaded(s, d, nthreads);
                if(seconds != nullptr)
                    *seconds = now() - t0;
                exportCounters(d.mapping(), dstFac, nullptr);
            });
    }

    /// View::isTriviallyRelocatable / stateBytes / blobBytes (view.cpp:145-162) of a fresh view,
    /// ArrayExtents::isFullyStatic and Mapping::runtimeStateBytes of its mapping.
    int ref_state_info(const char* schema, const char* extents, const std::uint64_t* dyn, std::size_t ndyn,
                       const char* layout, int wrap, std::uint64_t gran, int* fullyStatic, std::uint64_t* runtimeState,
                       int* relocatable, std::uint64_t* stateBytes, std::uint64_t* blobBytes)
    {
        return guarded(
            [&]
            {
                View v(makeMapping(schema, extents, dyn, ndyn, layout, wrap, gran));
                *fullyStatic = v.mapping().extents().isFullyStatic() ? 1 : 0;
                *runtimeState = v.mapping().runtimeStateBytes();
                *relocatable = v.isTriviallyRelocatable() ? 1 : 0;
                *stateBytes = v.stateBytes();
                *blobBytes = v.blobBytes();
            });
    }

    /// Writes logical values (storage bits of the leaf's own type, one u64 per
    /// (i, f), i-major) through View::write into a zero-initialised view.
    int ref_write_values(
        const char* schema,
        const char* extents,
        const std::uint64_t* dyn,
        std::size_t ndyn,
        const char* layout,
        const std::uint64_t* values,
        void* const* blobsOut)
    {
        return guarded(
            [&]
            {
                View v(makeMapping(schema, extents, dyn, ndyn, layout, 0, 0));
                const std::uint64_t n = v.elementCount();
                const std::size_t L = v.schema().leafCount();
                for(std::uint64_t i = 0; i < n; ++i)
                    for(std::size_t f = 0; f < L; ++f)
                        v.write(i, f, ScalarValue::fromStorageBits(v.schema().leaf(f).type, values[i * L + f]));
                giveBack(v, blobsOut);
            });
    }

    /// Reads every (i, f) through View::read; returns storage bits of the logical type.
    int ref_read_values(
        const char* schema,
        const char* extents,
        const std::uint64_t* dyn,
        std::size_t ndyn,
        const char* layout,
        void* const* blobs,
        std::uint64_t* valuesOut)
    {
        return guarded(
            [&]
            {
                View v = adopt(makeMapping(schema, extents, dyn, ndyn, layout, 0, 0), blobs);
                const std::uint64_t n = v.elementCount();
                const std::size_t L = v.schema().leafCount();
                for(std::uint64_t i = 0; i < n; ++i)
                    for(std::size_t f = 0; f < L; ++f)
                        valuesOut[i * L + f] = v.read(i, f).storageBits();
            });
    }

    /// oracle::scalarSample (tests/support/oracles.cpp:211-223) as storage bits.
    std::uint64_t ref_scalar_sample(int kind, std::uint64_t salt)
    {
        return oracle::scalarSample(static_cast<Scalar>(kind), salt).storageBits();
    }

    std::uint64_t ref_float_encode(double v, unsigned e, unsigned m)
    {
        return floatEncode(v, e, m);
    }

    double ref_float_decode(std::uint64_t p, unsigned e, unsigned m)
    {
        return floatDecode(p, e, m);
    }

    /// floatEncode over an array of f32 bit patterns (value widened to double as
    /// ScalarValue::asFloat does, scalar.hpp:209-214).
    void ref_float_encode_f32_array(const std::uint32_t* in, std::uint64_t* out, std::size_t n, unsigned e, unsigned m)
    {
        for(std::size_t i = 0; i < n; ++i)
        {
            float f;
            std::memcpy(&f, &in[i], 4);
            out[i] = floatEncode(static_cast<double>(f), e, m);
        }
    }

    /// ScalarValue f64 -> f32 -> bits (ChangeType write path, scalar.hpp:295-306).
    void ref_f64_to_f32_array(const std::uint64_t* in, std::uint32_t* out, std::size_t n)
    {
        for(std::size_t i = 0; i < n; ++i)
            out[i] = static_cast<std::uint32_t>(
                ScalarValue::fromStorageBits(Scalar::F64, in[i]).convertTo(Scalar::F32).storageBits());
    }

    void ref_f32_to_f64_array(const std::uint32_t* in, std::uint64_t* out, std::size_t n)
    {
        for(std::size_t i = 0; i < n; ++i)
            out[i] = ScalarValue::fromStorageBits(Scalar::F32, in[i]).convertTo(Scalar::F64).storageBits();
    }

    /// The reference n-body benchmark body (tools/nbody/runner.cpp:326-438 without
    /// the CLI): drawInitValues(seed) + initView, `steps` x (update, move) through the
    /// same accessor selection, then checksum. Blobs of the final view are copied
    /// out when blobsOut != nullptr. nthreads > 1 runs updateStep's i-loop body
    /// over disjoint W-aligned i-blocks (positions are read-only during update).
    int ref_nbody(
        const char* layout,
        std::uint64_t n,
        std::uint64_t steps,
        int f64,
        std::uint64_t seed,
        int width,
        int nthreads,
        void* const* blobsOut,
        double* checksum,
        double* updateSeconds,
        double* moveSeconds)
    {
        return guarded(
            [&]
            {
                auto run = [&]<typename T>(T)
                {
                    const RecordSchema schema = RecordSchema::parse(
                        std::is_same_v<T, float>
                            ? "Record{Pos: Record{x: f32, y: f32, z: f32}, Vel: Record{x: f32, y: f32, z: f32}, Mass: f32}"
                            : "Record{Pos: Record{x: f64, y: f64, z: f64}, Vel: Record{x: f64, y: f64, z: f64}, Mass: f64}");
                    const ArrayExtents extents(IndexType::I64, {n}, {});
                    MappingPtr mapping = parseLayout(layout, schema, extents);
                    View view(mapping);
                    // drawInitValues: runner.cpp:30-43 (restated; anonymous namespace there)
                    std::mt19937_64 gen(seed);
                    const auto uniform = [&] { return static_cast<double>(gen() >> 11) * 0x1.0p-53; };
                    for(std::uint64_t i = 0; i < n; ++i)
                    {
                        const double px = uniform(), py = uniform(), pz = uniform(), m = uniform();
                        view.write(i, nbody::kPosX, ScalarValue::of<T>(static_cast<T>(px)));
                        view.write(i, nbody::kPosY, ScalarValue::of<T>(static_cast<T>(py)));
                        view.write(i, nbody::kPosZ, ScalarValue::of<T>(static_cast<T>(pz)));
                        view.write(i, nbody::kVelX, ScalarValue::of<T>(T{0}));
                        view.write(i, nbody::kVelY, ScalarValue::of<T>(T{0}));
                        view.write(i, nbody::kVelZ, ScalarValue::of<T>(T{0}));
                        view.write(i, nbody::kMass, ScalarValue::of<T>(static_cast<T>(m)));
                    }
                    const bool affine = dynamic_cast<const AoSMapping*>(mapping.get()) != nullptr
                        || dynamic_cast<const SoAMapping*>(mapping.get()) != nullptr;
                    const auto* aosoa = dynamic_cast<const AoSoAMapping*>(mapping.get());
                    auto updateRange = [&](std::uint64_t lo, std::uint64_t hi)
                    {
                        // updateStep<T,1> restricted to [lo, hi): same j order per i
                        const T eps2 = static_cast<T>(nbody::kEps2);
                        const T dt = static_cast<T>(nbody::kDt);
                        auto body = [&](const auto& acc)
                        {
                            for(std::uint64_t i = lo; i < hi; ++i)
                            {
                                const T px = view.load<T>(i, nbody::kPosX);
                                const T py = view.load<T>(i, nbody::kPosY);
                                const T pz = view.load<T>(i, nbody::kPosZ);
                                T vx = view.load<T>(i, nbody::kVelX);
                                T vy = view.load<T>(i, nbody::kVelY);
                                T vz = view.load<T>(i, nbody::kVelZ);
                                for(std::uint64_t j = 0; j < n; ++j)
                                    nbody::pPInteraction(
                                        px,
                                        py,
                                        pz,
                                        vx,
                                        vy,
                                        vz,
                                        acc.template get<nbody::kPosX>(j),
                                        acc.template get<nbody::kPosY>(j),
                                        acc.template get<nbody::kPosZ>(j),
                                        acc.template get<nbody::kMass>(j),
                                        eps2,
                                        dt);
                                view.store<T>(i, nbody::kVelX, vx);
                                view.store<T>(i, nbody::kVelY, vy);
                                view.store<T>(i, nbody::kVelZ, vz);
                            }
                        };
                        if(affine)
                            body(nbody::AffineAccessor<T>(view));
                        else if(aosoa != nullptr)
                            body(nbody::AoSoAAccessor<T>(view, *aosoa));
                        else
                            body(nbody::FunnelAccessor<T>(view));
                    };
                    auto step = [&](bool update)
                    {
                        if(nthreads <= 1)
                        {
                            // the reference's own templates, width W
                            auto dispatch = [&]<std::size_t W>()
                            {
                                if(!update)
                                {
                                    nbody::moveStep<T, W>(view, n);
                                    return;
                                }
                                if(affine)
                                    nbody::updateStep<T, W>(view, nbody::AffineAccessor<T>(view), n);
                                else if(aosoa != nullptr)
                                    nbody::updateStep<T, W>(view, nbody::AoSoAAccessor<T>(view, *aosoa), n);
                                else
                                    nbody::updateStep<T, W>(view, nbody::FunnelAccessor<T>(view), n);
                            };
                            switch(width)
                            {
                            case 1: dispatch.template operator()<1>(); break;
                            case 2: dispatch.template operator()<2>(); break;
                            case 4: dispatch.template operator()<4>(); break;
                            case 8: dispatch.template operator()<8>(); break;
                            case 16: dispatch.template operator()<16>(); break;
                            default: throw std::invalid_argument("unsupported simd width");
                            }
                            return;
                        }
                        if(!update)
                        {
                            nbody::moveStep<T, 1>(view, n);
                            return;
                        }
                        std::vector<std::thread> pool;
                        for(int t = 0; t < nthreads; ++t)
                            pool.emplace_back([&, t] { updateRange(n * t / nthreads, n * (t + 1) / nthreads); });
                        for(auto& th : pool)
                            th.join();
                    };
                    double upd = 0, mov = 0;
                    for(std::uint64_t s = 0; s < steps; ++s)
                    {
                        const double t0 = now();
                        step(true);
                        const double t1 = now();
                        step(false);
                        const double t2 = now();
                        upd += t1 - t0;
                        mov += t2 - t1;
                    }
                    if(updateSeconds != nullptr)
                        *updateSeconds = steps ? upd / steps : 0;
                    if(moveSeconds != nullptr)
                        *moveSeconds = steps ? mov / steps : 0;
                    double sum = 0;
                    for(std::uint64_t i = 0; i < n; ++i)
                    {
                        sum += view.read(i, nbody::kPosX).asFloat();
                        sum += view.read(i, nbody::kPosY).asFloat();
                        sum += view.read(i, nbody::kPosZ).asFloat();
                    }
                    *checksum = sum;
                    if(blobsOut != nullptr)
                        giveBack(view, blobsOut);
                };
                if(f64)
                    run(double{});
                else
                    run(float{});
            });
    }

    /// The shipped CLI entry (runner.cpp:441-466) for KAT cross-checks; prints CSV.
    int ref_nbody_cli(const char* layout, std::uint64_t n, std::uint64_t steps, int f64, std::uint64_t seed, int width)
    {
        nbody::BenchConfig cfg;
        cfg.layout = layout;
        cfg.n = n;
        cfg.steps = steps;
        cfg.precision = f64 ? "f64" : "f32";
        cfg.seed = seed;
        cfg.simdWidth = static_cast<std::size_t>(width);
        return nbody::runBenchmark(cfg);
    }

    // Mapping::contiguousRun of the reference mapping (mapping.hpp:122-135)
    int ref_contiguous_run(const char* schema, const char* extents, const std::uint64_t* dyn, std::size_t ndyn,
                           const char* layout, int wrap, std::uint64_t gran, std::uint64_t linear, std::size_t leaf,
                           std::uint64_t n, int* has, std::size_t* nr, std::uint64_t* off)
    {
        return guarded(
            [&]
            {
                const MappingPtr m = makeMapping(schema, extents, dyn, ndyn, layout, wrap, gran);
                const auto run = m->contiguousRun(linear, leaf, n);
                *has = run ? 1 : 0;
                if(run)
                {
                    *nr = run->nr;
                    *off = run->offset;
                }
            });
    }

    // the runner with --trace-fields / --heatmap <g>: writes fields_{update,move}.csv and
    // heatmap_{update,move}.csv into reportDir (runner.cpp:344-436)
    int ref_nbody_trace(const char* layout, std::uint64_t n, std::uint64_t steps, int f64, std::uint64_t seed,
                        int traceFields, std::uint64_t heatGran, const char* reportDir, const char* csvPath)
    {
        nbody::BenchConfig cfg;
        cfg.layout = layout;
        cfg.n = n;
        cfg.steps = steps;
        cfg.precision = f64 ? "f64" : "f32";
        cfg.seed = seed;
        cfg.traceFields = traceFields != 0;
        cfg.heatmapGranularity = static_cast<std::size_t>(heatGran);
        cfg.reportDir = reportDir;
        cfg.csvPath = csvPath ? csvPath : "";
        return nbody::runBenchmark(cfg);
    }
}
