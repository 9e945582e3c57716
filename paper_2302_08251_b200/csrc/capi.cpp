// C ABI (include/lamina_b200.h): host-side plumbing of the B200 path.  Owns layout
// handles, device views (blobs + device plan + device counters), view dump/restore and the
// copy entry points.  The copy dispatch itself (copy_dispatch.cpp -> copy_tile_host.cpp):
//   copyView fast path (view.cpp:175-181)      -> lamk::blob_copy per blob
//   plan pairs with a specialised kernel        -> vec_transpose / pack32 / planes / vec_convert /
//                                                  uniform_direct / warp_tile (copy_tile_host.cpp)
//   everything else                              -> lamk::generic_copy (copy_generic.cu)
#include "capi_internal.hpp"

#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <vector>

using namespace lamb;

thread_local std::string g_lam_err;

namespace
{
    struct CudaError : std::runtime_error
    {
        using std::runtime_error::runtime_error;
    };

    template<typename F>
    int guard(F&& f)
    {
        try
        {
            f();
            return LAM_OK;
        }
        catch(const CudaError& e)
        {
            g_lam_err = e.what();
            return LAM_ECUDA;
        }
        catch(const std::invalid_argument& e)
        {
            g_lam_err = e.what();
            return LAM_EINVAL;
        }
        catch(const std::out_of_range& e)
        {
            g_lam_err = e.what();
            return LAM_ERANGE;
        }
        catch(const std::overflow_error& e)
        {
            g_lam_err = e.what();
            return LAM_EOVERFLOW;
        }
        catch(const std::logic_error& e)
        {
            g_lam_err = e.what();
            return LAM_ELOGIC;
        }
        catch(const std::exception& e)
        {
            g_lam_err = e.what();
            return LAM_ERUNTIME;
        }
    }

    size_t copyOut(const std::string& s, char* buf, size_t cap)
    {
        if(buf && cap)
        {
            const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
            std::memcpy(buf, s.data(), n);
            buf[n] = '\0';
        }
        return s.size();
    }

} // namespace

void lam_cuda_check(cudaError_t e, const char* what)
{
    if(e != cudaSuccess)
    {
        cudaGetLastError();
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
    }
}

// ---- device view images ------------------------------------------------------------------
namespace lamhost
{
    static size_t align16(size_t x)
    {
        return (x + 15) & ~size_t{15};
    }

    DeviceImage::~DeviceImage()
    {
        release();
    }

    void DeviceImage::release()
    {
        if(mem)
        {
            int cur = -1;
            cudaGetDevice(&cur);
            if(cur != device)
                cudaSetDevice(device);
            cudaFree(mem);
            if(heat && ownsHeat)
                cudaFree(heat);
            if(cur != device && cur >= 0)
                cudaSetDevice(cur);
        }
        mem = nullptr;
        heat = nullptr;
    }

    void DeviceImage::build(const Lowered& L, int dev, const std::vector<uint8_t*>& streamPtrs, void* sharedHeat)
    {
        release();
        device = dev;
        ownsHeat = sharedHeat == nullptr;
        const size_t nleaves = L.roots.size();
        const size_t nblobs = L.map->blobCount();
        // header | roots | nodes | streams | stream_ptr | heat_offset | fac
        offRoots = align16(sizeof(lamp_view));
        offNodes = align16(offRoots + nleaves * sizeof(uint16_t));
        offStreams = align16(offNodes + L.nodes.size() * sizeof(lamp_node));
        offPtrs = align16(offStreams + L.streams.size() * sizeof(lamp_stream));
        offHeatOff = align16(offPtrs + L.streams.size() * sizeof(uint8_t*));
        offFac = align16(offHeatOff + nblobs * sizeof(uint64_t));
        bytes = align16(offFac + 2 * nleaves * sizeof(uint64_t));
        host.assign(bytes, 0);
        lam_cuda_check(cudaMalloc(&mem, bytes), "cudaMalloc(view plan)");
        if(L.heat && L.heatTotal && sharedHeat)
            heat = sharedHeat;
        else if(L.heat && L.heatTotal)
        {
            lam_cuda_check(cudaMalloc(&heat, L.heatTotal * sizeof(uint64_t)), "cudaMalloc(heatmap)");
            lam_cuda_check(cudaMemset(heat, 0, L.heatTotal * sizeof(uint64_t)), "cudaMemset(heatmap)");
        }
        uint8_t* d = static_cast<uint8_t*>(mem);
        lamp_view h{};
        h.n = L.map->elementCount();
        h.nleaves = static_cast<uint32_t>(nleaves);
        h.nnodes = static_cast<uint32_t>(L.nodes.size());
        h.nstreams = static_cast<uint32_t>(L.streams.size());
        h.nblobs = static_cast<uint32_t>(nblobs);
        h.fac = L.fac;
        h.heat = L.heat;
        h.heat_gran = L.heatGran;
        h.roots = reinterpret_cast<const uint16_t*>(d + offRoots);
        h.nodes = reinterpret_cast<const lamp_node*>(d + offNodes);
        h.streams = reinterpret_cast<const lamp_stream*>(d + offStreams);
        h.stream_ptr = reinterpret_cast<uint8_t* const*>(d + offPtrs);
        h.heat_offset = reinterpret_cast<const uint64_t*>(d + offHeatOff);
        h.fac_counters = reinterpret_cast<unsigned long long*>(d + offFac);
        h.heat_counters = static_cast<unsigned long long*>(heat);
        std::memcpy(host.data(), &h, sizeof h);
        if(nleaves)
            std::memcpy(host.data() + offRoots, L.roots.data(), nleaves * sizeof(uint16_t));
        if(!L.nodes.empty())
            std::memcpy(host.data() + offNodes, L.nodes.data(), L.nodes.size() * sizeof(lamp_node));
        if(!L.streams.empty())
            std::memcpy(host.data() + offStreams, L.streams.data(), L.streams.size() * sizeof(lamp_stream));
        if(!streamPtrs.empty())
            std::memcpy(host.data() + offPtrs, streamPtrs.data(), streamPtrs.size() * sizeof(uint8_t*));
        if(L.heat && nblobs)
            std::memcpy(host.data() + offHeatOff, L.heatOffset.data(), nblobs * sizeof(uint64_t));
        lam_cuda_check(cudaMemcpy(mem, host.data(), bytes, cudaMemcpyHostToDevice), "cudaMemcpy(view plan)");
        hdr = reinterpret_cast<const lamp_view*>(mem);
        facDev = reinterpret_cast<unsigned long long*>(d + offFac);
    }

    void DeviceImage::setStreamPtrs(const std::vector<uint8_t*>& ptrs, cudaStream_t s)
    {
        std::memcpy(host.data() + offPtrs, ptrs.data(), ptrs.size() * sizeof(uint8_t*));
        lam_cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(mem) + offPtrs, host.data() + offPtrs,
                                       ptrs.size() * sizeof(uint8_t*), cudaMemcpyHostToDevice, s),
                       "cudaMemcpyAsync(stream ptrs)");
    }

    std::vector<uint8_t*> streamPtrsFor(const Lowered& L, const std::vector<void*>& blobs)
    {
        std::vector<uint8_t*> p;
        for(const auto& s : L.streams)
            p.push_back(static_cast<uint8_t*>(blobs[s.nr]) + s.base0);
        return p;
    }

} // namespace lamhost

using namespace lamhost;

// ---- C ABI ----------------------------------------------------------------------------------
extern "C"
{
    const char* lam_last_error(void)
    {
        return g_lam_err.c_str();
    }

    const char* lam_version(void)
    {
        return "lamina_b200 0.1 (sm_100a)";
    }

    int lam_layout_create(const char* schema, const char* extents, const uint64_t* dyn, size_t ndyn,
                          const char* layout, int wrap, uint64_t gran, lam_layout** out)
    {
        return guard(
            [&]
            {
                if(!schema || !extents || !layout || !out)
                    throw std::invalid_argument("null argument");
                const Schema s = Schema::parse(schema);
                const Extents e = Extents::parse(extents, dyn, ndyn);
                MapPtr m = parseLayout(layout, s, e);
                if(wrap & LAM_WRAP_FIELD_ACCESS_COUNT)
                    m = std::make_shared<FieldAccessCountMap>(m);
                if(wrap & LAM_WRAP_HEATMAP)
                    m = std::make_shared<HeatmapMap>(m, gran);
                auto* h = new lam_layout;
                h->L = lower(std::move(m));
                *out = h;
            });
    }

    void lam_layout_destroy(lam_layout* l)
    {
        delete l;
    }

    size_t lam_layout_name(const lam_layout* l, char* buf, size_t cap)
    {
        return copyOut(l->L->map->name(), buf, cap);
    }

    size_t lam_layout_schema(const lam_layout* l, char* buf, size_t cap)
    {
        return copyOut(l->L->map->schema().toString(), buf, cap);
    }

    size_t lam_layout_extents(const lam_layout* l, char* buf, size_t cap)
    {
        return copyOut(l->L->map->extents().toString(), buf, cap);
    }

    size_t lam_layout_blob_count(const lam_layout* l)
    {
        return l->L->map->blobCount();
    }

    uint64_t lam_layout_blob_size(const lam_layout* l, size_t nr)
    {
        return nr < l->L->map->blobCount() ? l->L->map->blobSize(nr) : 0;
    }

    uint64_t lam_layout_element_count(const lam_layout* l)
    {
        return l->L->map->elementCount();
    }

    size_t lam_layout_leaf_count(const lam_layout* l)
    {
        return l->L->map->schema().leafCount();
    }

    int lam_layout_leaf(const lam_layout* l, size_t f, int* kind, size_t* size, size_t* off)
    {
        return guard(
            [&]
            {
                if(f >= l->L->map->schema().leafCount())
                    throw std::out_of_range("index out of range: leaf " + std::to_string(f));
                const auto& d = l->L->map->schema().leaf(f);
                if(kind)
                    *kind = d.type;
                if(size)
                    *size = d.size;
                if(off)
                    *off = d.offsetPacked;
            });
    }

    size_t lam_layout_leaf_path(const lam_layout* l, size_t f, char* buf, size_t cap)
    {
        if(f >= l->L->map->schema().leafCount())
            return 0;
        return copyOut(l->L->map->schema().leaf(f).path, buf, cap);
    }

    int lam_layout_is_computed(const lam_layout* l, size_t f)
    {
        return f < l->L->map->schema().leafCount() && l->L->map->isComputed(f) ? 1 : 0;
    }

    int lam_layout_is_fully_physical(const lam_layout* l)
    {
        return l->L->map->isFullyPhysical() ? 1 : 0;
    }

    int lam_layout_has_mutable_state(const lam_layout* l)
    {
        return l->L->map->hasMutableState() ? 1 : 0;
    }

    int lam_layout_is_fully_static(const lam_layout* l)
    {
        return l->L->map->extents().isFullyStatic() ? 1 : 0;
    }

    uint64_t lam_layout_runtime_state_bytes(const lam_layout* l)
    {
        return l->L->map->runtimeStateBytes();
    }

    // View::isTriviallyRelocatable / blobBytes / stateBytes (view.cpp:145-162)
    int lam_view_is_trivially_relocatable(const lam_view* v)
    {
        const Map& m = *v->L->map;
        return m.extents().isFullyStatic() && !m.hasMutableState() && m.runtimeStateBytes() == 0 ? 1 : 0;
    }

    uint64_t lam_view_blob_bytes(const lam_view* v)
    {
        uint64_t total = 0;
        for(size_t nr = 0; nr < v->L->map->blobCount(); ++nr)
            total += v->L->map->blobSize(nr);
        return total;
    }

    uint64_t lam_view_state_bytes(const lam_view* v)
    {
        return lam_view_blob_bytes(v) + v->L->map->runtimeStateBytes();
    }

    int lam_layout_physical_offset(const lam_layout* l, uint64_t i, size_t f, size_t* nr, uint64_t* off)
    {
        return guard(
            [&]
            {
                const auto& m = *l->L->map;
                if(m.isComputed(f < m.schema().leafCount() ? f : 0) && f < m.schema().leafCount())
                    throw std::logic_error("computed leaf has no physical offset");
                if(i >= m.elementCount())
                    throw std::out_of_range("index out of range: element " + std::to_string(i));
                if(f >= m.schema().leafCount())
                    throw std::out_of_range("index out of range: leaf " + std::to_string(f));
                const auto o = m.offsetOf(i, f);
                *nr = o.first;
                *off = o.second;
            });
    }

    int lam_layout_contiguous_run(const lam_layout* l, uint64_t i, size_t f, uint64_t n, int* has, size_t* nr,
                                  uint64_t* off)
    {
        return guard(
            [&]
            {
                const Lowered& L = *l->L;
                const auto& m = *L.map;
                if(f >= m.schema().leafCount())
                    throw std::out_of_range("index out of range: leaf " + std::to_string(f));
                if(i >= m.elementCount())
                    throw std::out_of_range("index out of range: element " + std::to_string(i));
                *has = 0;
                // counting wrappers and computed leaves want per-element access (mapping.hpp:122-135)
                if(L.fac || L.heat)
                    return;
                const lamp_node& nd = L.nodes[L.roots[f]];
                if(nd.kind != LAMP_PHYS)
                    return;
                const lamp_stream& st = L.streams[nd.stream];
                const uint64_t size = scalarSize(nd.type);
                bool run = n <= 1;
                if(st.lanes == 1)
                    run = run || st.block_stride == size;                   // SoA; AoS of one leaf (mappings.cpp:44-50,96-101)
                else
                    run = run || (st.block_stride == st.lanes * size && nd.b == size) // one-leaf AoSoA
                        || (i % st.lanes + n <= st.lanes);                   // inside one block (mappings.cpp:140-148)
                if(!run)
                    return;
                const auto o = m.offsetOf(i, f);
                *has = 1;
                *nr = o.first;
                *off = o.second;
            });
    }

    uint64_t lam_layout_heatmap_blocks(const lam_layout* l, size_t nr)
    {
        if(!l->L->heat || nr >= l->L->map->blobCount())
            return 0;
        return (l->L->map->blobSize(nr) + l->L->heatGran - 1) / l->L->heatGran;
    }

    uint64_t lam_layout_shard_unit(const lam_layout* l)
    {
        return l->L->shardUnit;
    }

    size_t lam_layout_stream_count(const lam_layout* l)
    {
        return l->L->streams.size();
    }

    int lam_layout_stream_region(const lam_layout* l, size_t s, uint64_t begin, uint64_t end, size_t* nr,
                                 uint64_t* lo, uint64_t* hi)
    {
        return guard(
            [&]
            {
                if(s >= l->L->streams.size())
                    throw std::out_of_range("index out of range: stream " + std::to_string(s));
                if(begin > end || end > l->L->map->elementCount())
                    throw std::out_of_range("index out of range: elements");
                const lamp_stream& st = l->L->streams[s];
                uint64_t a, b;
                if(st.kind == LAMS_BITS)
                {
                    a = (begin * st.block_stride / 32) * 4;
                    b = ((end * st.block_stride + 31) / 32) * 4;
                }
                else
                {
                    a = st.base0 + (begin / st.lanes) * st.block_stride;
                    b = st.base0 + ((end + st.lanes - 1) / st.lanes) * st.block_stride;
                }
                const uint64_t size = l->L->map->blobSize(st.nr);
                *nr = st.nr;
                *lo = a < size ? a : size;
                *hi = b < size ? b : size;
            });
    }

    // ---- views ----------------------------------------------------------------------------
    int lam_view_alloc(const lam_layout* l, int device, void* stream, lam_view** out)
    {
        return guard(
            [&]
            {
                DeviceGuard g(device);
                auto v = std::make_unique<lam_view>();
                v->L = l->L;
                v->layout = l;
                v->device = device;
                v->owned = true;
                const auto& m = *l->L->map;
                auto s = static_cast<cudaStream_t>(stream);
                for(size_t nr = 0; nr < m.blobCount(); ++nr)
                {
                    void* p = nullptr;
                    const uint64_t sz = m.blobSize(nr);
                    if(sz)
                    {
                        lam_cuda_check(cudaMalloc(&p, sz), "cudaMalloc(blob)");
                        v->blobs.push_back(p); // registered before the memset so a failure frees it
                        lam_cuda_check(cudaMemsetAsync(p, 0, sz, s), "cudaMemsetAsync(blob)");
                    }
                    else
                        v->blobs.push_back(nullptr);
                }
                v->img.build(*l->L, device, streamPtrsFor(*l->L, v->blobs));
                *out = v.release();
            });
    }

    int lam_view_wrap(const lam_layout* l, int device, void* const* blobs, const uint64_t* bytes, size_t n,
                      lam_view** out)
    {
        return guard(
            [&]
            {
                const auto& m = *l->L->map;
                if(n != m.blobCount())
                    throw std::invalid_argument(
                        "blob count mismatch: mapping declares " + std::to_string(m.blobCount()) + ", got "
                        + std::to_string(n));
                if(bytes == nullptr && n > 0)
                    throw std::invalid_argument("blob size mismatch: the sizes of the adopted blobs are required");
                for(size_t nr = 0; nr < n; ++nr)
                {
                    if(bytes[nr] != m.blobSize(nr))
                        throw std::invalid_argument(
                            "blob size mismatch: blob " + std::to_string(nr) + " declares "
                            + std::to_string(m.blobSize(nr)) + ", got " + std::to_string(bytes[nr]));
                    if(reinterpret_cast<uintptr_t>(blobs[nr]) & 15)
                        throw std::invalid_argument("blob " + std::to_string(nr) + " is not 16-byte aligned");
                }
                DeviceGuard g(device);
                auto v = std::make_unique<lam_view>();
                v->L = l->L;
                v->layout = l;
                v->device = device;
                v->owned = false;
                v->blobs.assign(blobs, blobs + n);
                v->img.build(*l->L, device, streamPtrsFor(*l->L, v->blobs));
                *out = v.release();
            });
    }

    void lam_view_free(lam_view* v)
    {
        if(!v)
            return;
        {
            DeviceGuard g(v->device);
            if(v->owned)
                for(void* p : v->blobs)
                    if(p)
                        cudaFree(p);
            v->img.release();
        }
        delete v;
    }

    const lam_layout* lam_view_layout(const lam_view* v)
    {
        return v->layout;
    }

    const void* lam_view_device_plan(const lam_view* v)
    {
        return v ? v->img.hdr : nullptr;
    }

    void* lam_view_blob(const lam_view* v, size_t nr)
    {
        return nr < v->blobs.size() ? v->blobs[nr] : nullptr;
    }

    int lam_view_upload(lam_view* v, size_t nr, const void* host, void* stream)
    {
        return guard(
            [&]
            {
                if(nr >= v->blobs.size())
                    throw std::out_of_range("index out of range: blob " + std::to_string(nr));
                DeviceGuard g(v->device);
                const uint64_t sz = v->L->map->blobSize(nr);
                if(sz)
                    lam_cuda_check(cudaMemcpyAsync(v->blobs[nr], host, sz, cudaMemcpyHostToDevice,
                                                   static_cast<cudaStream_t>(stream)),
                                   "cudaMemcpyAsync(upload)");
            });
    }

    int lam_view_download(const lam_view* v, size_t nr, void* host, void* stream)
    {
        return guard(
            [&]
            {
                if(nr >= v->blobs.size())
                    throw std::out_of_range("index out of range: blob " + std::to_string(nr));
                DeviceGuard g(v->device);
                const uint64_t sz = v->L->map->blobSize(nr);
                if(sz)
                    lam_cuda_check(cudaMemcpyAsync(host, v->blobs[nr], sz, cudaMemcpyDeviceToHost,
                                                   static_cast<cudaStream_t>(stream)),
                                   "cudaMemcpyAsync(download)");
            });
    }

    // byte sub-range [offset, offset + nbytes) of one blob (View::blobs() spans, view.hpp:133-141)
    static void checkRange(const lam_view* v, size_t nr, uint64_t offset, uint64_t nbytes)
    {
        if(nr >= v->blobs.size())
            throw std::out_of_range("index out of range: blob " + std::to_string(nr));
        const uint64_t sz = v->L->map->blobSize(nr);
        if(offset > sz || nbytes > sz - offset)
            throw std::out_of_range("index out of range: bytes [" + std::to_string(offset) + ", "
                                    + std::to_string(offset + nbytes) + ") of blob " + std::to_string(nr)
                                    + " (size " + std::to_string(sz) + ")");
    }

    int lam_view_upload_range(lam_view* v, size_t nr, uint64_t offset, uint64_t nbytes, const void* host,
                              void* stream)
    {
        return guard(
            [&]
            {
                checkRange(v, nr, offset, nbytes);
                DeviceGuard g(v->device);
                if(nbytes)
                    lam_cuda_check(cudaMemcpyAsync(static_cast<char*>(v->blobs[nr]) + offset, host, nbytes,
                                                   cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)),
                                   "cudaMemcpyAsync(upload_range)");
            });
    }

    int lam_view_download_range(const lam_view* v, size_t nr, uint64_t offset, uint64_t nbytes, void* host,
                                void* stream)
    {
        return guard(
            [&]
            {
                checkRange(v, nr, offset, nbytes);
                DeviceGuard g(v->device);
                if(nbytes)
                    lam_cuda_check(cudaMemcpyAsync(host, static_cast<const char*>(v->blobs[nr]) + offset, nbytes,
                                                   cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)),
                                   "cudaMemcpyAsync(download_range)");
            });
    }

    // ---- view dump / restore (core/src/view_io.cpp:28-129) -------------------------------------
    // Same files as lamina::writeViewDump / readViewDump: <stem>.meta (key=value sidecar) and
    // <stem>.blob<nr>.bin (raw blob bytes), same error messages (std::runtime_error ->
    // LAM_ERUNTIME), so dumps move between the reference and this library in both directions.
    size_t lam_layout_dump_meta(const lam_layout* l, char* buf, size_t cap)
    {
        const Map& m = *l->L->map;
        std::string t = "schema=" + m.schema().toString() + "\nextents=" + m.extents().toString() + "\nextent-values=";
        const auto& dv = m.extents().dynamicValues();
        for(size_t i = 0; i < dv.size(); ++i)
            t += (i ? "," : "") + std::to_string(dv[i]);
        t += "\nmapping=" + m.name() + "\nblobs=" + std::to_string(m.blobCount()) + "\n";
        for(size_t nr = 0; nr < m.blobCount(); ++nr)
            t += "blob" + std::to_string(nr) + "-size=" + std::to_string(m.blobSize(nr)) + "\n";
        return copyOut(t, buf, cap);
    }

    int lam_view_dump(const lam_view* v, const char* stem)
    {
        return guard(
            [&]
            {
                if(!v || !stem)
                    throw std::invalid_argument("null argument");
                const std::string metaPath = std::string(stem) + ".meta";
                std::string meta(lam_layout_dump_meta(v->layout, nullptr, 0), '\0');
                lam_layout_dump_meta(v->layout, meta.data(), meta.size() + 1);
                {
                    std::ofstream out(metaPath);
                    if(!out)
                        throw std::runtime_error("cannot write " + metaPath);
                    out << meta;
                    out.close();
                    if(!out)
                        throw std::runtime_error("cannot write " + metaPath);
                }
                DeviceGuard g(v->device);
                // no stream argument (writeViewDump's signature): wait for every stream of the
                // device, non-blocking ones included, before reading the blobs back
                lam_cuda_check(cudaDeviceSynchronize(), "sync");
                const Map& m = *v->L->map;
                std::vector<char> host;
                for(size_t nr = 0; nr < m.blobCount(); ++nr)
                {
                    const std::string path = std::string(stem) + ".blob" + std::to_string(nr) + ".bin";
                    host.resize(m.blobSize(nr));
                    if(!host.empty())
                        lam_cuda_check(cudaMemcpy(host.data(), v->blobs[nr], host.size(), cudaMemcpyDeviceToHost),
                                       "cudaMemcpy(dump)");
                    std::ofstream out(path, std::ios::binary);
                    if(!out)
                        throw std::runtime_error("cannot write " + path);
                    out.write(host.data(), static_cast<std::streamsize>(host.size()));
                    out.close();
                    if(!out)
                        throw std::runtime_error("cannot write " + path);
                }
            });
    }

    int lam_view_restore(const char* stem, int device, void* stream, lam_layout** layoutOut, lam_view** viewOut)
    {
        lam_layout* lay = nullptr;
        lam_view* view = nullptr;
        const int rc = guard(
            [&]
            {
                if(!stem || !layoutOut || !viewOut)
                    throw std::invalid_argument("null argument");
                const std::string metaPath = std::string(stem) + ".meta";
                std::ifstream meta(metaPath);
                if(!meta)
                    throw std::runtime_error("cannot read " + metaPath);
                std::map<std::string, std::string> kv;
                std::string line;
                while(std::getline(meta, line))
                {
                    if(line.empty())
                        continue;
                    const size_t eq = line.find('=');
                    if(eq == std::string::npos)
                        throw std::runtime_error("malformed sidecar line: '" + line + "'");
                    kv[line.substr(0, eq)] = line.substr(eq + 1);
                }
                auto field = [&](const std::string& key) -> const std::string&
                {
                    const auto it = kv.find(key);
                    if(it == kv.end())
                        throw std::runtime_error("sidecar missing field '" + key + "'");
                    return it->second;
                };
                const std::string& schemaText = field("schema");
                std::vector<uint64_t> dyn;
                if(const std::string& vals = field("extent-values"); !vals.empty())
                {
                    size_t start = 0;
                    while(true)
                    {
                        const size_t comma = vals.find(',', start);
                        dyn.push_back(std::stoull(comma == std::string::npos ? vals.substr(start)
                                                                           : vals.substr(start, comma - start)));
                        if(comma == std::string::npos)
                            break;
                        start = comma + 1;
                    }
                }
                const std::string& extentsText = field("extents");
                const std::string& mappingText = field("mapping");
                const int rc1 = lam_layout_create(schemaText.c_str(), extentsText.c_str(), dyn.data(), dyn.size(),
                                                  mappingText.c_str(), 0, 1, &lay);
                if(rc1 != LAM_OK)
                    throw std::invalid_argument(g_lam_err);
                const Map& m = *lay->L->map;
                const size_t blobCount = std::stoull(field("blobs"));
                if(blobCount != m.blobCount())
                    throw std::runtime_error("blob count mismatch: sidecar says " + std::to_string(blobCount)
                                             + ", mapping declares " + std::to_string(m.blobCount()));
                std::vector<std::vector<char>> host(blobCount);
                for(size_t nr = 0; nr < blobCount; ++nr)
                {
                    const size_t declared = std::stoull(field("blob" + std::to_string(nr) + "-size"));
                    if(declared != m.blobSize(nr))
                        throw std::runtime_error("blob size mismatch: blob " + std::to_string(nr) + " sidecar says "
                                                 + std::to_string(declared) + ", mapping declares "
                                                 + std::to_string(m.blobSize(nr)));
                    const std::string path = std::string(stem) + ".blob" + std::to_string(nr) + ".bin";
                    std::ifstream in(path, std::ios::binary);
                    if(!in)
                        throw std::runtime_error("cannot read " + path);
                    host[nr].resize(declared);
                    in.read(host[nr].data(), static_cast<std::streamsize>(declared));
                    if(static_cast<size_t>(in.gcount()) != declared)
                        throw std::runtime_error("blob file truncated: " + path);
                }
                if(lam_view_alloc(lay, device, stream, &view) != LAM_OK)
                    throw CudaError(g_lam_err);
                for(size_t nr = 0; nr < blobCount; ++nr)
                    if(lam_view_upload(view, nr, host[nr].data(), stream) != LAM_OK)
                        throw CudaError(g_lam_err);
                DeviceGuard g(device);
                lam_cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "restore sync");
            });
        if(rc != LAM_OK)
        {
            const std::string err = g_lam_err;
            if(view)
                lam_view_free(view);
            if(lay)
                lam_layout_destroy(lay);
            g_lam_err = err;
            return rc;
        }
        *layoutOut = lay;
        *viewOut = view;
        return LAM_OK;
    }

    // ---- copy -----------------------------------------------------------------------------
    int lam_copy(const lam_view* src, lam_view* dst, void* stream)
    {
        return guard([&] { lamhost::copyViews(*src, *dst, 0, src->L->map->elementCount(), static_cast<cudaStream_t>(stream)); });
    }

    int lam_copy_range(const lam_view* src, lam_view* dst, uint64_t begin, uint64_t end, void* stream)
    {
        return guard([&] { lamhost::copyViews(*src, *dst, begin, end, static_cast<cudaStream_t>(stream)); });
    }

    int lam_copy_sharded(const lam_view* const* src, lam_view* const* dst, size_t n)
    {
        return guard(
            [&]
            {
                // one non-blocking stream per pair, all pairs in flight, then one join (each pair
                // on its own GPU: the weak-scaling layout of SURVEY 8(e) from a single process)
                std::vector<cudaStream_t> streams(n, nullptr);
                struct Cleanup
                {
                    std::vector<cudaStream_t>& s;
                    const lam_view* const* src;
                    ~Cleanup()
                    {
                        for(size_t k = 0; k < s.size(); ++k)
                            if(s[k])
                            {
                                cudaSetDevice(src[k]->device);
                                cudaStreamDestroy(s[k]);
                            }
                    }
                } cleanup{streams, src};
                for(size_t k = 0; k < n; ++k)
                {
                    DeviceGuard g(src[k]->device);
                    lam_cuda_check(cudaStreamCreateWithFlags(&streams[k], cudaStreamNonBlocking), "stream");
                    lamhost::copyViews(*src[k], *dst[k], 0, src[k]->L->map->elementCount(), streams[k]);
                }
                for(size_t k = 0; k < n; ++k)
                {
                    DeviceGuard g(src[k]->device);
                    lam_cuda_check(cudaStreamSynchronize(streams[k]), "sync");
                }
            });
    }

    int lam_copy_host(const lam_layout* sl, const void* const* sb, const lam_layout* dl, void* const* db, int device,
                      uint64_t* srcCounters, uint64_t* dstCounters)
    {
        return guard([&] { lamhost::copyHost(*sl, sb, *dl, db, device, srcCounters, dstCounters); });
    }

    // ---- counters ---------------------------------------------------------------------------
    int lam_counters_read(const lam_view* v, uint64_t* reads, uint64_t* writes)
    {
        return guard(
            [&]
            {
                const size_t L = v->L->roots.size();
                std::vector<uint64_t> c(2 * L, 0);
                if(v->L->fac && L)
                {
                    DeviceGuard g(v->device);
                    lam_cuda_check(cudaDeviceSynchronize(), "sync");
                    lam_cuda_check(cudaMemcpy(c.data(), v->img.facDev, 2 * L * 8, cudaMemcpyDeviceToHost),
                                   "cudaMemcpy(counters)");
                }
                if(reads)
                    std::memcpy(reads, c.data(), L * 8);
                if(writes)
                    std::memcpy(writes, c.data() + L, L * 8);
            });
    }

    int lam_counters_reset(lam_view* v, void* stream)
    {
        return guard(
            [&]
            {
                DeviceGuard g(v->device);
                auto s = static_cast<cudaStream_t>(stream);
                const size_t L = v->L->roots.size();
                if(v->L->fac && L)
                    lam_cuda_check(cudaMemsetAsync(v->img.facDev, 0, 2 * L * 8, s), "cudaMemsetAsync(counters)");
                if(v->L->heat && v->L->heatTotal)
                    lam_cuda_check(cudaMemsetAsync(v->img.heat, 0, v->L->heatTotal * 8, s), "cudaMemsetAsync(heatmap)");
            });
    }

    int lam_heatmap_read(const lam_view* v, size_t nr, uint64_t* out)
    {
        return guard(
            [&]
            {
                if(!v->L->heat)
                    throw std::invalid_argument("view has no heatmap");
                if(nr >= v->L->map->blobCount())
                    throw std::out_of_range("index out of range: blob " + std::to_string(nr));
                const uint64_t nb = (v->L->map->blobSize(nr) + v->L->heatGran - 1) / v->L->heatGran;
                if(!nb)
                    return;
                DeviceGuard g(v->device);
                lam_cuda_check(cudaDeviceSynchronize(), "sync");
                lam_cuda_check(cudaMemcpy(out, static_cast<uint64_t*>(v->img.heat) + v->L->heatOffset[nr], nb * 8,
                                          cudaMemcpyDeviceToHost),
                               "cudaMemcpy(heatmap)");
            });
    }

    // ---- funnel access -------------------------------------------------------------------------
    static void checkPairs(const lam_view* v, const uint64_t* lin, const uint32_t* leaf, size_t n)
    {
        const uint64_t N = v->L->map->elementCount();
        const size_t L = v->L->roots.size();
        for(size_t k = 0; k < n; ++k)
        {
            if(lin[k] >= N)
                throw std::out_of_range("index out of range: element " + std::to_string(lin[k]));
            if(leaf[k] >= L)
                throw std::out_of_range("index out of range: leaf " + std::to_string(leaf[k]));
        }
    }

    int lam_view_read_values(const lam_view* v, const uint64_t* lin, const uint32_t* leaf, uint64_t* out, size_t n,
                             void* stream)
    {
        return guard(
            [&]
            {
                checkPairs(v, lin, leaf, n);
                if(!n)
                    return;
                DeviceGuard g(v->device);
                auto s = static_cast<cudaStream_t>(stream);
                DevBuf<uint64_t> dl(n), dout(n);
                DevBuf<uint32_t> df(n);
                lam_cuda_check(cudaMemcpyAsync(dl.p, lin, n * 8, cudaMemcpyHostToDevice, s), "h2d");
                lam_cuda_check(cudaMemcpyAsync(df.p, leaf, n * 4, cudaMemcpyHostToDevice, s), "h2d");
                lam_cuda_check(lamk::read_values(v->img.hdr, dl.p, df.p, dout.p, n, s), "read_values");
                lam_cuda_check(cudaMemcpyAsync(out, dout.p, n * 8, cudaMemcpyDeviceToHost, s), "d2h");
                lam_cuda_check(cudaStreamSynchronize(s), "sync");
            });
    }

    int lam_view_write_values(lam_view* v, const uint64_t* lin, const uint32_t* leaf, const uint64_t* bits, size_t n,
                              void* stream)
    {
        return guard(
            [&]
            {
                checkPairs(v, lin, leaf, n);
                if(!n)
                    return;
                DeviceGuard g(v->device);
                auto s = static_cast<cudaStream_t>(stream);
                DevBuf<uint64_t> dl(n), din(n);
                DevBuf<uint32_t> df(n);
                lam_cuda_check(cudaMemcpyAsync(dl.p, lin, n * 8, cudaMemcpyHostToDevice, s), "h2d");
                lam_cuda_check(cudaMemcpyAsync(df.p, leaf, n * 4, cudaMemcpyHostToDevice, s), "h2d");
                lam_cuda_check(cudaMemcpyAsync(din.p, bits, n * 8, cudaMemcpyHostToDevice, s), "h2d");
                lam_cuda_check(lamk::write_values(v->img.hdr, dl.p, df.p, din.p, n, s), "write_values");
                lam_cuda_check(cudaStreamSynchronize(s), "sync");
            });
    }

    uint64_t lam_launch_count(void)
    {
        return lamk::launch_count();
    }

    int lam_device_sync(int device)
    {
        return guard(
            [&]
            {
                DeviceGuard g(device);
                lam_cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
            });
    }
}
