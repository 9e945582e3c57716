// copyView dispatch (view.cpp:168-189) and the host-buffer entry point.
#include "capi_internal.hpp"

#include <cstdio>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

using namespace lamb;

namespace lamhost
{
    static uint64_t gcd64(uint64_t a, uint64_t b)
    {
        while(b)
        {
            const uint64_t t = a % b;
            a = b;
            b = t;
        }
        return a;
    }

    static bool sameLayout(const Map& a, const Map& b)
    {
        // view.cpp:175-176
        return a.name() == b.name() && !a.hasMutableState() && !b.hasMutableState() && a.isFullyPhysical()
            && b.isFullyPhysical();
    }

    // Bit-packed <-> record-contiguous copies of 32-bit leaves that the one-pass kernels do not
    // take (k_rec_pack: AoS / AoSoA<L | 32> with one bit width; k_pack32: SoA / AoSoA<32k>) are
    // staged through an SoA multi-blob scratch view so both halves run on specialised kernels
    // (k_vec_transpose, k_pack32 / k_unpack32).  Every element is still read once from the source
    // view and written once to the destination view (counters unchanged).
    static bool hasBits(const Lowered& L)
    {
        for(const auto& st : L.streams)
            if(st.kind == LAMS_BITS)
                return true;
        return false;
    }

    static bool leafContig32(const Lowered& L)
    {
        // every leaf a 4-byte physical leaf in its own SoA array (what k_pack32 reads directly)
        for(uint16_t r : L.roots)
        {
            const lamp_node& nd = L.nodes[r];
            if(nd.kind != LAMP_PHYS || scalarSize(nd.type) != 4)
                return false;
            const lamp_stream& st = L.streams[nd.stream];
            if(!(st.lanes == 1 && st.block_stride == 4) && !(st.lanes % 32 == 0 && nd.b == 4))
                return false;
        }
        return true;
    }

    static bool all32(const Lowered& L)
    {
        for(const auto& l : L.map->schema().leaves())
            if(scalarSize(l.type) != 4)
                return false;
        return true;
    }

    // one record stream of 4-byte leaves (AoS packed, AoSoA<L> with L | 32, L < 32) against bit
    // streams of one width/format: k_rec_pack / k_rec_unpack do it in one pass (tryRecPack)
    static bool recordSide32(const Lowered& L)
    {
        const size_t nl = L.roots.size();
        if(nl < 2 || nl > 8)
            return false;
        const uint16_t s0 = L.nodes[L.roots[0]].stream;
        const lamp_stream& st = L.streams[s0];
        for(size_t f = 0; f < nl; ++f)
        {
            const lamp_node& nd = L.nodes[L.roots[f]];
            if(nd.kind != LAMP_PHYS || scalarSize(nd.type) != 4 || nd.stream != s0)
                return false;
            if(st.lanes == 1 ? (st.block_stride != nl * 4 || nd.a != f * 4)
                             : (st.lanes >= 32 || 32 % st.lanes || st.lane_shift == 0xFFFFFFFFu
                                || st.block_stride != st.lanes * nl * 4 || nd.a != f * 4 * st.lanes || nd.b != 4))
                return false;
        }
        return true;
    }

    static bool uniformBits(const Lowered& L)
    {
        const lamp_node& n0 = L.nodes[L.roots[0]];
        for(uint16_t r : L.roots)
        {
            const lamp_node& nd = L.nodes[r];
            if((nd.kind != LAMP_BITS_INT && nd.kind != LAMP_BITS_FLT) || nd.kind != n0.kind || nd.a != n0.a
               || nd.b != n0.b)
                return false;
        }
        return true;
    }

    static bool stagingHelps(const Lowered& S, const Lowered& D)
    {
        if(std::getenv("LAMB_STAGE") && std::getenv("LAMB_STAGE")[0] == '0')
            return false;
        if(!all32(S) || S.heat || D.heat)
            return false;
        const bool sb = hasBits(S), db = hasBits(D);
        if(!sb && !db)
            return false;
        // bit streams on both sides (different widths or formats, or the same computed layout):
        // k_repack32 when every leaf is one field of <= 32 bits (f32 formats E <= 8, M <= 23),
        // else unpack into the scratch and pack from it
        if(sb && db)
        {
            const char* rp = std::getenv("LAMB_REPACK");
            if(rp && rp[0] == '0')
                return true;
            for(const Lowered* L : {&S, &D})
                for(uint16_t r : L->roots)
                {
                    const lamp_node& nd = L->nodes[r];
                    const bool fast = (nd.a == 8 && nd.b == 10) || (nd.a == 5 && nd.b == 10) || (nd.a == 4 && nd.b == 3)
                        || (nd.a == 5 && nd.b == 2);
                    const bool fltOk = nd.kind == LAMP_BITS_FLT && nd.a >= 1 && nd.a <= 8 && nd.b <= 23 && (fast || (rp && rp[0] == '2'));
                    if(nd.kind == LAMP_BITS_INT ? nd.a > 32 : !fltOk)
                        return true;
                }
            return false;
        }
        const Lowered& phys = sb ? D : S; // the non-packed side
        for(uint16_t r : phys.roots)
            if(phys.nodes[r].kind != LAMP_PHYS)
                return true; // byte planes / ChangeType / Split against bits: both halves specialised
        if(recordSide32(phys) && uniformBits(sb ? S : D) && !(std::getenv("LAMB_RECPACK") && std::getenv("LAMB_RECPACK")[0] == '0'))
            return false;
        return !leafContig32(phys);
    }

    // Scratch SoA views for staged copies, cached per (device, schema+extents): allocation and
    // plan lowering happen once, not per copy (a 2^26-record scratch is 1.9 GB; at most 4 are
    // kept).  Users hold a shared_ptr, so an evicted scratch lives until its last user is done;
    // `use` serialises the enqueueing of the two staged copies, and `done` (recorded after
    // them) orders the next use on any stream after the previous one on the device.
    struct ScratchSoA
    {
        std::shared_ptr<Lowered> L;
        lam_view v;
        std::string key;
        std::mutex use;
        cudaEvent_t done = nullptr;
        ScratchSoA(const lam_view& like, std::string k) : key(std::move(k))
        {
            const Map& m = *like.L->map;
            L = lower(std::make_shared<SoAMap>(m.schema(), m.extents(), true));
            v.L = L;
            v.device = like.device;
            v.owned = false;
            DeviceGuard g(like.device);
            lam_cuda_check(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "scratch event");
            for(size_t nr = 0; nr < L->map->blobCount(); ++nr)
            {
                void* p = nullptr;
                lam_cuda_check(cudaMalloc(&p, std::max<uint64_t>(16, L->map->blobSize(nr))), "scratch blob");
                v.blobs.push_back(p);
            }
            v.img.build(*L, like.device, streamPtrsFor(*L, v.blobs));
        }
        ~ScratchSoA()
        {
            DeviceGuard g(v.device);
            if(done)
            {
                cudaEventSynchronize(done); // the last staged copy through this scratch
                cudaEventDestroy(done);
            }
            v.img.release();
            for(void* p : v.blobs)
                cudaFree(p);
        }
    };

    static std::shared_ptr<ScratchSoA> scratchFor(const lam_view& like)
    {
        static std::mutex mu;
        static std::vector<std::shared_ptr<ScratchSoA>> cache;
        const Map& m = *like.L->map;
        const std::string key = std::to_string(like.device) + "|" + m.schema().toString() + "|" + m.extents().toString();
        std::lock_guard<std::mutex> lk(mu);
        for(auto& c : cache)
            if(c->key == key)
                return c;
        if(cache.size() >= 4)
            cache.erase(cache.begin());
        cache.push_back(std::make_shared<ScratchSoA>(like, key));
        return cache.back();
    }

    void copyViews(const lam_view& src, lam_view& dst, uint64_t begin, uint64_t end, cudaStream_t s)
    {
        const Map& a = *src.L->map;
        const Map& b = *dst.L->map;
        if(!(a.schema() == b.schema()) || !(a.extents() == b.extents()))
            throw std::invalid_argument("incompatible views");
        if(src.device != dst.device)
            throw std::invalid_argument("views live on different devices");
        const uint64_t n = a.elementCount();
        if(begin > end || end > n)
            throw std::out_of_range("index out of range: elements [" + std::to_string(begin) + ", " + std::to_string(end) + ")");
        const bool full = begin == 0 && end == n;
        if(!full)
        {
            const uint64_t u1 = src.L->shardUnit, u2 = dst.L->shardUnit;
            const uint64_t unit = u1 / gcd64(u1, u2) * u2;
            if(begin % unit != 0 || (end != n && end % unit != 0))
                throw std::invalid_argument("copy range must start (and end, unless at the element count) on a "
                                            "multiple of the shard unit " + std::to_string(unit));
        }
        if(begin == end || a.schema().leafCount() == 0)
            return;
        DeviceGuard g(src.device);
        // LAMB_FORCE_TILE=1 (profiling only) routes equal layouts through the tile engine
        static const bool forceTile = std::getenv("LAMB_FORCE_TILE") && std::getenv("LAMB_FORCE_TILE")[0] == '1';
        if(full && sameLayout(a, b) && !forceTile)
        {
            std::vector<void*> dv(a.blobCount());
            std::vector<const void*> sv(a.blobCount());
            std::vector<uint64_t> bv(a.blobCount());
            for(size_t nr = 0; nr < a.blobCount(); ++nr)
            {
                dv[nr] = dst.blobs[nr];
                sv[nr] = src.blobs[nr];
                bv[nr] = a.blobSize(nr);
            }
            lam_cuda_check(lamk::blob_copy_multi(dv.data(), sv.data(), bv.data(), dv.size(), s), "blob_copy");
            return;
        }
        // LAMB_FORCE_GENERIC=1 (tests only): cross-check the specialised kernels against the
        // plan interpreter on identical inputs
        const char* fg = std::getenv("LAMB_FORCE_GENERIC");
        if(full && !(fg && fg[0] == '1') && stagingHelps(*src.L, *dst.L))
        {
            const std::shared_ptr<ScratchSoA> sc = scratchFor(src);
            std::lock_guard<std::mutex> lk(sc->use);
            lam_cuda_check(cudaStreamWaitEvent(s, sc->done, 0), "scratch wait");
            copyViews(src, sc->v, begin, end, s); // never staged again: the scratch side is plain SoA
            copyViews(sc->v, dst, begin, end, s);
            lam_cuda_check(cudaEventRecord(sc->done, s), "scratch record");
            return;
        }
        if(!(fg && fg[0] == '1') && tileCopy(src, dst, begin, end, s))
            return;
        if(std::getenv("LAMB_TRACE") && std::getenv("LAMB_TRACE")[0] == '1')
            std::fprintf(stderr, "lamb path: generic\n");
        lam_cuda_check(lamk::generic_copy(src.img.hdr, dst.img.hdr, begin, end,
                                          static_cast<uint32_t>(a.schema().leafCount()), src.L->fac, dst.L->fac, s),
                       "generic_copy");
    }

    void copyHost(const lam_layout& sl, const void* const* sb, const lam_layout& dl, void* const* db, int device,
                  uint64_t* srcCounters, uint64_t* dstCounters)
    {
        const Map& a = *sl.L->map;
        const Map& b = *dl.L->map;
        if(!(a.schema() == b.schema()) || !(a.extents() == b.extents()))
            throw std::invalid_argument("incompatible views");
        DeviceGuard g(device);
        HostPipeline& hp = HostPipeline::get(device);
        hp.run(sl, sb, dl, db, srcCounters, dstCounters);
    }
} // namespace lamhost
