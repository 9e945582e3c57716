// lam_copy_host: copyView over HOST views, streamed through the GPU in element chunks.
//
//   h2d stream :  src stream regions of chunk k (+ dst regions that hold bytes the copy
//                 never writes: padding, AoSoA tail lanes, the bit-stream tail word)
//   comp stream:  chunk-view stream pointers -> tile / generic copy kernel over [a, e)
//   d2h stream :  dst stream regions of chunk k back to the host blobs
// with kSlots rotating device slots, so H2D(k+1), copy(k) and D2H(k-1) overlap and
// PCIe runs full duplex.  A chunk starts on a multiple of both layouts' shard unit,
// hence every stream region starts on a fresh AoSoA block / bit-stream word and is
// 16-byte aligned; chunk views address the slot through "virtual" stream pointers
// (slot address minus the region's blob offset), so kernels keep global indices —
// heatmap blocks and counters stay exact.
#include "capi_internal.hpp"

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

using namespace lamb;

namespace lamhost
{
    namespace
    {
        std::mutex g_mu;
        std::map<int, HostPipeline*> g_pipes;

        uint64_t gcd64(uint64_t a, uint64_t b)
        {
            while(b)
            {
                const uint64_t t = a % b;
                a = b;
                b = t;
            }
            return a;
        }

        struct Region
        {
            uint64_t lo = 0, hi = 0; // blob byte range
        };

        Region regionOf(const lamp_stream& st, uint64_t a, uint64_t e, uint64_t blobSize)
        {
            Region r;
            if(st.kind == LAMS_BITS)
            {
                const uint64_t b = st.block_stride;
                r.lo = (a * b / 32) * 4;
                r.hi = ((e * b + 31) / 32) * 4;
            }
            else
            {
                r.lo = st.base0 + (a / st.lanes) * st.block_stride;
                r.hi = st.base0 + ((e + st.lanes - 1) / st.lanes) * st.block_stride;
            }
            if(r.hi > blobSize)
                r.hi = blobSize;
            if(r.lo > r.hi)
                r.lo = r.hi;
            return r;
        }

        uint64_t maxRegion(const lamp_stream& st, uint64_t C)
        {
            if(st.kind == LAMS_BITS)
                return (C * st.block_stride + 31) / 32 * 4 + 16;
            return (C / st.lanes + 2) * st.block_stride + 16;
        }

        bool sameLayout(const Map& a, const Map& b)
        {
            return a.name() == b.name() && !a.hasMutableState() && !b.hasMutableState() && a.isFullyPhysical()
                && b.isFullyPhysical();
        }

        // bytes of src+dst per chunk (LAMB_PIPE_MB overrides, for link experiments)
        // copy queues per direction (LAMB_PIPE_CE=2: stream regions alternate over two
        // queues, so consecutive DMA transfers overlap their start-up)
        int copyQueues()
        {
            static const int v = []
            {
                const char* e = getenv("LAMB_PIPE_CE");
                return e && atoi(e) == 2 ? 2 : 1;
            }();
            return v;
        }

        // bytes of the last chunk's region that the copy does not write (partial AoSoA block,
        // partial final bit-stream word): only then must the host's bytes be pre-uploaded
        bool tailHole(const lamp_stream& st, uint64_t n)
        {
            if(st.kind == LAMS_BITS)
                return (n * st.block_stride) % 32 != 0;
            return st.lanes > 1 && n % st.lanes != 0;
        }

        uint64_t slotTarget()
        {
            static const uint64_t v = []
            {
                const char* e = getenv("LAMB_PIPE_MB");
                const long mb = e ? atol(e) : 0;
                return mb > 0 ? static_cast<uint64_t>(mb) << 20 : uint64_t{192} << 20;
            }();
            return v;
        }
    } // namespace

    HostPipeline& HostPipeline::get(int device)
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_pipes.find(device);
        if(it == g_pipes.end())
            it = g_pipes.emplace(device, new HostPipeline(device)).first;
        return *it->second;
    }

    HostPipeline::HostPipeline(int device) : device_(device)
    {
        lam_cuda_check(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking), "stream");
        lam_cuda_check(cudaStreamCreateWithFlags(&comp_, cudaStreamNonBlocking), "stream");
        lam_cuda_check(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking), "stream");
        lam_cuda_check(cudaStreamCreateWithFlags(&h2dB_, cudaStreamNonBlocking), "stream");
        lam_cuda_check(cudaStreamCreateWithFlags(&d2hB_, cudaStreamNonBlocking), "stream");
        for(int k = 0; k < kSlots; ++k)
        {
            lam_cuda_check(cudaEventCreateWithFlags(&evIn_[k], cudaEventDisableTiming), "event");
            lam_cuda_check(cudaEventCreateWithFlags(&evDone_[k], cudaEventDisableTiming), "event");
            lam_cuda_check(cudaEventCreateWithFlags(&evFree_[k], cudaEventDisableTiming), "event");
            lam_cuda_check(cudaEventCreateWithFlags(&evInB_[k], cudaEventDisableTiming), "event");
            lam_cuda_check(cudaEventCreateWithFlags(&evFreeB_[k], cudaEventDisableTiming), "event");
        }
    }

    HostPipeline::~HostPipeline() = default; // process-lifetime singleton

    HostPipeline::Images& HostPipeline::images(const std::shared_ptr<Lowered>& S, const std::shared_ptr<Lowered>& D)
    {
        for(auto& c : cache_)
            if(c->S == S && c->D == D)
                return *c;
        if(cache_.size() >= 64)
        {
            lam_cuda_check(cudaDeviceSynchronize(), "sync");
            for(auto& c : cache_)
            {
                if(c->sheat)
                    cudaFree(c->sheat);
                if(c->dheat)
                    cudaFree(c->dheat);
            }
            cache_.clear();
        }
        auto im = std::make_unique<Images>();
        im->S = S;
        im->D = D;
        if(S->heat && S->heatTotal)
            lam_cuda_check(cudaMalloc(&im->sheat, S->heatTotal * 8), "cudaMalloc(heat)");
        if(D->heat && D->heatTotal)
            lam_cuda_check(cudaMalloc(&im->dheat, D->heatTotal * 8), "cudaMalloc(heat)");
        std::vector<uint8_t*> zeroS(S->streams.size(), nullptr), zeroD(D->streams.size(), nullptr);
        for(int k = 0; k < kSlots; ++k)
        {
            im->simg[k] = std::make_unique<DeviceImage>();
            im->dimg[k] = std::make_unique<DeviceImage>();
            im->simg[k]->build(*S, device_, zeroS, im->sheat);
            im->dimg[k]->build(*D, device_, zeroD, im->dheat);
        }
        cache_.push_back(std::move(im));
        return *cache_.back();
    }

    void HostPipeline::ensure(size_t bytes)
    {
        if(bytes <= slotBytes_)
            return;
        lam_cuda_check(cudaDeviceSynchronize(), "sync");
        for(auto& p : slot_)
        {
            if(p)
                cudaFree(p);
            p = nullptr;
        }
        for(auto& p : slot_)
            lam_cuda_check(cudaMalloc(&p, bytes), "cudaMalloc(pipeline slot)");
        slotBytes_ = bytes;
    }

    void HostPipeline::run(const lam_layout& sl, const void* const* sb, const lam_layout& dl, void* const* db,
                           uint64_t* srcCounters, uint64_t* dstCounters)
    {
        std::lock_guard<std::mutex> lk(g_mu);
        const Lowered& S = *sl.L;
        const Lowered& D = *dl.L;
        const Map& a = *S.map;
        const Map& b = *D.map;
        const uint64_t n = a.elementCount();
        const size_t leaves = a.schema().leafCount();

        // ---- copyView fast path: blob bytes streamed through the device blob copy ----------
        if(sameLayout(a, b))
        {
            const uint64_t cb = (slotTarget() / 2) & ~uint64_t{15};
            ensure(2 * cb);
            int k = 0;
            for(size_t nr = 0; nr < a.blobCount(); ++nr)
                for(uint64_t off = 0; off < a.blobSize(nr); off += cb, ++k)
                {
                    const int s = k % kSlots;
                    const uint64_t len = std::min(cb, a.blobSize(nr) - off);
                    uint8_t* in = static_cast<uint8_t*>(slot_[s]);
                    uint8_t* out = in + cb;
                    lam_cuda_check(cudaStreamWaitEvent(h2d_, evFree_[s], 0), "wait");
                    lam_cuda_check(cudaMemcpyAsync(in, static_cast<const uint8_t*>(sb[nr]) + off, len,
                                                   cudaMemcpyHostToDevice, h2d_), "h2d");
                    lam_cuda_check(cudaEventRecord(evIn_[s], h2d_), "record");
                    lam_cuda_check(cudaStreamWaitEvent(comp_, evIn_[s], 0), "wait");
                    lam_cuda_check(lamk::blob_copy(out, in, len, comp_), "blob_copy");
                    lam_cuda_check(cudaEventRecord(evDone_[s], comp_), "record");
                    lam_cuda_check(cudaStreamWaitEvent(d2h_, evDone_[s], 0), "wait");
                    lam_cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(db[nr]) + off, out, len,
                                                   cudaMemcpyDeviceToHost, d2h_), "d2h");
                    lam_cuda_check(cudaEventRecord(evFree_[s], d2h_), "record");
                }
            lam_cuda_check(cudaStreamSynchronize(d2h_), "sync");
            if(srcCounters && S.fac)
                std::memset(srcCounters, 0, 2 * leaves * 8);
            if(dstCounters && D.fac)
                std::memset(dstCounters, 0, 2 * leaves * 8);
            return;
        }
        if(n == 0 || leaves == 0)
            return;

        // ---- chunking ---------------------------------------------------------------------
        const uint64_t unit = S.shardUnit / gcd64(S.shardUnit, D.shardUnit) * D.shardUnit;
        double bpe = 0;
        for(const auto& st : S.streams)
            bpe += st.kind == LAMS_BITS ? st.block_stride / 8.0 : double(st.block_stride) / st.lanes;
        for(const auto& st : D.streams)
            bpe += st.kind == LAMS_BITS ? st.block_stride / 8.0 : double(st.block_stride) / st.lanes;
        uint64_t C = bpe > 0 ? static_cast<uint64_t>(slotTarget() / bpe) : n;
        // chunk boundaries on a multiple of 4096 elements too (when that keeps >= 2 chunks): every
        // stream region then starts on a host page boundary, which the DMA engines need
        // to run at full link rate
        {
            const char* e = getenv("LAMB_PIPE_PAGEALIGN");
            const uint64_t pageUnit = unit / gcd64(unit, 4096) * 4096;
            if((!e || atoi(e) != 0) && C >= 2 * pageUnit)
                C = C / pageUnit * pageUnit;
        }
        C = std::max<uint64_t>(unit, C / unit * unit);
        if(C > n)
            C = (n + unit - 1) / unit * unit;

        // fixed per-stream offsets inside a slot
        std::vector<uint64_t> soff(S.streams.size()), doff(D.streams.size());
        uint64_t used = 0;
        for(size_t s = 0; s < S.streams.size(); ++s)
        {
            soff[s] = used;
            used += (maxRegion(S.streams[s], C) + 15) & ~uint64_t{15};
        }
        for(size_t s = 0; s < D.streams.size(); ++s)
        {
            doff[s] = used;
            used += (maxRegion(D.streams[s], C) + 15) & ~uint64_t{15};
        }
        ensure(used);

        // per-slot chunk-view images (cached per layout pair) sharing one heatmap per side
        Images& im = images(sl.L, dl.L);
        void* sheat = im.sheat;
        void* dheat = im.dheat;
        lam_cuda_check(cudaStreamSynchronize(comp_), "sync");
        if(sheat)
            lam_cuda_check(cudaMemsetAsync(sheat, 0, S.heatTotal * 8, comp_), "memset");
        if(dheat)
            lam_cuda_check(cudaMemsetAsync(dheat, 0, D.heatTotal * 8, comp_), "memset");
        DeviceImage* simg[kSlots];
        DeviceImage* dimg[kSlots];
        for(int k = 0; k < kSlots; ++k)
        {
            simg[k] = im.simg[k].get();
            dimg[k] = im.dimg[k].get();
            if(S.fac)
                lam_cuda_check(cudaMemsetAsync(simg[k]->facDev, 0, 2 * leaves * 8, comp_), "memset");
            if(D.fac)
                lam_cuda_check(cudaMemsetAsync(dimg[k]->facDev, 0, 2 * leaves * 8, comp_), "memset");
        }
        const size_t ptrBytes = (S.streams.size() + D.streams.size()) * sizeof(uint8_t*);
        const size_t tabBytes = std::max<size_t>(ptrBytes, 8) * kSlots;
        if(tabBytes > pinnedBytes_)
        {
            if(pinnedPtrs_)
                cudaFreeHost(pinnedPtrs_);
            lam_cuda_check(cudaMallocHost(&pinnedPtrs_, tabBytes), "cudaMallocHost");
            pinnedBytes_ = tabBytes;
        }
        void* ptab = pinnedPtrs_;

        const uint64_t nchunks = (n + C - 1) / C;
        for(uint64_t k = 0; k < nchunks; ++k)
        {
            const int s = static_cast<int>(k % kSlots);
            const uint64_t lo = k * C, hi = std::min(n, lo + C);
            const bool last = k + 1 == nchunks;
            if(k >= static_cast<uint64_t>(kSlots))
                lam_cuda_check(cudaEventSynchronize(evFree_[s]), "sync slot");
            uint8_t* slot = static_cast<uint8_t*>(slot_[s]);
            auto* tab = reinterpret_cast<uint8_t**>(static_cast<uint8_t*>(ptab) + s * std::max<size_t>(ptrBytes, 8));

            const int nq = copyQueues();
            cudaStream_t hq[2] = {h2d_, h2dB_};
            int qi = 0;
            lam_cuda_check(cudaStreamWaitEvent(h2d_, evFree_[s], 0), "wait");
            if(nq == 2)
                lam_cuda_check(cudaStreamWaitEvent(h2dB_, evFree_[s], 0), "wait");
            auto up = [&](void* dev, const void* host, uint64_t bytes)
            {
                lam_cuda_check(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, hq[qi]), "h2d");
                qi = (qi + 1) % nq;
            };
            for(size_t t = 0; t < S.streams.size(); ++t)
            {
                const auto& st = S.streams[t];
                const Region r = regionOf(st, lo, hi, a.blobSize(st.nr));
                uint8_t* dev = slot + soff[t] + (r.lo & 15);
                tab[t] = dev - (r.lo - st.base0);
                if(r.hi > r.lo)
                    up(dev, static_cast<const uint8_t*>(sb[st.nr]) + r.lo, r.hi - r.lo);
            }
            for(size_t t = 0; t < D.streams.size(); ++t)
            {
                const auto& st = D.streams[t];
                const Region r = regionOf(st, lo, hi, b.blobSize(st.nr));
                uint8_t* dev = slot + doff[t] + (r.lo & 15);
                tab[S.streams.size() + t] = dev - (r.lo - st.base0);
                if((!st.holefree || (last && tailHole(st, n))) && r.hi > r.lo)
                    up(dev, static_cast<const uint8_t*>(db[st.nr]) + r.lo, r.hi - r.lo);
            }
            // the chunk views' stream-pointer tables ride on the h2d stream too: a small copy
            // queued on the compute stream would wait behind the next chunk's bulk H2D on the
            // copy engine and serialise the pipeline
            if(!S.streams.empty())
                lam_cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(simg[s]->mem) + simg[s]->offPtrs, tab,
                                               S.streams.size() * sizeof(uint8_t*), cudaMemcpyHostToDevice, h2d_),
                               "ptr table");
            if(!D.streams.empty())
                lam_cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(dimg[s]->mem) + dimg[s]->offPtrs,
                                               tab + S.streams.size(), D.streams.size() * sizeof(uint8_t*),
                                               cudaMemcpyHostToDevice, h2d_),
                               "ptr table");
            if(nq == 2)
            {
                lam_cuda_check(cudaEventRecord(evInB_[s], h2dB_), "record");
                lam_cuda_check(cudaStreamWaitEvent(h2d_, evInB_[s], 0), "wait");
            }
            lam_cuda_check(cudaEventRecord(evIn_[s], h2d_), "record");

            lam_cuda_check(cudaStreamWaitEvent(comp_, evIn_[s], 0), "wait");
            if(!tileCopyPtrs(S, *simg[s], tab, D, *dimg[s], tab + S.streams.size(), lo, hi, comp_))
                lam_cuda_check(lamk::generic_copy(simg[s]->hdr, dimg[s]->hdr, lo, hi, static_cast<uint32_t>(leaves),
                                                  S.fac, D.fac, comp_),
                               "generic_copy");
            lam_cuda_check(cudaEventRecord(evDone_[s], comp_), "record");

            cudaStream_t dq[2] = {d2h_, d2hB_};
            lam_cuda_check(cudaStreamWaitEvent(d2h_, evDone_[s], 0), "wait");
            if(nq == 2)
                lam_cuda_check(cudaStreamWaitEvent(d2hB_, evDone_[s], 0), "wait");
            qi = 0;
            for(size_t t = 0; t < D.streams.size(); ++t)
            {
                const auto& st = D.streams[t];
                const Region r = regionOf(st, lo, hi, b.blobSize(st.nr));
                if(r.hi > r.lo)
                {
                    lam_cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(db[st.nr]) + r.lo, slot + doff[t] + (r.lo & 15),
                                                   r.hi - r.lo, cudaMemcpyDeviceToHost, dq[qi]), "d2h");
                    qi = (qi + 1) % nq;
                }
            }
            if(nq == 2)
            {
                lam_cuda_check(cudaEventRecord(evFreeB_[s], d2hB_), "record");
                lam_cuda_check(cudaStreamWaitEvent(d2h_, evFreeB_[s], 0), "wait");
            }
            lam_cuda_check(cudaEventRecord(evFree_[s], d2h_), "record");
        }
        lam_cuda_check(cudaStreamSynchronize(d2h_), "sync");
        lam_cuda_check(cudaStreamSynchronize(comp_), "sync");

        // counters: FieldAccessCount summed over slots, then the heatmap blocks
        auto gather = [&](const Lowered& L, DeviceImage* const* imgs, void* heat, uint64_t* out)
        {
            if(!out)
                return;
            size_t pos = 0;
            if(L.fac)
            {
                std::vector<uint64_t> sum(2 * leaves, 0), part(2 * leaves);
                for(int k = 0; k < kSlots; ++k)
                {
                    lam_cuda_check(cudaMemcpy(part.data(), imgs[k]->facDev, 2 * leaves * 8, cudaMemcpyDeviceToHost),
                                   "counters");
                    for(size_t j = 0; j < 2 * leaves; ++j)
                        sum[j] += part[j];
                }
                std::memcpy(out, sum.data(), 2 * leaves * 8);
                pos = 2 * leaves;
            }
            if(L.heat && L.heatTotal)
                lam_cuda_check(cudaMemcpy(out + pos, heat, L.heatTotal * 8, cudaMemcpyDeviceToHost), "heatmap");
        };
        gather(S, simg, sheat, srcCounters);
        gather(D, dimg, dheat, dstCounters);
    }
} // namespace lamhost
