// Generic fieldwise copy: the reference hot loop
//     for i in [0,N) for f in [0,leaves): dst.write(i, f, src.read(i, f))   (view.cpp:184-188)
// with one thread per element i and the mapping trees resolved by the device plan
// interpreter (device_common.cuh).  Handles every mapping composition the layout grammar
// can express (Split, One, Null, nested ChangeType/Bytesplit, bit packing, instrumentation);
// the specialised kernels (copy_tile_host.cpp dispatch) take every shape they can express.  Bit-stream
// writes use word atomics, so neighbouring fields never race (bitpack.hpp:16-17).
#include "device_common.cuh"
#include "launch.h"

#include <cstdlib>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <utility>

namespace lamk
{
    static std::atomic<uint64_t> g_launches{0};
    void count_launch(uint64_t n)
    {
        g_launches.fetch_add(n, std::memory_order_relaxed);
    }
    uint64_t launch_count()
    {
        return g_launches.load(std::memory_order_relaxed);
    }

    cudaError_t opt_in_smem(const void* func, size_t smem)
    {
        // set even below 48 KB: a kernel with static shared memory needs the attribute once
        // static + dynamic passes 48 KB
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if(e != cudaSuccess)
            return e;
        static std::mutex mu;
        static std::map<std::pair<const void*, int>, size_t> done; // (kernel, device) -> bytes set
        std::lock_guard<std::mutex> g(mu);
        size_t& have = done[{func, dev}];
        if(have >= smem && have != 0)
            return cudaSuccess;
        e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if(e == cudaSuccess)
            have = smem;
        return e;
    }

    int sm_count(int device)
    {
        static int cache[64] = {0};
        if(device < 0 || device >= 64)
            return 148;
        if(cache[device] == 0)
        {
            int v = 0;
            if(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0)
                v = 148;
            cache[device] = v;
        }
        return cache[device];
    }

    // FieldAccessCount: warp-aggregated per-field shared counters, one global atomic per
    // CTA per field (instrument.cpp:57-72 counts one relaxed increment per access)
    template<typename Idx>
    __global__ void __launch_bounds__(256) k_generic_copy(const lamp_view* __restrict__ S, const lamp_view* __restrict__ D,
                                                           uint64_t begin, uint64_t end, uint32_t nleaves, int facS, int facD,
                                                           int countHeat)
    {
        extern __shared__ unsigned long long s_cnt[]; // [nleaves] reads, [nleaves] writes
        lamd::ViewCtx sv = lamd::make_ctx(S);
        lamd::ViewCtx dv = lamd::make_ctx(D);
        if(!countHeat)
        {
            sv.heat = nullptr;
            dv.heat = nullptr;
        }
        const uint16_t* sroots = S->roots;
        const uint16_t* droots = D->roots;
        if(facS | facD)
        {
            for(uint32_t k = threadIdx.x; k < 2 * nleaves; k += blockDim.x)
                s_cnt[k] = 0;
            __syncthreads();
        }
        const Idx stride = static_cast<Idx>(gridDim.x) * blockDim.x;
        const Idx n = static_cast<Idx>(end - begin);
        uint32_t mine = 0;
        for(Idx k = static_cast<Idx>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride)
        {
            const uint64_t i = begin + k;
            for(uint32_t f = 0; f < nleaves; ++f)
            {
                const uint64_t v = lamd::read_node<LAMP_MAX_DEPTH>(sv, sroots[f], i);
                lamd::write_node<LAMP_MAX_DEPTH>(dv, droots[f], i, v);
            }
            ++mine;
        }
        if(facS | facD)
        {
            const uint32_t warpTotal = __reduce_add_sync(0xFFFFFFFFu, mine);
            if((threadIdx.x & 31) == 0 && warpTotal)
                for(uint32_t f = 0; f < nleaves; ++f)
                {
                    if(facS)
                        atomicAdd(&s_cnt[f], static_cast<unsigned long long>(warpTotal));
                    if(facD)
                        atomicAdd(&s_cnt[nleaves + f], static_cast<unsigned long long>(warpTotal));
                }
            __syncthreads();
            for(uint32_t f = threadIdx.x; f < nleaves; f += blockDim.x)
            {
                if(facS && s_cnt[f])
                    atomicAdd(&S->fac_counters[f], s_cnt[f]); // src reads
                if(facD && s_cnt[nleaves + f])
                    atomicAdd(&D->fac_counters[nleaves + f], s_cnt[nleaves + f]); // dst writes
            }
        }
    }

    cudaError_t generic_copy(const lamp_view* src, const lamp_view* dst, uint64_t begin, uint64_t end,
                             uint32_t nleaves, bool facSrc, bool facDst, cudaStream_t s, bool countHeat)
    {
        if(end <= begin || nleaves == 0)
            return cudaSuccess;
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t n = end - begin;
        const uint64_t want = (n + 255) / 256;
        const uint64_t cap = static_cast<uint64_t>(sm_count(dev)) * 8;
        const unsigned grid = static_cast<unsigned>(want < cap ? want : cap);
        const size_t smem = (facSrc || facDst) ? 2 * nleaves * sizeof(unsigned long long) : 0;
        if(end <= 0x7FFFFFFFull)
            k_generic_copy<uint32_t><<<grid, 256, smem, s>>>(src, dst, begin, end, nleaves, facSrc, facDst, countHeat);
        else
            k_generic_copy<uint64_t><<<grid, 256, smem, s>>>(src, dst, begin, end, nleaves, facSrc, facDst, countHeat);
        count_launch();
        return cudaGetLastError();
    }

    // ---- blob copy: vectorised 16-byte path when both sides are aligned ----------------
    // U 16-byte loads per thread are in flight before the first store; consecutive threads
    // touch consecutive 16-byte words, so each warp instruction moves 512 contiguous bytes.
    template<int U>
    __global__ void __launch_bounds__(256) k_blob_copy16(uint4* __restrict__ d, const uint4* __restrict__ s, uint64_t n16)
    {
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        for(; i + (U - 1) * stride < n16; i += U * stride)
        {
            uint4 x[U];
#pragma unroll
            for(int k = 0; k < U; ++k)
                x[k] = __ldcs(s + i + k * stride);
#pragma unroll
            for(int k = 0; k < U; ++k)
                __stcs(d + i + k * stride, x[k]);
        }
        for(; i < n16; i += stride)
            __stcs(d + i, __ldcs(s + i));
    }

    // several blobs in one launch (blockIdx.y = blob): the same-layout copy of a multi-blob
    // mapping (SoA multi-blob: 7 blobs) without a launch gap and a tail per blob
    struct BlobSegs
    {
        uint4* d[16];
        const uint4* s[16];
        uint64_t n16[16];
    };
    template<int U>
    __global__ void __launch_bounds__(256) k_blob_copy16_multi(const __grid_constant__ BlobSegs p)
    {
        uint4* __restrict__ d = p.d[blockIdx.y];
        const uint4* __restrict__ s = p.s[blockIdx.y];
        const uint64_t n16 = p.n16[blockIdx.y];
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        for(; i + (U - 1) * stride < n16; i += U * stride)
        {
            uint4 x[U];
#pragma unroll
            for(int k = 0; k < U; ++k)
                x[k] = __ldcs(s + i + k * stride);
#pragma unroll
            for(int k = 0; k < U; ++k)
                __stcs(d + i + k * stride, x[k]);
        }
        for(; i < n16; i += stride)
            __stcs(d + i, __ldcs(s + i));
    }

    __global__ void k_blob_copy1(uint8_t* __restrict__ d, const uint8_t* __restrict__ s, uint64_t n)
    {
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        for(uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
            d[i] = s[i];
    }

    // Heatmap accounting of copyView over [begin, end): every element touches every leaf's
    // access ranges once (view.cpp:186-188 through Heatmap::read/write, instrument.cpp:163-176)
    __global__ void __launch_bounds__(256) k_heat_account(const lamp_view* __restrict__ V, uint64_t begin, uint64_t end,
                                                         uint32_t nleaves)
    {
        const lamd::ViewCtx c = lamd::make_ctx(V);
        for(uint64_t i = begin + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < end;
            i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
            for(uint32_t f = 0; f < nleaves; ++f)
                lamd::touch_node<LAMP_MAX_DEPTH>(c, V->roots[f], i);
    }

    cudaError_t heat_account(const lamp_view* v, uint64_t begin, uint64_t end, uint32_t nleaves, cudaStream_t s)
    {
        if(end <= begin)
            return cudaSuccess;
        const unsigned grid = stream_grid((end - begin + 255) / 256, "LAMB_HEAT_CTAS", 16);
        k_heat_account<<<grid, 256, 0, s>>>(v, begin, end, nleaves);
        count_launch();
        return cudaGetLastError();
    }

    // ---- Heatmap accounting over physical terminals, blocks owned per CTA ---------------------
    // Every terminal of the heat side is a physical byte range (PHYS leaves, ChangeType over
    // PHYS, byte splits): a CTA takes E consecutive elements, histograms the touched blocks of
    // one stream at a time in shared memory, then adds its counts to the global counters with
    // a plain read-modify-write for the blocks only it can touch (interior of its byte span)
    // and an atomic for the two edge blocks it may share with its neighbours.
    __global__ void __launch_bounds__(256) k_heat_phys(const __grid_constant__ HeatParams p)
    {
        extern __shared__ unsigned long long hist[];
        const uint64_t cb = p.begin + static_cast<uint64_t>(blockIdx.x) * p.E;
        const uint64_t ce = cb + p.E < p.end ? cb + p.E : p.end;
        for(uint32_t si = 0; si < p.nstreams; ++si)
        {
            const HeatStream& st = p.st[si];
            const uint64_t lo = st.base0 + (cb / st.lanes) * st.bs;
            const uint64_t hi = st.base0 + ((ce + st.lanes - 1) / st.lanes) * st.bs;
            const uint64_t b0 = lo / p.gran, b1 = (hi - 1) / p.gran;
            const uint32_t W = static_cast<uint32_t>(b1 - b0 + 1);
            for(uint32_t w = threadIdx.x; w < W; w += blockDim.x)
                hist[w] = 0;
            __syncthreads();
            // each thread walks a contiguous run of elements: block indices mostly repeat, so
            // touches are run-length combined before the shared-memory atomic
            const uint64_t per = (ce - cb + blockDim.x - 1) / blockDim.x;
            const uint64_t eb = cb + threadIdx.x * per, ee = eb + per < ce ? eb + per : ce;
            uint64_t cur = ~0ull;
            unsigned long long run = 0;
            for(uint64_t e = eb; e < ee; ++e)
            {
                uint64_t blk, lane;
                if(st.lanes == 1)
                {
                    blk = e;
                    lane = 0;
                }
                else if(st.lshift != 0xFFFFFFFFu)
                {
                    blk = e >> st.lshift;
                    lane = e & (st.lanes - 1);
                }
                else
                {
                    blk = e / st.lanes;
                    lane = e - blk * st.lanes;
                }
                for(uint32_t t = st.t0; t < st.t1; ++t)
                {
                    const HeatTerm& ht = p.term[t];
                    const uint64_t a = st.base0 + blk * st.bs + ht.inblock + lane * ht.ls;
                    const uint64_t f = p.gshift < 64 ? a >> p.gshift : a / p.gran;
                    const uint64_t l = p.gshift < 64 ? (a + ht.size - 1) >> p.gshift : (a + ht.size - 1) / p.gran;
                    for(uint64_t b = f; b <= l; ++b)
                    {
                        if(b == cur)
                            ++run;
                        else
                        {
                            if(run)
                                atomicAdd(&hist[cur - b0], run);
                            cur = b;
                            run = 1;
                        }
                    }
                }
            }
            if(run)
                atomicAdd(&hist[cur - b0], run);
            __syncthreads();
            unsigned long long* heat = p.heat + p.heatOff[st.nr];
            for(uint32_t w = threadIdx.x; w < W; w += blockDim.x)
            {
                const unsigned long long c = hist[w];
                if(!c)
                    continue;
                if(w == 0 || w == W - 1)
                    atomicAdd(heat + b0 + w, c);
                else
                    heat[b0 + w] += c;
            }
            __syncthreads();
        }
    }

    // Closed form for streams with one element per block stride (AoS, SoA, byte planes): heat
    // block b of stream y receives, for each term, the number of elements e in [begin, end) whose
    // range [base0 + e*bs + inblock, +size) overlaps [b*g, (b+1)*g).  One thread per block; a
    // stream's interior blocks are touched by no other stream, its two edge blocks may be.
    __device__ __forceinline__ int64_t floor_div(int64_t a, int64_t b)
    {
        return a >= 0 ? a / b : -((-a + b - 1) / b);
    }

    // floor(a / b) for b > 0 without the 64-bit division subroutine: a double-precision quotient
    // estimate (|a| < 2^53, so it is off by at most one) corrected with one integer multiply
    __device__ __forceinline__ int64_t floor_div_r(int64_t a, int64_t b, double invb)
    {
        int64_t q = static_cast<int64_t>(floor(static_cast<double>(a) * invb));
        const int64_t r = a - q * b;
        q += r < 0 ? -1 : (r >= b ? 1 : 0);
        return q;
    }

    // the same count on the host (pattern tables): exact integer floor division
    static int64_t floor_div_h(int64_t a, int64_t b)
    {
        return a >= 0 ? a / b : -((-a + b - 1) / b);
    }

#define HEAT_CLOSED_K 4
    __global__ void __launch_bounds__(256) k_heat_closed(const __grid_constant__ HeatParams p)
    {
        const HeatStream& st = p.st[blockIdx.y];
        const int64_t g = static_cast<int64_t>(p.gran), bs = static_cast<int64_t>(st.bs), b0 = static_cast<int64_t>(st.base0);
        const double invbs = 1.0 / static_cast<double>(bs), invg = 1.0 / static_cast<double>(g);
        const int64_t first = floor_div_r(b0 + static_cast<int64_t>(p.begin) * bs, g, invg);
        const int64_t last = floor_div_r(b0 + static_cast<int64_t>(p.end) * bs - 1, g, invg);
        const int64_t eb = static_cast<int64_t>(p.begin), ee = static_cast<int64_t>(p.end) - 1;
        unsigned long long* heat = p.heat + p.heatOff[st.nr];
        const int64_t P = st.period;
        const double invP = P ? 1.0 / static_cast<double>(P) : 0.0;
        // HEAT_K consecutive counters per thread: their read-modify-writes are independent, so all
        // HEAT_K loads are in flight together (one 8-byte RMW per thread left the pass latency-bound
        // at ~2 TB/s of counter traffic)
        constexpr int HEAT_K = HEAT_CLOSED_K;
        // streams with a count pattern: k_heat_pattern streams their interior [pLo, pHi]; this
        // kernel walks only the edge blocks (virtual index v -> block: below pLo, then above pHi)
        (void)invP;
        const int64_t nLow = P ? st.pLo - first : 0;
        const int64_t nv = P ? nLow + (last - st.pHi) : last - first + 1;
        auto blockOf = [&](int64_t v) { return P == 0 ? first + v : (v < nLow ? first + v : st.pHi + 1 + (v - nLow)); };
        for(int64_t vq = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * HEAT_K; vq < nv;
            vq += static_cast<int64_t>(gridDim.x) * blockDim.x * HEAT_K)
        {
            unsigned long long c[HEAT_K], h[HEAT_K];
            int64_t bk[HEAT_K];
#pragma unroll
            for(int k = 0; k < HEAT_K; ++k)
            {
                const int64_t b = blockOf(vq + k);
                bk[k] = b;
                c[k] = 0;
                if(vq + k >= nv || b > last)
                    continue;
                for(uint32_t t = st.t0; t < st.t1; ++t)
                {
                    const HeatTerm& ht = p.term[t];
                    const int64_t off = b0 + ht.inblock;
                    // overlap: off + e*bs < (b+1)g  and  off + e*bs + size > b*g
                    int64_t lo = floor_div_r(b * g - off - static_cast<int64_t>(ht.size), bs, invbs) + 1;
                    int64_t hi = floor_div_r((b + 1) * g - off - 1, bs, invbs);
                    lo = lo < eb ? eb : lo;
                    hi = hi > ee ? ee : hi;
                    if(hi >= lo)
                        c[k] += static_cast<unsigned long long>(hi - lo + 1);
                }
            }
#pragma unroll
            for(int k = 0; k < HEAT_K; ++k)
            {
                const int64_t b = bk[k];
                h[k] = (c[k] && b != first && b != last) ? heat[b] : 0;
            }
#pragma unroll
            for(int k = 0; k < HEAT_K; ++k)
            {
                const int64_t b = bk[k];
                if(!c[k])
                    continue;
                if(b == first || b == last)
                    atomicAdd(heat + b, c[k]); // edge blocks may be shared with another stream
                else
                    heat[b] = h[k] + c[k];
            }
        }
    }

    // interior heat blocks of the streams with a count pattern: a streaming read-modify-write.
    // A warp owns 32 * K consecutive counters, lane l the counters l, l + 32, ... (every load and
    // store instruction is 256 contiguous bytes); the period table is copied to shared memory
    // (per-lane indices into the constant bank would serialise).
    __global__ void __launch_bounds__(256) k_heat_pattern(const __grid_constant__ HeatParams p)
    {
        __shared__ uint32_t pat[2048];
        const HeatStream& st = p.st[blockIdx.y];
        const int64_t P = st.period;
        if(P == 0)
            return;
        for(uint32_t k = threadIdx.x; k < P; k += blockDim.x)
            pat[k] = p.pattern[st.patOff + k];
        __syncthreads();
        unsigned long long* heat = p.heat + p.heatOff[st.nr];
        const double invP = 1.0 / static_cast<double>(P);
        constexpr int K = 8;
        const int64_t lane = threadIdx.x & 31, warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
        const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
        const int64_t step32 = 32 - floor_div_r(32, P, invP) * P; // 32 mod P
        for(int64_t chunk = st.pLo + warp * 32 * K; chunk <= st.pHi; chunk += warps * 32 * K)
        {
            const int64_t b0 = chunk + lane;
            int64_t m = b0 - st.pb0;
            m -= floor_div_r(m, P, invP) * P;
            unsigned long long h[K];
#pragma unroll
            for(int k = 0; k < K; ++k)
                h[k] = b0 + 32 * k <= st.pHi ? heat[b0 + 32 * k] : 0;
#pragma unroll
            for(int k = 0; k < K; ++k)
            {
                if(b0 + 32 * k <= st.pHi)
                    heat[b0 + 32 * k] = h[k] + pat[m];
                m += step32;
                m = m >= P ? m - P : m;
            }
        }
    }

    cudaError_t heat_phys(const HeatParams& p, cudaStream_t s)
    {
        bool closed = p.nstreams > 0;
        uint64_t maxBlocks = 0;
        for(uint32_t k = 0; k < p.nstreams; ++k)
        {
            const HeatStream& st = p.st[k];
            closed = closed && st.lanes == 1;
            const uint64_t span = ((st.base0 + p.end * st.bs - 1) / p.gran) - ((st.base0 + p.begin * st.bs) / p.gran) + 1;
            maxBlocks = span > maxBlocks ? span : maxBlocks;
        }
        if(closed && p.end > p.begin)
        {
            // interior pattern per stream (P = bs / gcd(g, bs) blocks), computed with the kernel's
            // formula; blocks within ceil(bs / g) + 2 of either end stay exact
            HeatParams q = p;
            uint32_t used = 0;
            const int64_t g = static_cast<int64_t>(p.gran);
            for(uint32_t k = 0; k < q.nstreams; ++k)
            {
                HeatStream& st = q.st[k];
                st.period = 0;
                const int64_t bs = static_cast<int64_t>(st.bs), b0 = static_cast<int64_t>(st.base0);
                int64_t a = g, bb = bs;
                while(bb)
                {
                    const int64_t t = a % bb;
                    a = bb;
                    bb = t;
                }
                const int64_t P = bs / a;
                const int64_t first = floor_div_h(b0 + static_cast<int64_t>(p.begin) * bs, g);
                const int64_t last = floor_div_h(b0 + static_cast<int64_t>(p.end) * bs - 1, g);
                const int64_t D = (bs + g - 1) / g + 2;
                if(P < 1 || used + P > sizeof(q.pattern) / sizeof(q.pattern[0]) || last - first + 1 < 2 * D + P
                   || std::getenv("LAMB_HEAT_PATTERN") && std::getenv("LAMB_HEAT_PATTERN")[0] == '0')
                    continue;
                st.pb0 = first + D;
                st.pLo = first + D;
                st.pHi = last - D;
                st.period = static_cast<uint32_t>(P);
                st.patOff = used;
                for(int64_t j = 0; j < P; ++j)
                {
                    const int64_t b = st.pb0 + j;
                    uint64_t cnt = 0;
                    for(uint32_t t = st.t0; t < st.t1; ++t)
                    {
                        const HeatTerm& ht = q.term[t];
                        const int64_t off = b0 + ht.inblock;
                        const int64_t lo = floor_div_h(b * g - off - static_cast<int64_t>(ht.size), bs) + 1;
                        const int64_t hi = floor_div_h((b + 1) * g - off - 1, bs);
                        if(hi >= lo)
                            cnt += static_cast<uint64_t>(hi - lo + 1);
                    }
                    q.pattern[used + j] = static_cast<uint32_t>(cnt);
                }
                used += static_cast<uint32_t>(P);
            }
            // one pass, HEAT_CLOSED_K = 4 counters per thread (ncu: 84 instructions per counter, the
            // per-thread setup dominating; but 16 counters per thread and a grid-stride grid both
            // measured slower -- fewer counter loads in flight)
            uint64_t maxInterior = 0, maxRest = 0;
            for(uint32_t k = 0; k < q.nstreams; ++k)
            {
                const HeatStream& st = q.st[k];
                const uint64_t span = ((st.base0 + p.end * st.bs - 1) / p.gran) - ((st.base0 + p.begin * st.bs) / p.gran) + 1;
                const uint64_t inner = st.period ? static_cast<uint64_t>(st.pHi - st.pLo + 1) : 0;
                maxInterior = std::max(maxInterior, inner);
                maxRest = std::max(maxRest, span - inner);
            }
            if(maxInterior)
            {
                const unsigned gp = stream_grid((maxInterior + 8 * 256 - 1) / (8 * 256), "LAMB_HEAT_CTAS", 0);
                k_heat_pattern<<<dim3(gp, q.nstreams), 256, 0, s>>>(q);
                count_launch();
            }
            const unsigned gx = stream_grid((maxRest + HEAT_CLOSED_K * 256 - 1) / (HEAT_CLOSED_K * 256), "LAMB_HEAT_CTAS", 0);
            k_heat_closed<<<dim3(gx, q.nstreams), 256, 0, s>>>(q);
            count_launch();
            return cudaGetLastError();
        }
        if(p.end <= p.begin || p.nstreams == 0)
            return cudaSuccess;
        const uint64_t ctas = (p.end - p.begin + p.E - 1) / p.E; // E is sized on the host
        const size_t smem = static_cast<size_t>(p.maxWindow) * sizeof(unsigned long long);
        if(cudaError_t e = opt_in_smem(reinterpret_cast<const void*>(k_heat_phys), smem); e != cudaSuccess)
            return e;
        k_heat_phys<<<static_cast<unsigned>(ctas), 256, smem, s>>>(p);
        count_launch();
        return cudaGetLastError();
    }

    __global__ void k_fac_add(unsigned long long* src, unsigned long long* dst, uint32_t nl, unsigned long long cnt)
    {
        for(uint32_t f = threadIdx.x; f < nl; f += blockDim.x)
        {
            if(src)
                src[f] += cnt;
            if(dst)
                dst[nl + f] += cnt;
        }
    }

    cudaError_t fac_add(unsigned long long* srcCounters, unsigned long long* dstCounters, uint32_t nleaves,
                        uint64_t count, cudaStream_t s)
    {
        k_fac_add<<<1, 64, 0, s>>>(srcCounters, dstCounters, nleaves, count);
        count_launch();
        return cudaGetLastError();
    }

    unsigned stream_grid(uint64_t want, const char* env, uint64_t perSm)
    {
        if(const char* e = getenv(env))
            perSm = static_cast<uint64_t>(atoll(e));
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t cap = perSm ? perSm * static_cast<uint64_t>(sm_count(dev)) : want;
        const uint64_t g = want < cap ? want : cap;
        return static_cast<unsigned>(g == 0 ? 1 : (g > 0x7FFFFFFFull ? 0x7FFFFFFFull : g));
    }

    cudaError_t blob_copy(void* dst, const void* src, uint64_t bytes, cudaStream_t s)
    {
        if(bytes == 0)
            return cudaSuccess;
        int dev = 0;
        cudaGetDevice(&dev);
        const unsigned sms = static_cast<unsigned>(sm_count(dev));
        const bool aligned = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
        uint64_t head = 0;
        if(aligned)
        {
            const uint64_t n16 = bytes / 16;
            if(n16)
            {
                static const int U = [] { const char* e = getenv("LAMB_BLOB_U"); return e ? atoi(e) : 2; }();
                const unsigned grid = stream_grid((n16 + 256 * U - 1) / (256 * U), "LAMB_BLOB_CTAS", 0);
                auto* dp = static_cast<uint4*>(dst);
                auto* sp = static_cast<const uint4*>(src);
                if(U == 8)
                    k_blob_copy16<8><<<grid, 256, 0, s>>>(dp, sp, n16);
                else if(U == 2)
                    k_blob_copy16<2><<<grid, 256, 0, s>>>(dp, sp, n16);
                else if(U == 1)
                    k_blob_copy16<1><<<grid, 256, 0, s>>>(dp, sp, n16);
                else
                    k_blob_copy16<4><<<grid, 256, 0, s>>>(dp, sp, n16);
                count_launch();
            }
            head = n16 * 16;
        }
        if(head < bytes)
        {
            const uint64_t rest = bytes - head;
            const uint64_t want = (rest + 255) / 256;
            const unsigned grid = static_cast<unsigned>(want < sms * 8ull ? want : sms * 8ull);
            k_blob_copy1<<<grid, 256, 0, s>>>(static_cast<uint8_t*>(dst) + head, static_cast<const uint8_t*>(src) + head,
                                              rest);
            count_launch();
        }
        return cudaGetLastError();
    }

    cudaError_t blob_copy_multi(void* const* dst, const void* const* src, const uint64_t* bytes, size_t n, cudaStream_t s)
    {
        // 16-byte aligned, whole-vector blobs go through k_blob_copy16_multi, 16 per launch;
        // anything else through blob_copy
        BlobSegs g{};
        uint32_t cnt = 0;
        uint64_t maxN = 0;
        auto flush = [&]
        {
            if(cnt == 0)
                return;
            const unsigned grid = stream_grid((maxN + 256 * 2 - 1) / (256 * 2), "LAMB_BLOB_CTAS", 0);
            k_blob_copy16_multi<2><<<dim3(grid, cnt), 256, 0, s>>>(g);
            count_launch();
            g = BlobSegs{};
            cnt = 0;
            maxN = 0;
        };
        for(size_t k = 0; k < n; ++k)
        {
            if(bytes[k] == 0)
                continue;
            const bool whole = ((reinterpret_cast<uintptr_t>(dst[k]) | reinterpret_cast<uintptr_t>(src[k])) & 15) == 0
                && bytes[k] % 16 == 0;
            if(!whole)
            {
                const cudaError_t e = blob_copy(dst[k], src[k], bytes[k], s);
                if(e != cudaSuccess)
                    return e;
                continue;
            }
            g.d[cnt] = static_cast<uint4*>(dst[k]);
            g.s[cnt] = static_cast<const uint4*>(src[k]);
            g.n16[cnt] = bytes[k] / 16;
            maxN = g.n16[cnt] > maxN ? g.n16[cnt] : maxN;
            if(++cnt == 16)
                flush();
        }
        flush();
        return cudaGetLastError();
    }

    // ---- funnel access by (linear, leaf) pairs (View::read / View::write) ------------------
    __global__ void k_read_values(const lamp_view* __restrict__ V, const uint64_t* __restrict__ lin,
                                  const uint32_t* __restrict__ leaf, uint64_t* __restrict__ out, size_t n)
    {
        const lamd::ViewCtx c = lamd::make_ctx(V);
        for(size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
            k += static_cast<size_t>(gridDim.x) * blockDim.x)
            out[k] = lamd::read_node<LAMP_MAX_DEPTH>(c, V->roots[leaf[k]], lin[k]);
    }

    __global__ void k_write_values(const lamp_view* __restrict__ V, const uint64_t* __restrict__ lin,
                                   const uint32_t* __restrict__ leaf, const uint64_t* __restrict__ in, size_t n)
    {
        const lamd::ViewCtx c = lamd::make_ctx(V);
        for(size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
            k += static_cast<size_t>(gridDim.x) * blockDim.x)
        {
            const uint32_t r = V->roots[leaf[k]];
            uint64_t bits = in[k];
            const int t = V->nodes[r].type;
            // ScalarValue::fromStorageBits canonicalisation of the incoming value (scalar.hpp:251-271)
            bits = t == lamd::BOOL ? uint64_t((bits & 0xFF) != 0) : (bits & lamd::low_mask(8 * lamd::scalar_size(t)));
            lamd::write_node<LAMP_MAX_DEPTH>(c, r, lin[k], bits);
        }
    }

    cudaError_t read_values(const lamp_view* v, const uint64_t* lin, const uint32_t* leaf, uint64_t* out, size_t n,
                            cudaStream_t s)
    {
        if(n == 0)
            return cudaSuccess;
        const unsigned grid = static_cast<unsigned>(n / 256 + 1 < 4096 ? n / 256 + 1 : 4096);
        k_read_values<<<grid, 256, 0, s>>>(v, lin, leaf, out, n);
        count_launch();
        return cudaGetLastError();
    }

    cudaError_t write_values(const lamp_view* v, const uint64_t* lin, const uint32_t* leaf, const uint64_t* in,
                             size_t n, cudaStream_t s)
    {
        if(n == 0)
            return cudaSuccess;
        const unsigned grid = static_cast<unsigned>(n / 256 + 1 < 4096 ? n / 256 + 1 : 4096);
        k_write_values<<<grid, 256, 0, s>>>(v, lin, leaf, in, n);
        count_launch();
        return cudaGetLastError();
    }
} // namespace lamk
