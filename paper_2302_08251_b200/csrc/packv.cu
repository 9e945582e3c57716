// Bit packing for value sizes other than the 32-bit fast path (pack.cu k_pack32 /
// k_unpack32): 1-, 2- and 8-byte leaves (BitpackIntSoA on i8/u8/i16/u16/i64/u64 leaves,
// BitpackFloatSoA on f64 leaves, computed.cpp:48-222) and 4-byte leaves whose field is wider
// than 32 bits (e.g. bitpack-float:11,30 on f32).  Same ownership rule as k_pack32: a thread
// owns 32 consecutive values = w whole 32-bit words of the stream (w = field width, 1..64), so
// no word is shared and no read-modify-write is needed (bitpack.hpp:16-17).  The warp's 1024
// values move as coalesced 16-byte chunks through a padded shared-memory row per lane (row
// stride 2*VS+1 chunks: conflict-free both ways), the words through an odd-stride word slice
// that aliases it, then leave as coalesced 32-bit stores.
//   encode: integers keep the low w bits (packInt, bitpack.cpp:72-80); f32 -> float_encode_f32,
//           f64 -> float_encode (floatEncode, bitpack.cpp:96-163)
//   decode: zero/sign extension to the leaf width (unpackUnsigned/Signed, bitpack.cpp:82-94);
//           floatDecode -> the leaf's float type (bitpack.cpp:165-188)
#include "device_common.cuh"
#include "launch.h"

#include <utility>

namespace lamk
{
    __device__ __forceinline__ PackVParams leafv_params(const PackVMulti& M)
    {
        PackVParams p = M.base;
        const uint32_t y = blockIdx.y;
        p.vals = M.vals[y];
        p.bits = M.bits[y];
        p.vinb = M.vinb[y];
        p.sgn = M.sgn[y];
        return p;
    }

    namespace
    {
        template<int VS>
        __device__ __forceinline__ uint64_t vaddr(const PackVParams& p, uint64_t e)
        {
            if(p.vl == 1)
                return p.vals + e * VS;
            return p.vals + (e >> p.vsh) * p.vbs + p.vinb + (e & (p.vl - 1)) * VS;
        }

        template<int VS>
        __device__ __forceinline__ uint64_t enc(const PackVParams& p, uint64_t v)
        {
            if(p.kind == 0)
                return v & lamd::low_mask(p.w);
            if constexpr(VS == 4)
                return lamd::float_encode_f32(static_cast<uint32_t>(v), p.E, p.M);
            else
                return lamd::float_encode(v, p.E, p.M);
        }

        template<int VS>
        __device__ __forceinline__ uint64_t dec(const PackVParams& p, uint64_t pat)
        {
            if(p.kind == 0)
            {
                if(p.sgn && p.w < 64)
                {
                    const uint64_t s = 1ull << (p.w - 1);
                    pat = (pat ^ s) - s;
                }
                return pat & lamd::low_mask(8 * VS);
            }
            if constexpr(VS == 4)
            {
                if(p.E <= 8 && p.M <= 23)
                    return lamd::float_decode_f32(static_cast<uint32_t>(pat), p.E, p.M);
                return lamd::f64_to_f32_bits(lamd::float_decode(pat, p.E, p.M));
            }
            else
                return lamd::float_decode(pat, p.E, p.M);
        }

        // row of lane r: 32 values (32*VS bytes) + 16 bytes of padding
        template<int VS>
        __host__ __device__ constexpr uint32_t row_words()
        {
            return 8 * VS + 4;
        }
        template<int VS>
        __host__ __device__ constexpr uint32_t warp_words()
        {
            return 32 * row_words<VS>() > 32 * 65 ? 32 * row_words<VS>() : 32 * 65;
        }

        // value chunks (16 B) of the warp's span <-> rows: chunk c = row c / (2VS), column c % (2VS)
        template<int VS>
        __device__ __forceinline__ void g2s(const PackVParams& p, uint32_t* sm, uint64_t e0, uint32_t lane, uint32_t live)
        {
            constexpr uint32_t CPR = 2 * VS; // chunks per row
            const uint32_t chunks = live * CPR;
            if(live == 32)
            {
                uint4 x[CPR];
#pragma unroll
                for(uint32_t k = 0; k < CPR; ++k)
                    x[k] = __ldcs(reinterpret_cast<const uint4*>(vaddr<VS>(p, e0 + (lane + 32 * k) * 16 / VS)));
#pragma unroll
                for(uint32_t k = 0; k < CPR; ++k)
                {
                    const uint32_t c = lane + 32 * k;
                    *reinterpret_cast<uint4*>(sm + (c / CPR) * row_words<VS>() + (c % CPR) * 4) = x[k];
                }
                return;
            }
            for(uint32_t c = lane; c < chunks; c += 32)
                *reinterpret_cast<uint4*>(sm + (c / CPR) * row_words<VS>() + (c % CPR) * 4)
                    = __ldcs(reinterpret_cast<const uint4*>(vaddr<VS>(p, e0 + c * 16 / VS)));
        }

        // full-warp value span in two halves, so the next span's loads can be issued before the
        // current one is processed: global -> registers, registers -> rows
        template<int VS>
        __device__ __forceinline__ void g2r(const PackVParams& p, uint4 (&x)[2 * VS], uint64_t e0, uint32_t lane)
        {
#pragma unroll
            for(uint32_t k = 0; k < 2 * VS; ++k)
                x[k] = __ldcs(reinterpret_cast<const uint4*>(vaddr<VS>(p, e0 + (lane + 32 * k) * 16 / VS)));
        }
        template<int VS>
        __device__ __forceinline__ void r2s(uint32_t* sm, const uint4 (&x)[2 * VS], uint32_t lane)
        {
#pragma unroll
            for(uint32_t k = 0; k < 2 * VS; ++k)
            {
                const uint32_t c = lane + 32 * k;
                *reinterpret_cast<uint4*>(sm + (c / (2 * VS)) * row_words<VS>() + (c % (2 * VS)) * 4) = x[k];
            }
        }

        template<int VS>
        __device__ __forceinline__ void s2g(const PackVParams& p, const uint32_t* sm, uint64_t e0, uint32_t lane,
                                            uint32_t live)
        {
            constexpr uint32_t CPR = 2 * VS;
            const uint32_t chunks = live * CPR;
            for(uint32_t c = lane; c < chunks; c += 32)
                __stcs(reinterpret_cast<uint4*>(vaddr<VS>(p, e0 + c * 16 / VS)),
                       *reinterpret_cast<const uint4*>(sm + (c / CPR) * row_words<VS>() + (c % CPR) * 4));
        }

        // word q = lane + 32k of the warp's span lives in row q / w, column q % w of the word
        // slice (row stride ws); walked incrementally, no division in the loop
        struct WordWalk
        {
            uint32_t r, c, dr, dc, w;
            __device__ __forceinline__ WordWalk(uint32_t lane, uint32_t w_) : w(w_)
            {
                r = lane / w;
                c = lane - r * w;
                dr = 32 / w;
                dc = 32 - dr * w;
            }
            __device__ __forceinline__ void next()
            {
                r += dr;
                c += dc;
                if(c >= w)
                {
                    c -= w;
                    ++r;
                }
            }
        };

        // value i of a row held as 8*VS words
        template<int VS>
        __device__ __forceinline__ uint64_t value_of(const uint32_t* wd, int i)
        {
            if constexpr(VS == 1)
                return (wd[i >> 2] >> (8 * (i & 3))) & 0xFFu;
            else if constexpr(VS == 2)
                return (wd[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
            else if constexpr(VS == 4)
                return wd[i];
            else
                return static_cast<uint64_t>(wd[2 * i]) | (static_cast<uint64_t>(wd[2 * i + 1]) << 32);
        }
    } // namespace

    // W != 0: compile-time field width of an integer leaf of 1 or 2 bytes (word boundaries at
    // compile-time positions: pure shift/or chains, as k_pack32); W == 0: runtime width / float
    template<int VS, int W = 0>
    __global__ void __launch_bounds__(256, VS == 8 ? 2 : 3) k_packv(const __grid_constant__ PackVMulti M)
    {
        const PackVParams p = leafv_params(M);
        extern __shared__ __align__(16) uint32_t vsm[];
        const uint32_t lane = threadIdx.x & 31, w = W ? W : p.w, ws = w | 1u;
        uint32_t* sm = vsm + (threadIdx.x >> 5) * warp_words<VS>();
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        const uint64_t gEnd = (p.groups + 31) / 32 * 32;
        auto liveOf = [&](uint64_t warpG) -> uint32_t
        {
            return static_cast<uint32_t>(p.groups > warpG ? (p.groups - warpG < 32 ? p.groups - warpG : 32) : 0);
        };
        // software pipeline: the next full span's 16-byte loads are in flight while the current
        // span is packed and stored (one span of loads per warp was latency-bound)
        // (1- and 2-byte values only: a second span of 8-byte values would spill)
        constexpr bool PF = VS <= 2;
        uint4 xn[2 * VS];
        const uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        bool pre = PF && g0 - lane < gEnd && liveOf(g0 - lane) == 32;
        if(pre)
            g2r<VS>(p, xn, p.begin + (g0 - lane) * 32, lane);
        for(uint64_t g = g0; g - lane < gEnd; g += stride)
        {
            const uint64_t warpG = g - lane;
            const uint32_t live = liveOf(warpG);
            const uint64_t e0 = p.begin + warpG * 32;
            if(pre)
                r2s<VS>(sm, xn, lane);
            else
                g2s<VS>(p, sm, e0, lane, live);
            const uint64_t nextG = warpG + stride;
            pre = PF && nextG < gEnd && liveOf(nextG) == 32;
            if(pre)
                g2r<VS>(p, xn, p.begin + nextG * 32, lane);
            __syncwarp();
            uint32_t wd[8 * VS];
            const bool mine = g < p.groups;
            if(mine)
            {
#pragma unroll
                for(int q = 0; q < 2 * VS; ++q)
                {
                    const uint4 x = *reinterpret_cast<const uint4*>(sm + lane * row_words<VS>() + 4 * q);
                    wd[4 * q] = x.x;
                    wd[4 * q + 1] = x.y;
                    wd[4 * q + 2] = x.z;
                    wd[4 * q + 3] = x.w;
                }
            }
            __syncwarp(); // rows consumed: the word slice (aliasing them) may be written
            if(mine && W != 0)
            {
                uint32_t* my = sm + lane * ws;
                constexpr uint32_t mask = W >= 32 ? 0xFFFFFFFFu : (1u << (W ? W : 1)) - 1u;
                uint32_t e[32];
#pragma unroll
                for(int i = 0; i < 32; ++i)
                    e[i] = static_cast<uint32_t>(value_of<VS>(wd, i)) & mask;
                // word k = bits [32k, 32k+32): values floor(32k/W) .. floor((32k+31)/W)
#pragma unroll
                for(int k = 0; k < (W ? W : 1); ++k)
                {
                    uint32_t word = 0;
#pragma unroll
                    for(int i = (32 * k) / (W ? W : 1); i <= (32 * k + 31) / (W ? W : 1) && i < 32; ++i)
                    {
                        const int pos = i * W - 32 * k;
                        word |= pos >= 0 ? e[i] << pos : e[i] >> (-pos);
                    }
                    my[k] = word;
                }
            }
            else if(mine)
            {
                uint32_t* my = sm + lane * ws;
                unsigned long long acc = 0;
                uint32_t nb = 0, k = 0;
#pragma unroll
                for(int i = 0; i < 32; ++i)
                {
                    const uint64_t e = enc<VS>(p, value_of<VS>(wd, i));
                    if(VS <= 2 || w <= 32)
                    {
                        acc |= e << nb;
                        nb += w;
                        if(nb >= 32)
                        {
                            my[k++] = static_cast<uint32_t>(acc);
                            acc >>= 32;
                            nb -= 32;
                        }
                    }
                    else
                    {
                        acc |= (e & 0xFFFFFFFFull) << nb;
                        my[k++] = static_cast<uint32_t>(acc);
                        acc >>= 32;
                        acc |= (e >> 32) << nb;
                        nb += w - 32;
                        if(nb >= 32)
                        {
                            my[k++] = static_cast<uint32_t>(acc);
                            acc >>= 32;
                            nb -= 32;
                        }
                    }
                }
            }
            __syncwarp();
            uint32_t* dst = reinterpret_cast<uint32_t*>(p.bits) + e0 / 32 * w;
            if(W != 0 && live == 32)
            {
#pragma unroll
                for(int k = 0; k < (W ? W : 1); ++k)
                {
                    const uint32_t q = lane + 32 * k;
                    __stcs(dst + q, sm[(q / w) * ws + (q % w)]);
                }
            }
            else
            {
                WordWalk ww(lane, w);
                for(uint32_t q = lane; q < live * w; q += 32, ww.next())
                    __stcs(dst + q, sm[ww.r * ws + ww.c]);
            }
            __syncwarp();
        }
    }

    template<int VS, int W = 0>
    __global__ void __launch_bounds__(256, VS == 8 ? 2 : 3) k_unpackv(const __grid_constant__ PackVMulti M)
    {
        const PackVParams p = leafv_params(M);
        extern __shared__ __align__(16) uint32_t vsm[];
        const uint32_t lane = threadIdx.x & 31, w = W ? W : p.w, ws = w | 1u;
        uint32_t* sm = vsm + (threadIdx.x >> 5) * warp_words<VS>();
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        const uint64_t gEnd = (p.groups + 31) / 32 * 32;
        const uint64_t mask = lamd::low_mask(w);
        auto liveOf = [&](uint64_t warpG) -> uint32_t
        {
            return static_cast<uint32_t>(p.groups > warpG ? (p.groups - warpG < 32 ? p.groups - warpG : 32) : 0);
        };
        // compile-time widths: the next full span's W word loads are issued before the current
        // span is decoded and stored (software pipeline, as k_packv)
        uint32_t tn[W ? W : 1];
        const uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        auto words_of = [&](uint64_t warpG) { return reinterpret_cast<const uint32_t*>(p.bits) + (p.begin + warpG * 32) / 32 * w; };
        bool pre = W != 0 && g0 - lane < gEnd && liveOf(g0 - lane) == 32;
        if(pre)
        {
#pragma unroll
            for(int k = 0; k < (W ? W : 1); ++k)
                tn[k] = __ldcs(words_of(g0 - lane) + lane + 32 * k);
        }
        for(uint64_t g = g0; g - lane < gEnd; g += stride)
        {
            const uint64_t warpG = g - lane;
            const uint32_t live = liveOf(warpG);
            const uint64_t e0 = p.begin + warpG * 32;
            const uint32_t* src = words_of(warpG);
            const bool had = pre;
            if(had)
            {
#pragma unroll
                for(int k = 0; k < (W ? W : 1); ++k)
                {
                    const uint32_t q = lane + 32 * k;
                    sm[(q / w) * ws + (q % w)] = tn[k];
                }
            }
            const uint64_t nextG = warpG + stride;
            pre = W != 0 && nextG < gEnd && liveOf(nextG) == 32;
            if(pre)
            {
#pragma unroll
                for(int k = 0; k < (W ? W : 1); ++k)
                    tn[k] = __ldcs(words_of(nextG) + lane + 32 * k);
            }
            if(had)
            {
            }
            else
            {
                WordWalk ww(lane, w);
                for(uint32_t q = lane; q < live * w; q += 32, ww.next())
                    sm[ww.r * ws + ww.c] = __ldcs(src + q);
            }
            __syncwarp();
            uint32_t wd[8 * VS];
            const bool mine = g < p.groups;
            if(mine && W != 0)
            {
                const uint32_t* my = sm + lane * ws;
                uint32_t wds[W ? W : 1];
#pragma unroll
                for(int k = 0; k < (W ? W : 1); ++k)
                    wds[k] = my[k];
                constexpr uint32_t mask = W >= 32 ? 0xFFFFFFFFu : (1u << (W ? W : 1)) - 1u;
#pragma unroll
                for(int i = 0; i < 32; ++i)
                {
                    const int bit = i * W, k = bit >> 5, sh = bit & 31;
                    uint32_t pat = wds[k] >> sh;
                    if(sh + W > 32)
                        pat |= wds[k + 1] << (32 - sh);
                    pat &= mask;
                    if(p.sgn && W < 32)
                    {
                        const uint32_t sb = 1u << (W - 1);
                        pat = (pat ^ sb) - sb;
                    }
                    const uint32_t v = VS == 1 ? pat & 0xFFu : pat & 0xFFFFu;
                    if constexpr(VS == 1)
                    {
                        if((i & 3) == 0)
                            wd[i >> 2] = 0;
                        wd[i >> 2] |= v << (8 * (i & 3));
                    }
                    else
                    {
                        if((i & 1) == 0)
                            wd[i >> 1] = 0;
                        wd[i >> 1] |= v << (16 * (i & 1));
                    }
                }
            }
            else if(mine)
            {
                const uint32_t* my = sm + lane * ws;
                // stream the lane's words through a 64-bit window: at most one word refill per
                // value for w <= 32, two for wider fields
                unsigned long long acc = 0;
                uint32_t nb = 0, k = 0;
#pragma unroll
                for(int i = 0; i < 32; ++i)
                {
                    uint64_t pat;
                    if(VS <= 2 || w <= 32)
                    {
                        if(nb < w)
                        {
                            acc |= static_cast<unsigned long long>(my[k++]) << nb;
                            nb += 32;
                        }
                        pat = acc & mask;
                        acc >>= w;
                        nb -= w;
                    }
                    else
                    {
                        // w in (32, 64]: low 32 bits, then the remaining w - 32
                        if(nb < 32)
                        {
                            acc |= static_cast<unsigned long long>(my[k++]) << nb;
                            nb += 32;
                        }
                        pat = acc & 0xFFFFFFFFull;
                        acc >>= 32;
                        nb -= 32;
                        const uint32_t hw = w - 32;
                        if(nb < hw)
                        {
                            acc |= static_cast<unsigned long long>(my[k++]) << nb;
                            nb += 32;
                        }
                        pat |= (acc & lamd::low_mask(hw)) << 32;
                        acc >>= hw;
                        nb -= hw;
                    }
                    const uint64_t v = dec<VS>(p, pat);
                    if constexpr(VS == 1)
                    {
                        if((i & 3) == 0)
                            wd[i >> 2] = 0;
                        wd[i >> 2] |= static_cast<uint32_t>(v) << (8 * (i & 3));
                    }
                    else if constexpr(VS == 2)
                    {
                        if((i & 1) == 0)
                            wd[i >> 1] = 0;
                        wd[i >> 1] |= static_cast<uint32_t>(v) << (16 * (i & 1));
                    }
                    else if constexpr(VS == 4)
                        wd[i] = static_cast<uint32_t>(v);
                    else
                    {
                        wd[2 * i] = static_cast<uint32_t>(v);
                        wd[2 * i + 1] = static_cast<uint32_t>(v >> 32);
                    }
                }
            }
            __syncwarp(); // words consumed: rows (aliasing them) may be written
            if(mine)
            {
#pragma unroll
                for(int q = 0; q < 2 * VS; ++q)
                    *reinterpret_cast<uint4*>(sm + lane * row_words<VS>() + 4 * q)
                        = make_uint4(wd[4 * q], wd[4 * q + 1], wd[4 * q + 2], wd[4 * q + 3]);
            }
            __syncwarp();
            s2g<VS>(p, sm, e0, lane, live);
            __syncwarp();
        }
    }

    template<int VS, int W = 0>
    static void launch_v(const PackVMulti& m, uint32_t n, bool pack, cudaStream_t s)
    {
        const PackVParams& p = m.base;
        int dev = 0;
        cudaGetDevice(&dev);
        const size_t smem = 8 * warp_words<VS>() * sizeof(uint32_t);
        auto kern = pack ? k_packv<VS, W> : k_unpackv<VS, W>;
        lam_cuda_check(opt_in_smem(reinterpret_cast<const void*>(kern), smem), "opt_in_smem");
        int occ = 0;
        if(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem) != cudaSuccess || occ < 1)
            occ = 1;
        const uint64_t want = (p.groups + 255) / 256;
        const uint64_t cap = static_cast<uint64_t>(sm_count(dev)) * occ * 4;
        const unsigned grid = static_cast<unsigned>(want < cap ? want : cap);
        kern<<<dim3(grid, n), 256, smem, s>>>(m);
    }

    // integer leaves of 1 / 2 bytes: a compile-time width per kernel
    template<int VS, int... Ws>
    static bool dispatch_narrow(const PackVMulti& m, uint32_t n, bool pack, cudaStream_t s,
                                std::integer_sequence<int, Ws...>)
    {
        bool hit = false;
        ((static_cast<int>(m.base.w) == Ws + 1 ? (launch_v<VS, Ws + 1>(m, n, pack, s), hit = true) : false), ...);
        return hit;
    }

    // jobs[0..n): leaves with the same value size, width, format and range, one launch (leaf = blockIdx.y)
    bool packv(const PackVParams* jobs, uint32_t n, uint32_t vsize, bool pack, cudaStream_t s)
    {
        if(n == 0 || n > 8)
            return false;
        const PackVParams& p = jobs[0];
        if(p.groups == 0 || p.w < 1 || p.w > 64 || (p.kind == 0 && p.w > 8 * vsize))
            return false;
        PackVMulti m{};
        m.base = p;
        for(uint32_t k = 0; k < n; ++k)
        {
            const PackVParams& j = jobs[k];
            if(j.w != p.w || j.kind != p.kind || j.E != p.E || j.M != p.M || j.groups != p.groups || j.begin != p.begin
               || j.vbs != p.vbs || j.vl != p.vl || j.vsh != p.vsh)
                return false;
            m.vals[k] = j.vals;
            m.bits[k] = j.bits;
            m.vinb[k] = j.vinb;
            m.sgn[k] = j.sgn;
        }
        switch(vsize)
        {
        case 1:
            if(p.kind != 0 || !dispatch_narrow<1>(m, n, pack, s, std::make_integer_sequence<int, 8>{}))
                launch_v<1>(m, n, pack, s);
            break;
        case 2:
            if(p.kind != 0 || !dispatch_narrow<2>(m, n, pack, s, std::make_integer_sequence<int, 16>{}))
                launch_v<2>(m, n, pack, s);
            break;
        case 4:
            launch_v<4>(m, n, pack, s);
            break;
        case 8:
            launch_v<8>(m, n, pack, s);
            break;
        default:
            return false;
        }
        count_launch();
        lam_cuda_check(cudaGetLastError(), "kernel launch");
        return true;
    }
} // namespace lamk
