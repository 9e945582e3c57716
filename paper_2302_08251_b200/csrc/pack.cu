// Register-direct kernels for the computed mappings on the benchmark configs.
//
// K3/K4  bit packing (BitpackIntSoA / BitpackFloatSoA, computed.cpp:48-222): a thread owns
//        32 consecutive values = `w` whole 32-bit words of the bit stream (w = field width),
//        so words are never shared between threads (no RMW, bitpack.hpp:16-17).  Values move
//        as 16-byte vectors; the word spans of a warp are staged in a warp-private smem slice
//        (lane stride w words) so global stream traffic is coalesced 128-byte lines.
//        f32 e8m10 / e5m10 use the exact integer/half fast encoders (device_common.cuh),
//        every other (E, M) the integer-exact floatEncode restatement.
// K5     convert-on-access + byte split (ChangeType f64->f32 then Bytesplit into plane
//        streams, computed.cpp:363-378, 473-490): a thread owns 4 records, loads them as
//        16-byte vectors, converts with x86 NaN rules and writes one 32-bit word per plane.
#include "device_common.cuh"

#include <cstdlib>
#include "launch.h"

namespace lamk
{
    struct PackParams
    {
        unsigned long long vals;   // value stream (leaf-contiguous, 4-byte values, element 0)
        unsigned long long bits;   // bit stream (word 0 = element 0)
        unsigned long long begin;  // first element (multiple of 32)
        unsigned long long groups; // groups of 32 elements
        uint32_t w;                // field width (bits), 1..32
        uint32_t kind;             // 0 int, 1 float
        uint32_t sgn;              // int: sign-extend on unpack
        uint32_t E, M;             // float format
        uint32_t valType;          // LAM_I32/U32/F32 ... of the values
        unsigned long long facSrc, facDst;
        uint32_t facS, facD, leaf, nleaves;
        uint32_t vbs, vl, vsh, vinb; // value-stream geometry: AoSoA lanes (vl % 32 == 0) or SoA (vl == 1)
    };

    __device__ __forceinline__ uint64_t val_addr(const PackParams& p, uint64_t e0)
    {
        if(p.vl == 1)
            return p.vals + e0 * 4;
        return p.vals + (e0 >> p.vsh) * p.vbs + p.vinb + (e0 & (p.vl - 1)) * 4;
    }

    __device__ __forceinline__ uint32_t encode_value(const PackParams& p, uint32_t v)
    {
        if(p.kind == 0)
            return p.w >= 32 ? v : (v & ((1u << p.w) - 1u));
        if(p.E == 8 && p.M == 10)
            return lamd::encode_e8m10_f32(v);
        if(p.E == 5 && p.M == 10)
            return lamd::encode_e5m10_f32(v);
        return static_cast<uint32_t>(lamd::float_encode_f32(v, p.E, p.M));
    }

    __device__ __forceinline__ uint32_t decode_value(const PackParams& p, uint32_t pat)
    {
        if(p.kind == 0)
        {
            if(p.sgn && p.w < 32)
            {
                const uint32_t s = 1u << (p.w - 1);
                return (pat ^ s) - s;
            }
            return pat;
        }
        if(p.E == 8 && p.M == 10)
        {
            const uint32_t sign = (pat >> 18) << 31;
            if((pat & 0x3FC00u) == 0x3FC00u && (pat & 0x3FFu))
                return sign | 0x7FC00000u;
            return sign | ((pat & 0x3FFFFu) << 13);
        }
        if(p.E == 5 && p.M == 10)
        {
            if((pat & 0x7C00u) == 0x7C00u && (pat & 0x3FFu))
                return ((pat >> 15) << 31) | 0x7FC00000u;
            return __float_as_uint(__half2float(__ushort_as_half(static_cast<unsigned short>(pat))));
        }
        if(p.E <= 8 && p.M <= 23)
            return lamd::float_decode_f32(pat, p.E, p.M);
        return lamd::f64_to_f32_bits(lamd::float_decode(pat, p.E, p.M));
    }

    __device__ __forceinline__ void fac_flush(const PackParams& p, unsigned long long cnt)
    {
        if(!(p.facS || p.facD))
            return;
        for(int o = 16; o > 0; o >>= 1)
            cnt += __shfl_down_sync(0xFFFFFFFFu, cnt, o);
        if((threadIdx.x & 31) == 0 && cnt)
        {
            if(p.facS)
                atomicAdd(reinterpret_cast<unsigned long long*>(p.facSrc) + p.leaf, cnt);
            if(p.facD)
                atomicAdd(reinterpret_cast<unsigned long long*>(p.facDst) + p.nleaves + p.leaf, cnt);
        }
    }

    // Compile-time field width: the 32 values of a thread map to exactly W words, and the
    // word boundaries fall at compile-time positions, so packing is pure shift/or chains.
    // FMT: 0 integer, 1 f32 e8m10 (W=19), 2 f32 e5m10 (W=16), 3 any f32 format with E <= 8,
    // M <= 23 (runtime E, M; the 32-bit codec), 4 any float format (runtime E, M).
    template<int FMT>
    __device__ __forceinline__ uint32_t enc_t(const PackParams& p, const lamd::F32Codec& fc, uint32_t v, uint32_t mask)
    {
        if constexpr(FMT == 0)
            return v & mask;
        else if constexpr(FMT == 1)
            return lamd::encode_e8m10_f32(v);
        else if constexpr(FMT == 2)
            return lamd::encode_e5m10_f32(v);
        else if constexpr(FMT == 3)
            return lamd::f32_encode_bf(fc, v);
        else if constexpr(FMT == 5)
            return lamd::f32_encode_bf(lamd::f32_codec(4, 3), v); // e4m3: every constant an immediate
        else if constexpr(FMT == 6)
            return lamd::f32_encode_bf(lamd::f32_codec(5, 2), v); // e5m2
        else
            return static_cast<uint32_t>(lamd::float_encode_f32(v, p.E, p.M));
    }

    template<int FMT>
    __device__ __forceinline__ uint32_t dec_t(const PackParams& p, const lamd::F32Codec& fc, uint32_t pat, uint32_t w)
    {
        if constexpr(FMT == 0)
        {
            if(p.sgn && w < 32)
            {
                const uint32_t s = 1u << (w - 1);
                return (pat ^ s) - s;
            }
            return pat;
        }
        else if constexpr(FMT == 1)
        {
            const uint32_t sign = (pat >> 18) << 31;
            if((pat & 0x3FC00u) == 0x3FC00u && (pat & 0x3FFu))
                return sign | 0x7FC00000u;
            return sign | ((pat & 0x3FFFFu) << 13);
        }
        else if constexpr(FMT == 2)
        {
            if((pat & 0x7C00u) == 0x7C00u && (pat & 0x3FFu))
                return ((pat >> 15) << 31) | 0x7FC00000u;
            return __float_as_uint(__half2float(__ushort_as_half(static_cast<unsigned short>(pat))));
        }
        else if constexpr(FMT == 3)
            return lamd::f32_decode_bf(fc, pat);
        else if constexpr(FMT == 5)
            return lamd::f32_decode_bf(lamd::f32_codec(4, 3), pat);
        else if constexpr(FMT == 6)
            return lamd::f32_decode_bf(lamd::f32_codec(5, 2), pat);
        else if(p.E <= 8 && p.M <= 23)
            return lamd::float_decode_f32(pat, p.E, p.M);
        else
            return lamd::f64_to_f32_bits(lamd::float_decode(pat, p.E, p.M));
    }

    // Warp smem slice: 32 lanes x VSTRIDE words of values, aliased by 32 lanes x wstride words
    // of the bit stream.  VSTRIDE = 36 keeps 16-byte value accesses conflict-free both in lane order
    // and in coalesced (global) order; wstride = w rounded up to odd keeps the per-lane word
    // accesses conflict-free.
    constexpr uint32_t VSTRIDE = 36;
    __host__ __device__ constexpr uint32_t wstride_of(uint32_t w)
    {
        return w | 1u;
    }
    // the word slice and the value slice alias: each kernel moves one of them into registers
    // (with a __syncwarp) before it writes the other
    __host__ __device__ constexpr uint32_t slice_words(uint32_t w)
    {
        return (32 * VSTRIDE > 32 * wstride_of(w) ? 32 * VSTRIDE : 32 * wstride_of(w)) + 4;
    }

    // value side, coalesced: chunk c (16 B) of the warp's 32 x 32 values <-> lane c/8, quad c%8
    __device__ __forceinline__ void values_g2s(const PackParams& p, uint32_t* vs, uint64_t warpE0, uint32_t lane,
                                               uint32_t liveLanes)
    {
        if(liveLanes == 32)
        {
            // full warp: all 8 loads in flight before the first shared-memory store (4 KB per
            // warp outstanding; a load->store loop would expose the HBM latency 8 times)
            uint4 x[8];
#pragma unroll
            for(int k = 0; k < 8; ++k)
                x[k] = __ldcs(reinterpret_cast<const uint4*>(val_addr(p, warpE0 + 4ull * (lane + 32 * k))));
#pragma unroll
            for(int k = 0; k < 8; ++k)
            {
                const uint32_t c = lane + 32 * k;
                *reinterpret_cast<uint4*>(vs + (c >> 3) * VSTRIDE + (c & 7) * 4) = x[k];
            }
            return;
        }
        const uint32_t chunks = liveLanes * 8;
        for(uint32_t c = lane; c < chunks; c += 32)
        {
            const uint64_t e = warpE0 + 4ull * c;
            const uint4 x = __ldcs(reinterpret_cast<const uint4*>(val_addr(p, e)));
            *reinterpret_cast<uint4*>(vs + (c >> 3) * VSTRIDE + (c & 7) * 4) = x;
        }
    }

    __device__ __forceinline__ void values_s2g(const PackParams& p, const uint32_t* vs, uint64_t warpE0, uint32_t lane,
                                               uint32_t liveLanes)
    {
        if(liveLanes == 32)
        {
#pragma unroll
            for(int k = 0; k < 8; ++k)
            {
                const uint32_t c = lane + 32 * k;
                __stcs(reinterpret_cast<uint4*>(val_addr(p, warpE0 + 4ull * c)),
                       *reinterpret_cast<const uint4*>(vs + (c >> 3) * VSTRIDE + (c & 7) * 4));
            }
            return;
        }
        const uint32_t chunks = liveLanes * 8;
        for(uint32_t c = lane; c < chunks; c += 32)
        {
            const uint64_t e = warpE0 + 4ull * c;
            __stcs(reinterpret_cast<uint4*>(val_addr(p, e)),
                   *reinterpret_cast<const uint4*>(vs + (c >> 3) * VSTRIDE + (c & 7) * 4));
        }
    }

    // pack: 32 values -> W words per thread (W = 0: runtime width p.w)
    // register bound: 3 CTAs/SM (80 registers) except the integer widths that spill there (even
    // W from 10 to 30 but 16); a (256, 4) bound on e8m10 had cost it 17% (profiles/README.md)
    __host__ __device__ constexpr int pack_minb(int W, int FMT)
    {
        return (FMT == 0 && W >= 10 && W % 2 == 0 && W != 16 && W != 32) || ((FMT == 3 || FMT >= 5) && W != 0) ? 2 : 3;
    }

    template<int W, int FMT>
    __global__ void __launch_bounds__(256, pack_minb(W, FMT)) k_pack32(const __grid_constant__ PackParams p)
    {
        extern __shared__ __align__(16) uint32_t psm[];
        const uint32_t w = W ? W : p.w;
        const uint32_t ws = wstride_of(w);
        const uint32_t lane = threadIdx.x & 31;
        uint32_t* vs = psm + (threadIdx.x >> 5) * slice_words(w);
        uint32_t* slice = vs; // aliases the value slice (see the __syncwarp before the word writes)
        const uint32_t mask = w >= 32 ? 0xFFFFFFFFu : ((1u << w) - 1u);
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        unsigned long long cnt = 0;
        const lamd::F32Codec fc = lamd::f32_codec(p.E, p.M); // FMT 3 only (dead code otherwise)
        const uint64_t gEnd = (p.groups + 31) / 32 * 32; // whole warps iterate together
        for(uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g - lane < gEnd; g += stride)
        {
            const uint64_t warpG = g - lane;
            const uint32_t liveLanes =
                static_cast<uint32_t>(p.groups > warpG ? (p.groups - warpG < 32 ? p.groups - warpG : 32) : 0);
            values_g2s(p, vs, p.begin + warpG * 32, lane, liveLanes);
            __syncwarp();
            const bool live = g < p.groups;
            uint32_t v[32];
            if(live)
            {
#pragma unroll
                for(int q = 0; q < 8; ++q)
                {
                    const uint4 x = *reinterpret_cast<const uint4*>(vs + lane * VSTRIDE + 4 * q);
                    v[4 * q] = x.x;
                    v[4 * q + 1] = x.y;
                    v[4 * q + 2] = x.z;
                    v[4 * q + 3] = x.w;
                }
            }
            // every lane's values are in registers: the word slice may now overwrite the value
            // slice (they alias, which halves the smem per warp and raises occupancy)
            __syncwarp();
            if(live)
            {
                uint32_t* my = slice + lane * ws;
                if constexpr(W != 0)
                {
                    // encode once per value (a value can straddle two words)
#pragma unroll
                    for(int i = 0; i < 32; ++i)
                        v[i] = enc_t<FMT>(p, fc, v[i], mask);
                    // word k = bits [32k, 32k+32): values floor(32k/W) .. floor((32k+31)/W)
#pragma unroll
                    for(int k = 0; k < W; ++k)
                    {
                        uint32_t word = 0;
#pragma unroll
                        for(int i = (32 * k) / W; i <= (32 * k + 31) / W && i < 32; ++i)
                        {
                            const int pos = i * W - 32 * k; // bit position of value i inside word k
                            const uint32_t e = v[i];
                            if(pos >= 0)
                                word |= e << pos;
                            else
                                word |= e >> (-pos);
                        }
                        my[k] = word;
                    }
                }
                else
                {
                    unsigned long long acc = 0;
                    uint32_t nb = 0, k = 0;
#pragma unroll
                    for(int i = 0; i < 32; ++i)
                    {
                        acc |= static_cast<unsigned long long>(enc_t<FMT>(p, fc, v[i], mask)) << nb;
                        nb += w;
                        if(nb >= 32)
                        {
                            my[k++] = static_cast<uint32_t>(acc);
                            acc >>= 32;
                            nb -= 32;
                        }
                    }
                }
                cnt += 32;
            }
            __syncwarp();
            // coalesced stream write of the warp's span (32 * w words)
            uint32_t* dst = reinterpret_cast<uint32_t*>(p.bits) + (p.begin + warpG * 32) / 32 * w;
            const uint32_t words = liveLanes * w;
            if(W != 0 && liveLanes == 32)
            {
#pragma unroll
                for(int k = 0; k < (W ? W : 1); ++k)
                {
                    const uint32_t q = lane + 32 * k;
                    __stcs(dst + q, slice[(q / w) * ws + (q % w)]);
                }
            }
            else
                for(uint32_t q = lane; q < words; q += 32)
                    __stcs(dst + q, slice[(q / w) * ws + (q % w)]);
            __syncwarp();
        }
        fac_flush(p, cnt);
    }

    // unpack: W words -> 32 values per thread
    // unpack: 3 CTAs/SM (80 registers) except the widths that spill there
    __host__ __device__ constexpr int unpack_minb(int W, int FMT)
    {
        return ((FMT == 0 || FMT == 3) && (W == 24 || W == 26 || W == 28 || W == 30)) || (FMT == 3 && (W == 14 || W == 27))
                || (FMT == 0 && W == 6)
            ? 2
            : 3;
    }

    template<int W, int FMT>
    __global__ void __launch_bounds__(256, unpack_minb(W, FMT)) k_unpack32(const __grid_constant__ PackParams p)
    {
        extern __shared__ __align__(16) uint32_t psm[];
        const uint32_t w = W ? W : p.w;
        const uint32_t ws = wstride_of(w);
        const uint32_t lane = threadIdx.x & 31;
        uint32_t* vs = psm + (threadIdx.x >> 5) * slice_words(w);
        uint32_t* slice = vs; // aliases the value slice (see the __syncwarp before the value writes)
        const uint32_t mask = w >= 32 ? 0xFFFFFFFFu : ((1u << w) - 1u);
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        unsigned long long cnt = 0;
        const lamd::F32Codec fc = lamd::f32_codec(p.E, p.M); // FMT 3 only (dead code otherwise)
        const uint64_t gEnd = (p.groups + 31) / 32 * 32;
        auto liveOf = [&](uint64_t warpG) -> uint32_t
        {
            return static_cast<uint32_t>(p.groups > warpG ? (p.groups - warpG < 32 ? p.groups - warpG : 32) : 0);
        };
        auto words_at = [&](uint64_t warpG)
        { return reinterpret_cast<const uint32_t*>(p.bits) + (p.begin + warpG * 32) / 32 * w; };
        // full warps with a compile-time width: the next span's W coalesced word loads are issued
        // before the current span is decoded and stored (software pipeline; for narrow widths a
        // span is only W * 128 bytes of loads per warp, too little to cover the latency alone)
        // (widths <= 8 only: wider spans already carry enough bytes, and the extra registers
        // would spill under the 80-register bound)
        constexpr bool PF = W != 0 && W <= 8;
        uint32_t tn[W ? W : 1];
        const uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        bool pre = PF && g0 - lane < gEnd && liveOf(g0 - lane) == 32;
        if(pre)
        {
#pragma unroll
            for(int k = 0; k < (W ? W : 1); ++k)
                tn[k] = __ldcs(words_at(g0 - lane) + lane + 32 * k);
        }
        for(uint64_t g = g0; g - lane < gEnd; g += stride)
        {
            const uint64_t warpG = g - lane;
            const uint32_t liveLanes = liveOf(warpG);
            const uint32_t* srcw = words_at(warpG);
            const uint32_t words = liveLanes * w;
            if(!PF && W != 0 && liveLanes == 32)
            {
                // full warp: the W coalesced word loads are all in flight before any smem store
                uint32_t t[W ? W : 1];
#pragma unroll
                for(int k = 0; k < (W ? W : 1); ++k)
                    t[k] = __ldcs(srcw + lane + 32 * k);
#pragma unroll
                for(int k = 0; k < (W ? W : 1); ++k)
                {
                    const uint32_t q = lane + 32 * k;
                    slice[(q / w) * ws + (q % w)] = t[k];
                }
            }
            else if(pre)
            {
#pragma unroll
                for(int k = 0; k < (W ? W : 1); ++k)
                {
                    const uint32_t q = lane + 32 * k;
                    slice[(q / w) * ws + (q % w)] = tn[k];
                }
                const uint64_t nextG = warpG + stride;
                pre = PF && nextG < gEnd && liveOf(nextG) == 32;
                if(pre)
                {
#pragma unroll
                    for(int k = 0; k < (W ? W : 1); ++k)
                        tn[k] = __ldcs(words_at(nextG) + lane + 32 * k);
                }
            }
            else
                for(uint32_t q = lane; q < words; q += 32)
                    slice[(q / w) * ws + (q % w)] = __ldcs(srcw + q);
            __syncwarp();
            const bool live = g < p.groups;
            uint32_t v[32];
            if(live)
            {
                const uint32_t* my = slice + lane * ws;
                if constexpr(W != 0)
                {
                    uint32_t wd[W];
#pragma unroll
                    for(int k = 0; k < W; ++k)
                        wd[k] = my[k];
#pragma unroll
                    for(int i = 0; i < 32; ++i)
                    {
                        const int bit = i * W, k = bit >> 5, sh = bit & 31;
                        uint32_t pat = wd[k] >> sh;
                        if(sh + W > 32)
                            pat |= wd[k + 1] << (32 - sh);
                        v[i] = dec_t<FMT>(p, fc, pat & mask, w);
                    }
                }
                else
                {
                    unsigned long long acc = my[0];
                    uint32_t nb = 32, k = 1;
#pragma unroll
                    for(int i = 0; i < 32; ++i)
                    {
                        if(nb < w)
                        {
                            acc |= static_cast<unsigned long long>(my[k < w ? k : w - 1]) << nb;
                            ++k;
                            nb += 32;
                        }
                        v[i] = dec_t<FMT>(p, fc, static_cast<uint32_t>(acc) & mask, w);
                        acc >>= w;
                        nb -= w;
                    }
                }
            }
            // every lane's words are consumed: the value slice may now overwrite the word slice
            __syncwarp();
            if(live)
            {
#pragma unroll
                for(int q = 0; q < 8; ++q)
                    *reinterpret_cast<uint4*>(vs + lane * VSTRIDE + 4 * q)
                        = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                cnt += 32;
            }
            __syncwarp();
            values_s2g(p, vs, p.begin + warpG * 32, lane, liveLanes);
            __syncwarp();
        }
        fac_flush(p, cnt);
    }

    // ---- record-contiguous side <-> bit streams in one pass ----------------------------------
    // AoS (packed, 4-byte leaves) or AoSoA<L> (L | 32) against BitpackIntSoA / BitpackFloatSoA
    // with one width for every leaf (computed.cpp:48-222).  A CTA owns 1024 consecutive records:
    // their record bytes are one contiguous region (28 KB for the n-body record), moved with
    // 16-byte coalesced accesses into shared memory padded by one word per 32 records.  Warp l
    // packs leaf l, lane g the 32 records of group g (its W words of stream l): the value reads
    // are conflict-free because the group padding puts the 32 lanes on 32 banks.  Every record
    // byte and every stream word crosses HBM exactly once.
    struct RecPackParams
    {
        unsigned long long rec;     // record region of element 0 (AoS stream / AoSoA block 0)
        unsigned long long bits[8]; // bit stream of each leaf (word 0 = element 0)
        unsigned long long begin;   // first element (multiple of 32 and of lanes)
        unsigned long long groups;  // groups of 32 elements
        uint32_t nl, lanes, lsh, sgnMask;
        uint32_t w, E, M;
        uint32_t gmag; // ceil(2^24 / (32 nl)): region word -> group by multiply-shift (exact below 2^13 words)
    };

    // region word w (record e, leaf l) sits at smem word w + e / 32 (one pad word per group of 32
    // records); lane `g` of warp `l` reads record i of its group at base + (i >> lsh) * nl * L + (i & (L - 1))
    __device__ __forceinline__ uint32_t rec_base(const RecPackParams& q, uint32_t lane, uint32_t wp)
    {
        return lane * (32 * q.nl + 1) + wp * q.lanes;
    }

    __device__ __forceinline__ uint32_t pad_of(const RecPackParams& q, uint32_t w0)
    {
        return (w0 * q.gmag) >> 24;
    }

    // region word `w0 + c` (c = 0..3 of a 16-byte chunk) lives at smem w0 + c + group; the four
    // components are visited in a lane-rotated order so each STS/LDS.32 hits 32 distinct banks
    __device__ __forceinline__ uint32_t comp(const uint4& x, uint32_t c)
    {
        return c == 0 ? x.x : c == 1 ? x.y : c == 2 ? x.z : x.w;
    }
#ifndef LAMB_REC_ROTATE
#define LAMB_REC_ROTATE 0
#endif
    // rotated: conflict-free STS/LDS.32 at 3 selects per word; plain: 4-way conflicts (MIO
    // wavefronts, not issue slots -- the kernels are issue-bound, so plain measured faster)
#if LAMB_REC_ROTATE
#define STORE4(d, vec)                                                                                                   \
    _Pragma("unroll") for(uint32_t j = 0; j < 4; ++j)                                                                  \
    {                                                                                                                  \
        const uint32_t c = (j + rot) & 3;                                                                              \
        (d)[c] = comp((vec), c);                                                                                         \
    }
#define LOAD4(r, s)                                                                                                    \
    _Pragma("unroll") for(uint32_t j = 0; j < 4; ++j)                                                                  \
    {                                                                                                                  \
        const uint32_t c = (j + rot) & 3;                                                                              \
        (r)[c] = (s)[c];                                                                                               \
    }
#else
#define STORE4(d, vec)                                                                                                   \
    {                                                                                                                  \
        (void)rot;                                                                                                     \
        (d)[0] = (vec).x;                                                                                                \
        (d)[1] = (vec).y;                                                                                                \
        (d)[2] = (vec).z;                                                                                                \
        (d)[3] = (vec).w;                                                                                                \
    }
#define LOAD4(r, s)                                                                                                    \
    {                                                                                                                  \
        (void)rot;                                                                                                     \
        (r)[0] = (s)[0];                                                                                               \
        (r)[1] = (s)[1];                                                                                               \
        (r)[2] = (s)[2];                                                                                               \
        (r)[3] = (s)[3];                                                                                               \
    }
#endif

    template<int W, int FMT>
    __global__ void __launch_bounds__(256) k_rec_pack(const __grid_constant__ RecPackParams q)
    {
        extern __shared__ __align__(16) uint32_t psm[];
        const uint32_t w = W ? W : q.w;
        const uint32_t ws = wstride_of(w);
        const uint32_t lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
        const uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * 32;
        const uint32_t ng = static_cast<uint32_t>(q.groups - g0 < 32 ? q.groups - g0 : 32);
        const uint64_t e0 = q.begin + g0 * 32;
        const uint4* src = reinterpret_cast<const uint4*>(q.rec + e0 * q.nl * 4);
        const uint32_t chunks = ng * 8 * q.nl;
        const uint32_t rot = lane >> 3;
        if(ng == 32)
        {
            uint4 x[8];
#pragma unroll
            for(int k = 0; k < 8; ++k)
                if(k < static_cast<int>(q.nl))
                    x[k] = __ldcs(src + threadIdx.x + 256 * k);
#pragma unroll
            for(int k = 0; k < 8; ++k)
                if(k < static_cast<int>(q.nl))
                {
                    const uint32_t w0 = 4 * (threadIdx.x + 256 * k);
                    uint32_t* d = psm + w0 + pad_of(q, w0);
                    STORE4(d, x[k]);
                }
        }
        else
            for(uint32_t ch = threadIdx.x; ch < chunks; ch += 256)
            {
                const uint4 x = __ldcs(src + ch);
                const uint32_t w0 = 4 * ch;
                uint32_t* d = psm + w0 + pad_of(q, w0);
                STORE4(d, x);
            }
        __syncthreads();
        const bool live = wp < q.nl && lane < ng;
        uint32_t words[W ? W : 32];
        if(live)
        {
            PackParams p{};
            p.E = q.E;
            p.M = q.M;
            const lamd::F32Codec fc = lamd::f32_codec(q.E, q.M);
            const uint32_t mask = w >= 32 ? 0xFFFFFFFFu : ((1u << w) - 1u);
            uint32_t v[32];
            const uint32_t* pv = psm + rec_base(q, lane, wp);
            if(q.lanes == 1)
            {
#pragma unroll
                for(int i = 0; i < 32; ++i)
                    v[i] = pv[i * q.nl];
            }
            else
            {
                const uint32_t nlL = q.nl * q.lanes, lm = q.lanes - 1;
#pragma unroll
                for(int i = 0; i < 32; ++i)
                    v[i] = pv[(i >> q.lsh) * nlL + (i & lm)];
            }
#pragma unroll
            for(int i = 0; i < 32; ++i)
                v[i] = enc_t<FMT>(p, fc, v[i], mask);
            if constexpr(W != 0)
            {
#pragma unroll
                for(int k = 0; k < W; ++k)
                {
                    uint32_t word = 0;
#pragma unroll
                    for(int i = (32 * k) / W; i <= (32 * k + 31) / W && i < 32; ++i)
                    {
                        const int pos = i * W - 32 * k;
                        word |= pos >= 0 ? v[i] << pos : v[i] >> (-pos);
                    }
                    words[k] = word;
                }
            }
            else
            {
                unsigned long long acc = 0;
                uint32_t nb = 0, k = 0;
#pragma unroll
                for(int i = 0; i < 32; ++i)
                {
                    acc |= static_cast<unsigned long long>(v[i]) << nb;
                    nb += w;
                    if(nb >= 32)
                    {
                        words[k++] = static_cast<uint32_t>(acc);
                        acc >>= 32;
                        nb -= 32;
                    }
                }
            }
        }
        __syncthreads(); // the region is consumed: the word slices may overwrite it
        if(wp < q.nl)
        {
            uint32_t* slice = psm + wp * 32 * ws;
            if(live)
            {
#pragma unroll
                for(int k = 0; k < (W ? W : 32); ++k)
                    if(W || k < static_cast<int>(w))
                        slice[lane * ws + k] = words[k];
            }
            __syncwarp();
            uint32_t* dst = reinterpret_cast<uint32_t*>(q.bits[wp]) + (q.begin / 32 + g0) * w;
            const uint32_t nw = ng * w;
            for(uint32_t t = lane; t < nw; t += 32)
                __stcs(dst + t, slice[(t / w) * ws + (t % w)]);
        }
    }

    template<int W, int FMT>
    __global__ void __launch_bounds__(256) k_rec_unpack(const __grid_constant__ RecPackParams q)
    {
        extern __shared__ __align__(16) uint32_t psm[];
        const uint32_t w = W ? W : q.w;
        const uint32_t ws = wstride_of(w);
        const uint32_t lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
        const uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * 32;
        const uint32_t ng = static_cast<uint32_t>(q.groups - g0 < 32 ? q.groups - g0 : 32);
        const uint64_t e0 = q.begin + g0 * 32;
        const bool live = wp < q.nl && lane < ng;
        uint32_t v[32];
        if(wp < q.nl)
        {
            uint32_t* slice = psm + wp * 32 * ws;
            const uint32_t* srcw = reinterpret_cast<const uint32_t*>(q.bits[wp]) + (q.begin / 32 + g0) * w;
            const uint32_t nw = ng * w;
            if(W != 0 && ng == 32)
            {
                uint32_t t[W ? W : 1];
#pragma unroll
                for(int k = 0; k < (W ? W : 1); ++k)
                    t[k] = __ldcs(srcw + lane + 32 * k);
#pragma unroll
                for(int k = 0; k < (W ? W : 1); ++k)
                {
                    const uint32_t x = lane + 32 * k;
                    slice[(x / w) * ws + (x % w)] = t[k];
                }
            }
            else
                for(uint32_t x = lane; x < nw; x += 32)
                    slice[(x / w) * ws + (x % w)] = __ldcs(srcw + x);
            __syncwarp();
            if(live)
            {
                PackParams p{};
                p.E = q.E;
                p.M = q.M;
                const lamd::F32Codec fc = lamd::f32_codec(q.E, q.M);
                p.sgn = (q.sgnMask >> wp) & 1u;
                const uint32_t mask = w >= 32 ? 0xFFFFFFFFu : ((1u << w) - 1u);
                const uint32_t* my = slice + lane * ws;
                if constexpr(W != 0)
                {
                    uint32_t wd[W];
#pragma unroll
                    for(int k = 0; k < W; ++k)
                        wd[k] = my[k];
#pragma unroll
                    for(int i = 0; i < 32; ++i)
                    {
                        const int bit = i * W, k = bit >> 5, sh = bit & 31;
                        uint32_t pat = wd[k] >> sh;
                        if(sh + W > 32)
                            pat |= wd[k + 1] << (32 - sh);
                        v[i] = dec_t<FMT>(p, fc, pat & mask, w);
                    }
                }
                else
                {
                    unsigned long long acc = my[0];
                    uint32_t nb = 32, k = 1;
#pragma unroll
                    for(int i = 0; i < 32; ++i)
                    {
                        if(nb < w)
                        {
                            acc |= static_cast<unsigned long long>(my[k < w ? k : w - 1]) << nb;
                            ++k;
                            nb += 32;
                        }
                        v[i] = dec_t<FMT>(p, fc, static_cast<uint32_t>(acc) & mask, w);
                        acc >>= w;
                        nb -= w;
                    }
                }
            }
        }
        __syncthreads(); // every slice is consumed: the record region may overwrite them
        if(live)
        {
            uint32_t* pv = psm + rec_base(q, lane, wp);
            if(q.lanes == 1)
            {
#pragma unroll
                for(int i = 0; i < 32; ++i)
                    pv[i * q.nl] = v[i];
            }
            else
            {
                const uint32_t nlL = q.nl * q.lanes, lm = q.lanes - 1;
#pragma unroll
                for(int i = 0; i < 32; ++i)
                    pv[(i >> q.lsh) * nlL + (i & lm)] = v[i];
            }
        }
        __syncthreads();
        uint4* dst = reinterpret_cast<uint4*>(q.rec + e0 * q.nl * 4);
        const uint32_t chunks = ng * 8 * q.nl;
        const uint32_t rot = lane >> 3;
        for(uint32_t ch = threadIdx.x; ch < chunks; ch += 256)
        {
            const uint32_t w0 = 4 * ch;
            const uint32_t* s = psm + w0 + pad_of(q, w0);
            uint32_t r[4];
            LOAD4(r, s);
            __stcs(dst + ch, make_uint4(r[0], r[1], r[2], r[3]));
        }
    }

    template<int W, int FMT>
    static void launch_rec(const RecPackParams& q, bool pack, unsigned grid, size_t smem, cudaStream_t s)
    {
        if(pack)
        {
            lam_cuda_check(opt_in_smem(reinterpret_cast<const void*>(k_rec_pack<W, FMT>), smem), "opt_in_smem");
            k_rec_pack<W, FMT><<<grid, 256, smem, s>>>(q);
        }
        else
        {
            lam_cuda_check(opt_in_smem(reinterpret_cast<const void*>(k_rec_unpack<W, FMT>), smem), "opt_in_smem");
            k_rec_unpack<W, FMT><<<grid, 256, smem, s>>>(q);
        }
    }

    template<int... Ws>
    static bool dispatch_rec_int(int w, const RecPackParams& q, bool pack, unsigned grid, size_t smem, cudaStream_t s,
                                 std::integer_sequence<int, Ws...>)
    {
        bool hit = false;
        ((w == Ws + 1 ? (launch_rec<Ws + 1, 0>(q, pack, grid, smem, s), hit = true) : false), ...);
        return hit;
    }

    // kind: 0 int, 1 float
    static int envNum32(const char* name, int dflt)
    {
        const char* e = std::getenv(name);
        return e ? std::atoi(e) : dflt;
    }

    bool rec_pack(const RecPackParams& q, uint32_t kind, bool pack, cudaStream_t s)
    {
        if(q.groups == 0 || q.w < 1 || q.w > 32 || q.nl < 1 || q.nl > 8 || q.begin % 32
           || (q.lanes != 1 && (32 % q.lanes || q.begin % q.lanes)))
            return false;
        const uint64_t blocks = (q.groups + 31) / 32;
        if(blocks > 0x7FFFFFFFull)
            return false;
        const size_t region = 1024 * q.nl + 32, slices = static_cast<size_t>(q.nl) * 32 * wstride_of(q.w);
        const size_t smem = (region > slices ? region : slices) * sizeof(uint32_t);
        const unsigned grid = static_cast<unsigned>(blocks);
        if(kind == 0)
            dispatch_rec_int(static_cast<int>(q.w), q, pack, grid, smem, s, std::make_integer_sequence<int, 32>{});
        else if(q.E == 8 && q.M == 10)
            launch_rec<19, 1>(q, pack, grid, smem, s);
        else if(q.E == 5 && q.M == 10)
            launch_rec<16, 2>(q, pack, grid, smem, s);
        else if(q.E <= 8 && q.M <= 23)
        {
            // the branch-free f32 codec (FMT 3); compile-time W for the 8- and 16-bit formats
            if(q.E == 4 && q.M == 3 && envNum32("LAMB_PACK_CONSTFMT", 1))
                launch_rec<8, 5>(q, pack, grid, smem, s);
            else if(q.E == 5 && q.M == 2 && envNum32("LAMB_PACK_CONSTFMT", 1))
                launch_rec<8, 6>(q, pack, grid, smem, s);
            else if(q.w == 8)
                launch_rec<8, 3>(q, pack, grid, smem, s);
            else if(q.w == 16)
                launch_rec<16, 3>(q, pack, grid, smem, s);
            else
                launch_rec<0, 3>(q, pack, grid, smem, s);
        }
        else
            launch_rec<0, 4>(q, pack, grid, smem, s);
        count_launch();
        lam_cuda_check(cudaGetLastError(), "kernel launch");
        return true;
    }

    // grid-stride kernels: never launch more CTAs than can be resident at once (a partial
    // second wave would run a full share of the work late)
    // grid-stride with 32 CTAs per SM (8-10 waves of the resident count): measured best across
    // the C3 widths (8: 84-98%, 32: 84-103%, 128 and uncapped: some widths drop to 76-83%)
    template<typename K>
    static unsigned resident_grid(K, unsigned want, size_t, bool)
    {
        return stream_grid(want, "LAMB_PACK_CTAS", 32);
    }

    template<int W, int FMT>
    static void launch_pack(const PackParams& p, bool pack, unsigned grid, size_t smem, cudaStream_t s)
    {
        // opt in to > 48 KB of dynamic shared memory once per instantiation, size and device
        // (one launch per leaf: a launch over several leaves through an indexed parameter array
        // moved the parameter reads out of the constant bank and cost the C3 kernels up to 8%)
        if(pack)
        {
            lam_cuda_check(opt_in_smem(reinterpret_cast<const void*>(k_pack32<W, FMT>), smem), "opt_in_smem");
            k_pack32<W, FMT><<<resident_grid(k_pack32<W, FMT>, grid, smem, false), 256, smem, s>>>(p);
        }
        else
        {
            lam_cuda_check(opt_in_smem(reinterpret_cast<const void*>(k_unpack32<W, FMT>), smem), "opt_in_smem");
            k_unpack32<W, FMT><<<resident_grid(k_unpack32<W, FMT>, grid, smem, false), 256, smem, s>>>(p);
        }
    }

    template<int... Ws>
    static bool dispatch_int(int w, const PackParams& p, bool pack, unsigned grid, size_t smem, cudaStream_t s,
                             std::integer_sequence<int, Ws...>)
    {
        bool hit = false;
        ((w == Ws + 1 ? (launch_pack<Ws + 1, 0>(p, pack, grid, smem, s), hit = true) : false), ...);
        return hit;
    }

    // any other (E, M) with 1 + E + M <= 32: compile-time width, runtime format
    template<int... Ws>
    static bool dispatch_flt(int w, const PackParams& p, bool pack, unsigned grid, size_t smem, cudaStream_t s,
                             std::integer_sequence<int, Ws...>)
    {
        bool hit = false;
        ((w == Ws + 2 ? (launch_pack<Ws + 2, 3>(p, pack, grid, smem, s), hit = true) : false), ...);
        return hit;
    }

    // ---- bit stream -> bit stream (different widths / formats, or the same computed layout) ----
    // copyView reads each value from the source field (decode / sign-extend) and writes it to the
    // destination field (encode / truncate); a thread owns 32 values = ws source words and wd
    // destination words.  The warp's 32*ws source words and 32*wd destination words are
    // contiguous: they move with coalesced accesses through lane rows of stride ws|1 / wd|1
    // (conflict-free), so every bit crosses HBM once, without the SoA scratch round trip.
    __global__ void __launch_bounds__(256) k_repack32(const __grid_constant__ RepackParams p)
    {
        extern __shared__ __align__(16) uint32_t rsm[];
        const uint32_t ws = p.ws, wd = p.wd, wsp = ws | 1u, wdp = wd | 1u;
        const uint32_t lane = threadIdx.x & 31;
        uint32_t* srow = rsm + (threadIdx.x >> 5) * 32 * (wsp + wdp);
        uint32_t* drow = srow + 32 * wsp;
        const uint32_t smag = static_cast<uint32_t>(((1ull << 32) + ws - 1) / ws);
        const uint32_t dmag = static_cast<uint32_t>(((1ull << 32) + wd - 1) / wd);
        const uint32_t smask = ws >= 32 ? 0xFFFFFFFFu : ((1u << ws) - 1u);
        const uint32_t dmask = wd >= 32 ? 0xFFFFFFFFu : ((1u << wd) - 1u);
        const lamd::F32Codec cs = lamd::f32_codec(p.sE, p.sM), cd = lamd::f32_codec(p.dE, p.dM);
        const uint32_t* src = reinterpret_cast<const uint32_t*>(p.src);
        uint32_t* dst = reinterpret_cast<uint32_t*>(p.dst);
        const uint64_t gEnd = (p.groups + 31) / 32 * 32; // whole warps iterate together
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        for(uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g - lane < gEnd; g += stride)
        {
            const uint64_t warpG = g - lane;
            const uint32_t live = static_cast<uint32_t>(p.groups > warpG ? (p.groups - warpG < 32 ? p.groups - warpG : 32) : 0);
            const uint32_t* ws0 = src + (p.begin / 32 + warpG) * ws;
            // t / ws by a multiply-high (exact for t < 1024, ws <= 32)
            for(uint32_t t = lane; t < live * ws; t += 32)
            {
                const uint32_t r = __umulhi(t, smag);
                srow[r * wsp + (t - r * ws)] = __ldcs(ws0 + t);
            }
            __syncwarp();
            if(lane < live)
            {
                const uint32_t* my = srow + lane * wsp;
                uint32_t* out = drow + lane * wdp;
                unsigned long long acc = my[0], oacc = 0;
                uint32_t nb = 32, k = 1, onb = 0, ok = 0;
#pragma unroll 4
                for(int i = 0; i < 32; ++i)
                {
                    if(nb < ws)
                    {
                        acc |= static_cast<unsigned long long>(my[k < ws ? k : ws - 1]) << nb;
                        ++k;
                        nb += 32;
                    }
                    uint32_t v = static_cast<uint32_t>(acc) & smask;
                    acc >>= ws;
                    nb -= ws;
                    if(p.kind)
                        v = lamd::f32_encode_bf(cd, lamd::f32_decode_bf(cs, v));
                    else
                    {
                        if(p.ssgn && ws < 32)
                        {
                            const uint32_t sb = 1u << (ws - 1);
                            v = (v ^ sb) - sb;
                        }
                        v &= dmask;
                    }
                    oacc |= static_cast<unsigned long long>(v) << onb;
                    onb += wd;
                    if(onb >= 32)
                    {
                        out[ok++] = static_cast<uint32_t>(oacc);
                        oacc >>= 32;
                        onb -= 32;
                    }
                }
            }
            __syncwarp();
            uint32_t* wd0 = dst + (p.begin / 32 + warpG) * wd;
            for(uint32_t t = lane; t < live * wd; t += 32)
            {
                const uint32_t r = __umulhi(t, dmag);
                __stcs(wd0 + t, drow[r * wdp + (t - r * wd)]);
            }
            __syncwarp();
        }
    }

    // minifloat -> minifloat with both formats compile-time (FMT 1 e8m10 / 2 e5m10 / 5 e4m3 /
    // 6 e5m2): the same warp structure as k_repack32, widths and codecs fully unrolled
    template<int FS>
    __device__ __forceinline__ uint32_t rp_dec(uint32_t pat)
    {
        if constexpr(FS == 1)
        {
            const uint32_t sign = (pat >> 18) << 31;
            if((pat & 0x3FC00u) == 0x3FC00u && (pat & 0x3FFu))
                return sign | 0x7FC00000u;
            return sign | ((pat & 0x3FFFFu) << 13);
        }
        else if constexpr(FS == 2)
        {
            if((pat & 0x7C00u) == 0x7C00u && (pat & 0x3FFu))
                return ((pat >> 15) << 31) | 0x7FC00000u;
            return __float_as_uint(__half2float(__ushort_as_half(static_cast<unsigned short>(pat))));
        }
        else if constexpr(FS == 5)
            return lamd::f32_decode_bf(lamd::f32_codec(4, 3), pat);
        else
            return lamd::f32_decode_bf(lamd::f32_codec(5, 2), pat);
    }
    template<int FD>
    __device__ __forceinline__ uint32_t rp_enc(uint32_t v)
    {
        if constexpr(FD == 1)
            return lamd::encode_e8m10_f32(v);
        else if constexpr(FD == 2)
            return lamd::encode_e5m10_f32(v);
        else if constexpr(FD == 5)
            return lamd::f32_encode_bf(lamd::f32_codec(4, 3), v);
        else
            return lamd::f32_encode_bf(lamd::f32_codec(5, 2), v);
    }
    template<int FS, int FD>
    __global__ void __launch_bounds__(256) k_repack_flt(const __grid_constant__ RepackParams p)
    {
        constexpr uint32_t WS = FS == 1 ? 19 : FS == 2 ? 16 : 8, WD = FD == 1 ? 19 : FD == 2 ? 16 : 8;
        constexpr uint32_t WSP = WS | 1u, WDP = WD | 1u;
        extern __shared__ __align__(16) uint32_t fsm[];
        const uint32_t lane = threadIdx.x & 31;
        uint32_t* srow = fsm + (threadIdx.x >> 5) * 32 * (WSP + WDP);
        uint32_t* drow = srow + 32 * WSP;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(p.src);
        uint32_t* dst = reinterpret_cast<uint32_t*>(p.dst);
        const uint64_t gEnd = (p.groups + 31) / 32 * 32;
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        for(uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g - lane < gEnd; g += stride)
        {
            const uint64_t warpG = g - lane;
            const uint32_t live = static_cast<uint32_t>(p.groups > warpG ? (p.groups - warpG < 32 ? p.groups - warpG : 32) : 0);
            const uint32_t* ws0 = src + (p.begin / 32 + warpG) * WS;
            for(uint32_t t = lane; t < live * WS; t += 32)
                srow[(t / WS) * WSP + t % WS] = __ldcs(ws0 + t);
            __syncwarp();
            if(lane < live)
            {
                const uint32_t* my = srow + lane * WSP;
                uint32_t wv[WS], ov[WD];
#pragma unroll
                for(uint32_t k = 0; k < WS; ++k)
                    wv[k] = my[k];
#pragma unroll
                for(uint32_t k = 0; k < WD; ++k)
                    ov[k] = 0;
#pragma unroll
                for(uint32_t i = 0; i < 32; ++i)
                {
                    const uint32_t bit = i * WS, k = bit >> 5, sh = bit & 31;
                    uint32_t pat = wv[k] >> sh;
                    if(sh + WS > 32)
                        pat |= wv[k + 1] << (32 - sh);
                    pat &= (1u << WS) - 1u;
                    uint32_t e;
                    if constexpr(FS == FD)
                    {
                        // same format: decode then encode is the identity (every such minifloat is an
                        // exact f32) except that a NaN comes back as the canonical quiet NaN
                        // (sign | all-ones exponent | 1 << (M - 1), bitpack.cpp:107-115)
                        constexpr uint32_t M = FS == 1 || FS == 2 ? 10 : FS == 5 ? 3 : 2;
                        constexpr uint32_t EXP = ((1u << (WS - 1)) - 1u) & ~((1u << M) - 1u);
                        constexpr uint32_t MAN = (1u << M) - 1u;
                        const bool nan = (pat & EXP) == EXP && (pat & MAN);
                        e = nan ? ((pat & (1u << (WS - 1))) | EXP | (1u << (M - 1))) : pat;
                    }
                    else
                        e = rp_enc<FD>(rp_dec<FS>(pat));
                    const uint32_t ob = i * WD, ok = ob >> 5, osh = ob & 31;
                    ov[ok] |= e << osh;
                    if(osh + WD > 32)
                        ov[ok + 1] |= e >> (32 - osh);
                }
                uint32_t* out = drow + lane * WDP;
#pragma unroll
                for(uint32_t k = 0; k < WD; ++k)
                    out[k] = ov[k];
            }
            __syncwarp();
            uint32_t* wd0 = dst + (p.begin / 32 + warpG) * WD;
            for(uint32_t t = lane; t < live * WD; t += 32)
                __stcs(wd0 + t, drow[(t / WD) * WDP + t % WD]);
            __syncwarp();
        }
    }

    // the compile-time format code of (E, M), or 0
    static int fast_fmt(uint32_t E, uint32_t M)
    {
        return E == 8 && M == 10 ? 1 : E == 5 && M == 10 ? 2 : E == 4 && M == 3 ? 5 : E == 5 && M == 2 ? 6 : 0;
    }

    template<int FS, int FD>
    static void launch_repack_flt(const RepackParams& p, cudaStream_t s)
    {
        constexpr uint32_t WS = FS == 1 ? 19 : FS == 2 ? 16 : 8, WD = FD == 1 ? 19 : FD == 2 ? 16 : 8;
        const size_t smem = static_cast<size_t>(8) * 32 * ((WS | 1u) + (WD | 1u)) * sizeof(uint32_t);
        lam_cuda_check(opt_in_smem(reinterpret_cast<const void*>(k_repack_flt<FS, FD>), smem), "opt_in_smem");
        k_repack_flt<FS, FD><<<stream_grid((p.groups + 255) / 256, "LAMB_PACK_CTAS", 32), 256, smem, s>>>(p);
    }

    template<int FS>
    static bool dispatch_repack_flt_d(int fd, const RepackParams& p, cudaStream_t s)
    {
        switch(fd)
        {
        case 1: launch_repack_flt<FS, 1>(p, s); return true;
        case 2: launch_repack_flt<FS, 2>(p, s); return true;
        case 5: launch_repack_flt<FS, 5>(p, s); return true;
        case 6: launch_repack_flt<FS, 6>(p, s); return true;
        default: return false;
        }
    }

    bool repack_flt_fast(const RepackParams& p, cudaStream_t s)
    {
        const int fs = fast_fmt(p.sE, p.sM), fd = fast_fmt(p.dE, p.dM);
        if(p.groups == 0 || !fs || !fd)
            return false;
        bool ok = false;
        switch(fs)
        {
        case 1: ok = dispatch_repack_flt_d<1>(fd, p, s); break;
        case 2: ok = dispatch_repack_flt_d<2>(fd, p, s); break;
        case 5: ok = dispatch_repack_flt_d<5>(fd, p, s); break;
        case 6: ok = dispatch_repack_flt_d<6>(fd, p, s); break;
        default: return false;
        }
        if(!ok)
            return false;
        count_launch();
        lam_cuda_check(cudaGetLastError(), "kernel launch");
        return true;
    }

    bool repack32(const RepackParams& p, cudaStream_t s)
    {
        if(p.groups == 0 || p.ws < 1 || p.ws > 32 || p.wd < 1 || p.wd > 32)
            return false;
        const size_t smem = static_cast<size_t>(8) * 32 * ((p.ws | 1u) + (p.wd | 1u)) * sizeof(uint32_t);
        lam_cuda_check(opt_in_smem(reinterpret_cast<const void*>(k_repack32), smem), "opt_in_smem");
        const unsigned grid = stream_grid((p.groups + 255) / 256, "LAMB_PACK_CTAS", 32);
        k_repack32<<<grid, 256, smem, s>>>(p);
        count_launch();
        lam_cuda_check(cudaGetLastError(), "kernel launch");
        return true;
    }

    bool pack32(const PackParams& p, bool pack, cudaStream_t s)
    {
        if(p.groups == 0 || p.w < 1 || p.w > 32)
            return false;
        const uint64_t want = (p.groups + 255) / 256;
        const unsigned grid = static_cast<unsigned>(want < 0x7FFFFFFFull ? want : 0x7FFFFFFFull);
        const size_t smem = 8 * slice_words(p.w) * sizeof(uint32_t);
        if(p.kind == 0)
            dispatch_int(static_cast<int>(p.w), p, pack, grid, smem, s, std::make_integer_sequence<int, 32>{});
        else if(p.E == 8 && p.M == 10)
            launch_pack<19, 1>(p, pack, grid, smem, s);
        else if(p.E == 5 && p.M == 10)
            launch_pack<16, 2>(p, pack, grid, smem, s);
        else if(p.E > 8 || p.M > 23
                || !((p.E == 4 && p.M == 3 && envNum32("LAMB_PACK_CONSTFMT", 1) ? (launch_pack<8, 5>(p, pack, grid, smem, s), true)
                      : p.E == 5 && p.M == 2 && envNum32("LAMB_PACK_CONSTFMT", 1) ? (launch_pack<8, 6>(p, pack, grid, smem, s), true)
                                                                                   : false)
                     || dispatch_flt(static_cast<int>(p.w), p, pack, grid, smem, s, std::make_integer_sequence<int, 31>{})))
            launch_pack<0, 4>(p, pack, grid, smem, s);
        count_launch();
        lam_cuda_check(cudaGetLastError(), "kernel launch");
        return true;
    }

} // namespace lamk
