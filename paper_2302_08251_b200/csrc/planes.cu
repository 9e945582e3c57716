// Record <-> byte-plane kernels: Bytesplit over a record-contiguous (AoS / packed) side,
// optionally through ChangeType f64 <-> f32 (computed.cpp:405-502 bytesplit, 363-378 changetype;
// the C5 layout `changetype:f64=f32:bytesplit:soa-mb` and plain `bytesplit:soa-mb`).
//   forward  (records -> planes): a thread reads 4 records (4 x NL x SB bytes as 16-byte vectors),
//            converts, and writes one 32-bit word (byte k of the 4 elements) to each plane.
//   backward (planes -> records): a thread reads one word per plane, assembles 4 values per leaf,
//            converts, and stages the 4 records in its warp's smem slice so each store
//            instruction writes 512 contiguous bytes of the record stream.
// SB = source/destination record leaf bytes (4 or 8); CVT = f64 record leaf <-> f32 planes.
#include "device_common.cuh"
#include "launch.h"

#include <cstdlib>

namespace lamk
{
    struct PlaneParams
    {
        unsigned long long rec;           // record stream, element 0
        unsigned long long plane[8][8];   // plane[f][k]: byte k of leaf f, element 0
        unsigned long long begin, groups; // groups of 4 elements
        uint32_t nl;
    };

    template<int NL, int SB, bool CVT>
    __global__ void __launch_bounds__(256) k_rec_to_planes(const __grid_constant__ PlaneParams p, int stage)
    {
        constexpr int PB = CVT ? 4 : SB;          // plane bytes per leaf
        constexpr int NV = NL * SB * 4 / 16;      // 16-byte vectors per 4 records
        constexpr int NVP = NV | 1;               // lane row stride in the slice (conflict-free)
        using PV = typename std::conditional<PB == 8, unsigned long long, uint32_t>::type;
        extern __shared__ __align__(16) uint4 rsl[];
        const uint32_t lane = threadIdx.x & 31;
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        for(uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < p.groups; g += stride)
        {
            const uint64_t e0 = p.begin + g * 4;
            uint32_t w[NV * 4];
            // full warps: the warp's 32 x 4 records are one contiguous span of 32*NV vectors,
            // loaded with 512-byte coalesced loads into the warp's slice, then read back per lane
            const bool fullWarp = stage && __activemask() == 0xFFFFFFFFu && (g - lane) + 32 <= p.groups;
            if(fullWarp)
            {
                uint4* slice = rsl + (threadIdx.x >> 5) * (32 * NVP);
                const uint4* wsrc = reinterpret_cast<const uint4*>(p.rec + (e0 - uint64_t(lane) * 4) * (NL * SB));
                uint4 t[NV];
#pragma unroll
                for(int q = 0; q < NV; ++q)
                    t[q] = __ldcs(wsrc + q * 32 + lane);
#pragma unroll
                for(int q = 0; q < NV; ++q)
                {
                    const uint32_t i = q * 32 + lane;
                    slice[(i / NV) * NVP + i % NV] = t[q];
                }
                __syncwarp();
#pragma unroll
                for(int q = 0; q < NV; ++q)
                {
                    const uint4 x = slice[lane * NVP + q];
                    w[4 * q] = x.x;
                    w[4 * q + 1] = x.y;
                    w[4 * q + 2] = x.z;
                    w[4 * q + 3] = x.w;
                }
                __syncwarp();
            }
            else
            {
                const uint4* src = reinterpret_cast<const uint4*>(p.rec + e0 * (NL * SB));
#pragma unroll
                for(int q = 0; q < NV; ++q)
                {
                    const uint4 x = __ldcs(src + q);
                    w[4 * q] = x.x;
                    w[4 * q + 1] = x.y;
                    w[4 * q + 2] = x.z;
                    w[4 * q + 3] = x.w;
                }
            }
            PV v[4][NL]; // value of leaf f of element q
#pragma unroll
            for(int q = 0; q < 4; ++q)
#pragma unroll
                for(int f = 0; f < NL; ++f)
                {
                    const int word = (q * NL + f) * (SB / 4);
                    if constexpr(SB == 4)
                        v[q][f] = w[word];
                    else
                    {
                        const uint64_t d = (uint64_t(w[word + 1]) << 32) | w[word];
                        if constexpr(CVT)
                            v[q][f] = lamd::f64_to_f32_bits(d);
                        else
                            v[q][f] = d;
                    }
                }
#pragma unroll
            for(int f = 0; f < NL; ++f)
#pragma unroll
                for(int k = 0; k < PB; ++k)
                {
                    const uint32_t word = static_cast<uint32_t>((v[0][f] >> (8 * k)) & 0xFF)
                        | static_cast<uint32_t>(((v[1][f] >> (8 * k)) & 0xFF) << 8)
                        | static_cast<uint32_t>(((v[2][f] >> (8 * k)) & 0xFF) << 16)
                        | static_cast<uint32_t>(((v[3][f] >> (8 * k)) & 0xFF) << 24);
                    __stcs(reinterpret_cast<uint32_t*>(p.plane[f][k] + e0), word);
                }
        }
    }

    template<int NL, int SB, bool CVT>
    __global__ void __launch_bounds__(256) k_planes_to_rec(const __grid_constant__ PlaneParams p)
    {
        constexpr int PB = CVT ? 4 : SB;
        constexpr int NV = NL * SB * 4 / 16;
        extern __shared__ __align__(16) uint4 rsm[];
        const uint32_t lane = threadIdx.x & 31;
        uint4* slice = rsm + (threadIdx.x >> 5) * (32 * NV);
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        const uint64_t gEnd = (p.groups + 31) / 32 * 32;
        for(uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g - lane < gEnd; g += stride)
        {
            const bool live = g < p.groups;
            const uint64_t e0 = p.begin + g * 4;
            uint32_t w[NV * 4];
            if(live)
            {
                uint32_t pw[NL][PB];
#pragma unroll
                for(int f = 0; f < NL; ++f)
#pragma unroll
                    for(int k = 0; k < PB; ++k)
                        pw[f][k] = __ldcs(reinterpret_cast<const uint32_t*>(p.plane[f][k] + e0));
#pragma unroll
                for(int q = 0; q < 4; ++q)
#pragma unroll
                    for(int f = 0; f < NL; ++f)
                    {
                        uint64_t x = 0;
#pragma unroll
                        for(int k = 0; k < PB; ++k)
                            x |= uint64_t((pw[f][k] >> (8 * q)) & 0xFF) << (8 * k);
                        const int word = (q * NL + f) * (SB / 4);
                        if constexpr(SB == 4)
                            w[word] = static_cast<uint32_t>(x);
                        else
                        {
                            const uint64_t d = CVT ? lamd::f32_to_f64_bits(static_cast<uint32_t>(x)) : x;
                            w[word] = static_cast<uint32_t>(d);
                            w[word + 1] = static_cast<uint32_t>(d >> 32);
                        }
                    }
#pragma unroll
                for(int q = 0; q < NV; ++q)
                    slice[lane * NV + q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
            }
            __syncwarp();
            // the warp's live lanes own one contiguous record span: 512 contiguous bytes per store
            const uint64_t warpG = g - lane;
            const uint32_t liveLanes =
                static_cast<uint32_t>(p.groups > warpG ? (p.groups - warpG < 32 ? p.groups - warpG : 32) : 0);
            uint4* dst = reinterpret_cast<uint4*>(p.rec + (p.begin + warpG * 4) * (NL * SB));
            for(uint32_t c = lane; c < liveLanes * NV; c += 32)
                __stcs(dst + c, slice[c]);
            __syncwarp();
        }
    }

    template<int NL, int SB, bool CVT>
    static void launch_planes(const PlaneParams& p, bool toPlanes, cudaStream_t s)
    {
        constexpr int NV = NL * SB * 4 / 16;
        if(toPlanes)
        {
            // LAMB_PLANES_SSTAGE=0: per-thread record loads (no slice)
            static const int stage = std::getenv("LAMB_PLANES_SSTAGE") ? std::atoi(std::getenv("LAMB_PLANES_SSTAGE")) : 1;
            const size_t smem = stage ? 8 * 32 * (NV | 1) * sizeof(uint4) : 0;
            if(stage)
                lam_cuda_check(opt_in_smem(reinterpret_cast<const void*>(k_rec_to_planes<NL, SB, CVT>), smem), "opt_in_smem");
            k_rec_to_planes<NL, SB, CVT><<<stream_grid((p.groups + 255) / 256, "LAMB_PLANES_CTAS", 0), 256, smem, s>>>(p, stage);
        }
        else
        {
            const size_t smem = 8 * 32 * NV * sizeof(uint4);
            lam_cuda_check(opt_in_smem(reinterpret_cast<const void*>(k_planes_to_rec<NL, SB, CVT>), smem),
                           "opt_in_smem");
            k_planes_to_rec<NL, SB, CVT><<<stream_grid((p.groups + 255) / 256, "LAMB_PLANES_CTAS", 0), 256, smem, s>>>(p);
        }
    }

    template<int SB, bool CVT>
    static bool dispatch_nl(const PlaneParams& p, bool toPlanes, cudaStream_t s)
    {
        switch(p.nl)
        {
        case 1: launch_planes<1, SB, CVT>(p, toPlanes, s); break;
        case 2: launch_planes<2, SB, CVT>(p, toPlanes, s); break;
        case 3: launch_planes<3, SB, CVT>(p, toPlanes, s); break;
        case 4: launch_planes<4, SB, CVT>(p, toPlanes, s); break;
        case 5: launch_planes<5, SB, CVT>(p, toPlanes, s); break;
        case 6: launch_planes<6, SB, CVT>(p, toPlanes, s); break;
        case 7: launch_planes<7, SB, CVT>(p, toPlanes, s); break;
        case 8: launch_planes<8, SB, CVT>(p, toPlanes, s); break;
        default: return false;
        }
        return true;
    }

    // sb = record leaf bytes (4 / 8), cvt = f64 records with f32 planes
    bool planes_copy(const PlaneParams& p, uint32_t sb, bool cvt, bool toPlanes, cudaStream_t s)
    {
        if(p.groups == 0)
            return false;
        bool ok;
        if(sb == 4 && !cvt)
            ok = dispatch_nl<4, false>(p, toPlanes, s);
        else if(sb == 8 && !cvt)
            ok = dispatch_nl<8, false>(p, toPlanes, s);
        else if(sb == 8 && cvt)
            ok = dispatch_nl<8, true>(p, toPlanes, s);
        else
            return false;
        if(!ok)
            return false;
        count_launch();
        lam_cuda_check(cudaGetLastError(), "kernel launch");
        return true;
    }
} // namespace lamk
