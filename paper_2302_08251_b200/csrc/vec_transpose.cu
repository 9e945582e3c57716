// Register-transpose copy for uniform physical layout pairs (the C2 matrix: AoS, SoA single/
// multi blob, AoSoA<L>, any ordered pair).  A thread owns a group of V consecutive elements
// (V * leafSize = 16 bytes) and moves them with NL 16-byte loads and NL 16-byte stores:
//   leaf-contiguous side  (SoA, AoSoA with L % V == 0): one 16-byte vector per leaf
//   record-contiguous side (AoS with uniform leaves):    the V records are NL vectors
// The AoS <-> SoA/AoSoA permutation is a compile-time renaming of registers (NL is a
// template parameter), so there is no shared memory, no synchronisation and no wasted
// HBM traffic; every load/store instruction of a warp covers 512 contiguous bytes on the
// leaf-contiguous side and a fully written 3.5 KB span (7 x 16 B per thread) on the
// record side.  Same reference semantics as copyView's fieldwise loop (view.cpp:184-188):
// a pure byte permutation of the leaf bytes, nothing else written.
#include "device_common.cuh"
#include "launch.h"
#include "tile.h"

#include <cstdlib>

namespace lamk
{
    struct VecSide
    {
        unsigned long long leafBase[LAMT_UNI_LEAVES]; // leaf-contiguous: address of element 0 of leaf f
        unsigned long long recBase;                   // record-contiguous: address of record 0
        uint32_t recordContig;
        uint32_t bs, lanes, lshift;                   // leaf-contiguous block geometry
    };

    struct VecParams
    {
        VecSide s, d;
        unsigned long long begin;
        unsigned long long groups; // groups of V elements
        unsigned long long facSrc, facDst;
        uint32_t nl, facS, facD;
    };

    template<int V>
    __device__ __forceinline__ uint64_t leaf_off(const VecSide& sd, uint64_t e0)
    {
        // e0 is a multiple of V and V divides the lane count: the V elements are adjacent
        if(sd.lanes == 1)
            return e0 * sd.bs;
        return (e0 >> sd.lshift) * sd.bs + (e0 & (sd.lanes - 1)) * (16 / V);
    }

    template<int NL, int V>
    __global__ void __launch_bounds__(256, 4) k_vec_transpose(const __grid_constant__ VecParams p)
    {
        constexpr int S = 16 / V; // leaf size in bytes
        using W = typename std::conditional<S == 4, uint32_t, unsigned long long>::type;
        extern __shared__ __align__(16) uint8_t vsm[];
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        uint64_t cnt = 0;
        for(uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < p.groups; g += stride)
        {
            const uint64_t e0 = p.begin + g * V;
            W v[NL][V];
            // ---- load ----
            if(p.s.recordContig)
            {
                const uint4* base = reinterpret_cast<const uint4*>(p.s.recBase + e0 * (NL * S));
                uint4 x[NL];
#pragma unroll
                for(int k = 0; k < NL; ++k)
                    x[k] = __ldcs(base + k);
#pragma unroll
                for(int k = 0; k < NL; ++k)
                {
                    const W* w = reinterpret_cast<const W*>(&x[k]);
#pragma unroll
                    for(int j = 0; j < V; ++j)
                    {
                        constexpr int dummy = 0;
                        (void)dummy;
                        const int word = k * V + j; // record-major word index
                        v[word % NL][word / NL] = w[j];
                    }
                }
            }
            else
            {
                const uint64_t off = leaf_off<V>(p.s, e0);
                uint4 x[NL];
#pragma unroll
                for(int f = 0; f < NL; ++f)
                    x[f] = __ldcs(reinterpret_cast<const uint4*>(p.s.leafBase[f] + off));
#pragma unroll
                for(int f = 0; f < NL; ++f)
                {
                    const W* w = reinterpret_cast<const W*>(&x[f]);
#pragma unroll
                    for(int j = 0; j < V; ++j)
                        v[f][j] = w[j];
                }
            }
            // ---- store ----
            if(p.d.recordContig)
            {
                // the warp's 32 groups are one contiguous span of 32*NL vectors: stage them in
                // the warp's smem slice (lane stride NL*16 B: conflict-free for 16-byte
                // accesses), then write 512 contiguous bytes per store instruction
                uint4* slice = reinterpret_cast<uint4*>(vsm) + (threadIdx.x >> 5) * (32 * NL);
                const uint32_t lane = threadIdx.x & 31;
                const bool fullWarp = __activemask() == 0xFFFFFFFFu && (g - lane) + 32 <= p.groups;
                if(fullWarp)
                {
#pragma unroll
                    for(int k = 0; k < NL; ++k)
                    {
                        uint4 x;
                        W* w = reinterpret_cast<W*>(&x);
#pragma unroll
                        for(int j = 0; j < V; ++j)
                        {
                            const int word = k * V + j;
                            w[j] = v[word % NL][word / NL];
                        }
                        slice[lane * NL + k] = x;
                    }
                    __syncwarp();
                    uint4* base = reinterpret_cast<uint4*>(p.d.recBase + (e0 - uint64_t(lane) * V) * (NL * S));
#pragma unroll
                    for(int k = 0; k < NL; ++k)
                        __stcs(base + k * 32 + lane, slice[k * 32 + lane]);
                    __syncwarp();
                }
                else
                {
                    uint4* base = reinterpret_cast<uint4*>(p.d.recBase + e0 * (NL * S));
#pragma unroll
                    for(int k = 0; k < NL; ++k)
                    {
                        uint4 x;
                        W* w = reinterpret_cast<W*>(&x);
#pragma unroll
                        for(int j = 0; j < V; ++j)
                        {
                            const int word = k * V + j;
                            w[j] = v[word % NL][word / NL];
                        }
                        __stcs(base + k, x);
                    }
                }
            }
            else
            {
                const uint64_t off = leaf_off<V>(p.d, e0);
#pragma unroll
                for(int f = 0; f < NL; ++f)
                {
                    uint4 x;
                    W* w = reinterpret_cast<W*>(&x);
#pragma unroll
                    for(int j = 0; j < V; ++j)
                        w[j] = v[f][j];
                    __stcs(reinterpret_cast<uint4*>(p.d.leafBase[f] + off), x);
                }
            }
            cnt += V;
        }
        // FieldAccessCount: warp-aggregated, one global atomic per warp per field
        if(p.facS || p.facD)
        {
            unsigned long long w = cnt;
            for(int o = 16; o > 0; o >>= 1)
                w += __shfl_down_sync(0xFFFFFFFFu, w, o);
            if((threadIdx.x & 31) == 0 && w)
                for(uint32_t f = 0; f < p.nl; ++f)
                {
                    if(p.facS)
                        atomicAdd(reinterpret_cast<unsigned long long*>(p.facSrc) + f, w);
                    if(p.facD)
                        atomicAdd(reinterpret_cast<unsigned long long*>(p.facDst) + p.nl + f, w);
                }
        }
    }

    template<int NL, int V>
    static void launch_vec(const VecParams& p, unsigned grid, cudaStream_t s)
    {
        const size_t smem = p.d.recordContig ? 8 * 32 * NL * 16 : 0; // 8 warps x one staged span
        k_vec_transpose<NL, V><<<grid, 256, smem, s>>>(p);
    }

    // Host entry: returns false when NL/leaf size has no instantiation.
    bool vec_transpose(const VecParams& p, uint32_t leafSize, cudaStream_t s)
    {
        int dev = 0;
        cudaGetDevice(&dev);
        // one pass, uncapped (see stream_grid); with FieldAccessCount the per-warp counter flush
        // favours a persistent grid of 16 CTAs per SM
        const uint64_t want = (p.groups + 255) / 256;
        const unsigned grid = stream_grid(want, "LAMB_VEC_CTAS", (p.facS || p.facD) ? 16 : 0);
        if(leafSize == 4)
        {
            switch(p.nl)
            {
            case 1: launch_vec<1, 4>(p, grid, s); break;
            case 2: launch_vec<2, 4>(p, grid, s); break;
            case 3: launch_vec<3, 4>(p, grid, s); break;
            case 4: launch_vec<4, 4>(p, grid, s); break;
            case 5: launch_vec<5, 4>(p, grid, s); break;
            case 6: launch_vec<6, 4>(p, grid, s); break;
            case 7: launch_vec<7, 4>(p, grid, s); break;
            case 8: launch_vec<8, 4>(p, grid, s); break;
            default: return false;
            }
        }
        else if(leafSize == 8)
        {
            switch(p.nl)
            {
            case 1: launch_vec<1, 2>(p, grid, s); break;
            case 2: launch_vec<2, 2>(p, grid, s); break;
            case 3: launch_vec<3, 2>(p, grid, s); break;
            case 4: launch_vec<4, 2>(p, grid, s); break;
            case 5: launch_vec<5, 2>(p, grid, s); break;
            case 6: launch_vec<6, 2>(p, grid, s); break;
            case 7: launch_vec<7, 2>(p, grid, s); break;
            case 8: launch_vec<8, 2>(p, grid, s); break;
            default: return false;
            }
        }
        else
            return false;
        count_launch();
        lam_cuda_check(cudaGetLastError(), "kernel launch");
        return true;
    }
} // namespace lamk
