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
        uint32_t sstage; // AoS source loaded warp-coalesced through the smem slice (k_vec_transpose)
    };

    template<int V>
    __device__ __forceinline__ uint64_t leaf_off(const VecSide& sd, uint64_t e0)
    {
        // e0 is a multiple of V and V divides the lane count: the V elements are adjacent
        if(sd.lanes == 1)
            return e0 * sd.bs;
        return (e0 >> sd.lshift) * sd.bs + (e0 & (sd.lanes - 1)) * (16 / V);
    }

    template<int NL, int V, int MINB = 4>
    __global__ void __launch_bounds__(256, MINB) k_vec_transpose(const __grid_constant__ VecParams p)
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
                uint4 x[NL];
                // the warp's 32 groups are one contiguous span of 32*NL vectors: on full warps it
                // is loaded with 512-byte coalesced loads into the warp's smem slice, and each lane
                // then reads its NL vectors (lane stride NL*16 B, conflict-free for odd NL)
                const uint32_t lane = threadIdx.x & 31;
                const bool fullWarp = p.sstage && __activemask() == 0xFFFFFFFFu && (g - lane) + 32 <= p.groups;
                if(fullWarp)
                {
                    uint4* slice = reinterpret_cast<uint4*>(vsm) + (threadIdx.x >> 5) * (32 * NL);
                    const uint4* wbase = reinterpret_cast<const uint4*>(p.s.recBase + (e0 - uint64_t(lane) * V) * (NL * S));
                    uint4 t[NL];
#pragma unroll
                    for(int k = 0; k < NL; ++k)
                        t[k] = __ldcs(wbase + k * 32 + lane);
#pragma unroll
                    for(int k = 0; k < NL; ++k)
                        slice[k * 32 + lane] = t[k];
                    __syncwarp();
#pragma unroll
                    for(int k = 0; k < NL; ++k)
                        x[k] = slice[lane * NL + k];
                    __syncwarp(); // the slice may be reused for the destination below
                }
                else
                {
                    const uint4* base = reinterpret_cast<const uint4*>(p.s.recBase + e0 * (NL * S));
#pragma unroll
                    for(int k = 0; k < NL; ++k)
                        x[k] = __ldcs(base + k);
                }
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
                uint4 x[NL];
                // AoSoA<L> source without padding, L | 32V (sstage 2): the warp's 32V elements are
                // 32V/L whole blocks, one contiguous span of 32*NL vectors: loaded coalesced into the
                // slice, then lane t reads leaf f of its elements at vector
                // (tV / L) * bs/16 + f * L*S/16 + (tV % L) * S/16 (conflict-free for L | 32V)
                const uint32_t lane = threadIdx.x & 31;
                const bool fullWarp = p.sstage == 2 && __activemask() == 0xFFFFFFFFu && (g - lane) + 32 <= p.groups;
                if(fullWarp)
                {
                    uint4* slice = reinterpret_cast<uint4*>(vsm) + (threadIdx.x >> 5) * (32 * NL);
                    const uint64_t ew = e0 - uint64_t(lane) * V;
                    const uint4* wbase = reinterpret_cast<const uint4*>(p.s.recBase + (ew >> p.s.lshift) * p.s.bs);
                    uint4 t[NL];
#pragma unroll
                    for(int k = 0; k < NL; ++k)
                        t[k] = __ldcs(wbase + k * 32 + lane);
#pragma unroll
                    for(int k = 0; k < NL; ++k)
                        slice[k * 32 + lane] = t[k];
                    __syncwarp();
                    const uint32_t el = lane * V;
                    const uint32_t vi = (el >> p.s.lshift) * (p.s.bs >> 4) + (((el & (p.s.lanes - 1)) * S) >> 4);
                    const uint32_t fstep = (p.s.lanes * S) >> 4;
#pragma unroll
                    for(int f = 0; f < NL; ++f)
                        x[f] = slice[vi + f * fstep];
                    __syncwarp(); // the slice may be reused for the destination below
                }
                else
                {
                    const uint64_t off = leaf_off<V>(p.s, e0);
#pragma unroll
                    for(int f = 0; f < NL; ++f)
                        x[f] = __ldcs(reinterpret_cast<const uint4*>(p.s.leafBase[f] + off));
                }
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
                // recordContig 2: AoSoA<V> blocks (leaf-major), vector k = leaf k's V values
                const bool blockMajor = p.d.recordContig == 2;
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
                            w[j] = blockMajor ? v[k][j] : v[word % NL][word / NL];
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
                            w[j] = blockMajor ? v[k][j] : v[word % NL][word / NL];
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
        const size_t smem = (p.d.recordContig || p.sstage) ? 8 * 32 * NL * 16 : 0; // 8 warps x one staged span
        static const int minb = std::getenv("LAMB_VEC_MINB") ? std::atoi(std::getenv("LAMB_VEC_MINB")) : 3;
        if constexpr(V == 4 && NL >= 7)
            if(minb == 3)
            {
                k_vec_transpose<NL, V, 3><<<grid, 256, smem, s>>>(p);
                return;
            }
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

    // ---- ChangeType f32 <-> f64 on a uniform pair: the register transpose plus one conversion
    // per value (ScalarValue::convertTo, scalar.hpp:295-306, x86 NaN rules).  A thread owns 4
    // consecutive elements: per leaf 4 x SS bytes in, 4 x DS bytes out; record-contiguous sides
    // move the 4 records as 16-byte vectors (destination staged through the warp's smem slice).
    template<int SS, int DS>
    __device__ __forceinline__ uint64_t cvt_bits(uint64_t v)
    {
        if constexpr(SS == 4 && DS == 8)
            return lamd::f32_to_f64_bits(static_cast<uint32_t>(v));
        else if constexpr(SS == 8 && DS == 4)
            return lamd::f64_to_f32_bits(v);
        else
            return v;
    }

    __device__ __forceinline__ uint64_t side_off(const VecSide& sd, uint64_t e0, uint32_t size)
    {
        if(sd.lanes == 1)
            return e0 * sd.bs;
        return (e0 >> sd.lshift) * sd.bs + (e0 & (sd.lanes - 1)) * size;
    }

    template<int NL, int SS, int DS>
    __global__ void __launch_bounds__(256) k_vec_convert(const __grid_constant__ VecParams p)
    {
        constexpr int NVS = NL * SS / 4, NVD = NL * DS / 4; // 16-byte vectors per 4 records
        extern __shared__ __align__(16) uint8_t csm[];
        const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        const uint32_t lane = threadIdx.x & 31;
        const bool live = g < p.groups;
        const uint64_t e0 = p.begin + g * 4;
        uint64_t v[NL][4];
        if(live)
        {
            if(p.s.recordContig)
            {
                const uint4* base = reinterpret_cast<const uint4*>(p.s.recBase + e0 * (NL * SS));
                uint32_t w[NVS * 4];
#pragma unroll
                for(int q = 0; q < NVS; ++q)
                {
                    const uint4 x = __ldcs(base + q);
                    w[4 * q] = x.x;
                    w[4 * q + 1] = x.y;
                    w[4 * q + 2] = x.z;
                    w[4 * q + 3] = x.w;
                }
#pragma unroll
                for(int r = 0; r < 4; ++r)
#pragma unroll
                    for(int f = 0; f < NL; ++f)
                    {
                        const int k = (r * NL + f) * (SS / 4);
                        v[f][r] = SS == 4 ? w[k] : ((uint64_t(w[k + 1]) << 32) | w[k]);
                    }
            }
            else
            {
                const uint64_t off = side_off(p.s, e0, SS);
#pragma unroll
                for(int f = 0; f < NL; ++f)
                {
                    const uint4* b = reinterpret_cast<const uint4*>(p.s.leafBase[f] + off);
                    const uint4 x = __ldcs(b);
                    if constexpr(SS == 4)
                    {
                        v[f][0] = x.x;
                        v[f][1] = x.y;
                        v[f][2] = x.z;
                        v[f][3] = x.w;
                    }
                    else
                    {
                        const uint4 y = __ldcs(b + 1);
                        v[f][0] = (uint64_t(x.y) << 32) | x.x;
                        v[f][1] = (uint64_t(x.w) << 32) | x.z;
                        v[f][2] = (uint64_t(y.y) << 32) | y.x;
                        v[f][3] = (uint64_t(y.w) << 32) | y.z;
                    }
                }
            }
#pragma unroll
            for(int f = 0; f < NL; ++f)
#pragma unroll
                for(int r = 0; r < 4; ++r)
                    v[f][r] = cvt_bits<SS, DS>(v[f][r]);
        }
        if(p.d.recordContig)
        {
            uint4* slice = reinterpret_cast<uint4*>(csm) + (threadIdx.x >> 5) * (32 * NVD);
            if(live)
            {
                uint32_t w[NVD * 4];
#pragma unroll
                for(int r = 0; r < 4; ++r)
#pragma unroll
                    for(int f = 0; f < NL; ++f)
                    {
                        const int k = (r * NL + f) * (DS / 4);
                        w[k] = static_cast<uint32_t>(v[f][r]);
                        if constexpr(DS == 8)
                            w[k + 1] = static_cast<uint32_t>(v[f][r] >> 32);
                    }
#pragma unroll
                for(int q = 0; q < NVD; ++q)
                    slice[lane * NVD + q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
            }
            __syncwarp();
            const uint64_t warpG = g - lane;
            const uint32_t liveLanes =
                static_cast<uint32_t>(p.groups > warpG ? (p.groups - warpG < 32 ? p.groups - warpG : 32) : 0);
            uint4* dst = reinterpret_cast<uint4*>(p.d.recBase + (p.begin + warpG * 4) * (NL * DS));
            for(uint32_t c = lane; c < liveLanes * NVD; c += 32)
                __stcs(dst + c, slice[c]);
        }
        else if(live)
        {
            const uint64_t off = side_off(p.d, e0, DS);
#pragma unroll
            for(int f = 0; f < NL; ++f)
            {
                uint4* b = reinterpret_cast<uint4*>(p.d.leafBase[f] + off);
                if constexpr(DS == 4)
                    __stcs(b, make_uint4(static_cast<uint32_t>(v[f][0]), static_cast<uint32_t>(v[f][1]),
                                         static_cast<uint32_t>(v[f][2]), static_cast<uint32_t>(v[f][3])));
                else
                {
                    __stcs(b, make_uint4(static_cast<uint32_t>(v[f][0]), static_cast<uint32_t>(v[f][0] >> 32),
                                         static_cast<uint32_t>(v[f][1]), static_cast<uint32_t>(v[f][1] >> 32)));
                    __stcs(b + 1, make_uint4(static_cast<uint32_t>(v[f][2]), static_cast<uint32_t>(v[f][2] >> 32),
                                             static_cast<uint32_t>(v[f][3]), static_cast<uint32_t>(v[f][3] >> 32)));
                }
            }
        }
    }

    template<int NL, int SS, int DS>
    static void launch_convert(const VecParams& p, cudaStream_t s)
    {
        const size_t smem = p.d.recordContig ? 8 * 32 * (NL * DS / 4) * 16 : 0;
        lam_cuda_check(opt_in_smem(reinterpret_cast<const void*>(k_vec_convert<NL, SS, DS>), smem), "opt_in_smem");
        k_vec_convert<NL, SS, DS><<<stream_grid((p.groups + 255) / 256, "LAMB_VEC_CTAS", 0), 256, smem, s>>>(p);
    }

    template<int SS, int DS>
    static bool convert_nl(const VecParams& p, cudaStream_t s)
    {
        switch(p.nl)
        {
        case 1: launch_convert<1, SS, DS>(p, s); break;
        case 2: launch_convert<2, SS, DS>(p, s); break;
        case 3: launch_convert<3, SS, DS>(p, s); break;
        case 4: launch_convert<4, SS, DS>(p, s); break;
        case 5: launch_convert<5, SS, DS>(p, s); break;
        case 6: launch_convert<6, SS, DS>(p, s); break;
        case 7: launch_convert<7, SS, DS>(p, s); break;
        case 8: launch_convert<8, SS, DS>(p, s); break;
        default: return false;
        }
        return true;
    }

    // groups are 4 elements; ss/ds = leaf bytes of the two sides (4 <-> 8)
    bool vec_convert(const VecParams& p, uint32_t ss, uint32_t ds, cudaStream_t s)
    {
        bool ok;
        if(ss == 4 && ds == 8)
            ok = convert_nl<4, 8>(p, s);
        else if(ss == 8 && ds == 4)
            ok = convert_nl<8, 4>(p, s);
        else
            return false;
        if(!ok)
            return false;
        count_launch();
        lam_cuda_check(cudaGetLastError(), "kernel launch");
        return true;
    }
} // namespace lamk
