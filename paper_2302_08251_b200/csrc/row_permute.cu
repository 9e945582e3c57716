// Byte-permutation copy through per-thread rows for physical pairs the register transposes
// cannot take: records with mixed leaf sizes (Record{a:f64,b:u16,c:i8,d:f32}), unaligned packed
// leaves, padded destinations (aos-aligned), mixed with SoA / AoSoA<L> sides.  The reference
// semantics are copyView's fieldwise loop (view.cpp:184-188) on physical leaves: a byte copy of
// every leaf value (bool leaves canonicalised to 0/1 on read, scalar.hpp:259-261), nothing else
// written.
//
// A thread owns G = 16 consecutive elements.  For every stream of each side the bytes of those
// elements form one contiguous, 16-byte aligned span (a record stream or AoSoA<L> with L | 16:
// 16/L blocks; an AoSoA<L> with 16 | L or SoA: one run of 16 values per leaf), loaded with 16-byte
// vectors into the thread's private shared-memory row (odd word stride: conflict-free), the leaf
// values moved inside the row (4-byte moves where both offsets allow, else bytes), and the
// destination spans written back with 16-byte vectors.  A destination with bytes copyView never
// writes (padding) is read into the row first, so whole-span stores keep those bytes.
#include "device_common.cuh"
#include "launch.h"

namespace lamk
{
    __device__ __forceinline__ uint64_t rp_span_addr(const RPSpan& s, uint64_t e0)
    {
        return s.base + (e0 >> s.lsh) * s.bs + (e0 & s.lmask) * s.ls;
    }

    __global__ void __launch_bounds__(64) k_row_permute(const __grid_constant__ RPParams p)
    {
        extern __shared__ __align__(16) uint32_t rsm[];
        uint32_t* row = rsm + threadIdx.x * p.rowWords;
        uint8_t* rb = reinterpret_cast<uint8_t*>(row);
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        for(uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < p.groups; g += stride)
        {
            const uint64_t e0 = p.begin + g * RP_G;
            // ---- spans -> row (source; destination too when it has holes) ----
            const uint32_t nin = p.ns + (p.preload ? p.nd : 0);
            for(uint32_t sp = 0; sp < nin; ++sp)
            {
                const RPSpan& s = sp < p.ns ? p.s[sp] : p.d[sp - p.ns];
                const uint4* src = reinterpret_cast<const uint4*>(rp_span_addr(s, e0));
                uint32_t* at = row + s.row / 4;
                const uint32_t nv = s.len / 16;
                uint32_t k = 0;
                for(; k + 4 <= nv; k += 4)
                {
                    uint4 x[4];
#pragma unroll
                    for(int u = 0; u < 4; ++u)
                        x[u] = __ldcs(src + k + u);
#pragma unroll
                    for(int u = 0; u < 4; ++u)
                    {
                        at[4 * (k + u)] = x[u].x;
                        at[4 * (k + u) + 1] = x[u].y;
                        at[4 * (k + u) + 2] = x[u].z;
                        at[4 * (k + u) + 3] = x[u].w;
                    }
                }
                for(; k < nv; ++k)
                {
                    const uint4 x = __ldcs(src + k);
                    at[4 * k] = x.x;
                    at[4 * k + 1] = x.y;
                    at[4 * k + 2] = x.z;
                    at[4 * k + 3] = x.w;
                }
            }
            // ---- leaf values: source row bytes -> destination row bytes ----
            for(uint32_t f = 0; f < p.nl; ++f)
            {
                const RPLeaf& L = p.leaf[f];
#pragma unroll 4
                for(uint32_t j = 0; j < RP_G; ++j)
                {
                    const uint32_t so = L.srow + (j >> L.slsh) * L.sbs + (j & L.slmask) * L.sls;
                    const uint32_t d = L.drow + (j >> L.dlsh) * L.dbs + (j & L.dlmask) * L.dls;
                    if(L.isBool)
                        rb[d] = rb[so] != 0;
                    else if(L.size >= 4 && ((so | d) & 3) == 0)
                        for(uint32_t b = 0; b < L.size; b += 4)
                            row[(d + b) / 4] = row[(so + b) / 4];
                    else
                        for(uint32_t b = 0; b < L.size; ++b)
                            rb[d + b] = rb[so + b];
                }
            }
            // ---- destination row -> spans ----
            for(uint32_t sp = 0; sp < p.nd; ++sp)
            {
                const RPSpan& s = p.d[sp];
                uint4* dst = reinterpret_cast<uint4*>(rp_span_addr(s, e0));
                const uint32_t* at = row + s.row / 4;
                const uint32_t nv = s.len / 16;
                for(uint32_t k = 0; k < nv; ++k)
                    __stcs(dst + k, make_uint4(at[4 * k], at[4 * k + 1], at[4 * k + 2], at[4 * k + 3]));
            }
        }
    }

    bool row_permute(const RPParams& p, cudaStream_t s)
    {
        if(p.groups == 0)
            return false;
        const size_t smem = static_cast<size_t>(64) * p.rowWords * sizeof(uint32_t);
        if(smem > 200 * 1024)
            return false;
        lam_cuda_check(opt_in_smem(reinterpret_cast<const void*>(k_row_permute), smem), "opt_in_smem");
        int dev = 0, occ = 0;
        cudaGetDevice(&dev);
        if(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_row_permute, 64, smem) != cudaSuccess || occ < 1)
            occ = 1;
        const uint64_t want = (p.groups + 63) / 64;
        const uint64_t cap = static_cast<uint64_t>(sm_count(dev)) * occ * 8;
        const unsigned grid = static_cast<unsigned>(want < cap ? want : cap);
        k_row_permute<<<grid, 64, smem, s>>>(p);
        count_launch();
        lam_cuda_check(cudaGetLastError(), "kernel launch");
        return true;
    }
} // namespace lamk
