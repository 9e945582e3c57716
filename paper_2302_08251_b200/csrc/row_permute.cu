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
// vectors into the thread's private shared-memory row (odd word stride: conflict-free; every
// vector of the group in flight at once), the leaf values moved inside the row (word-aligned
// destinations: one funnel shift per word from any source offset; else bytes), and the
// destination spans written back with 16-byte vectors.  A destination with bytes copyView never
// writes (padding) is read into the row first, so whole-span stores keep those bytes.
#include "device_common.cuh"
#include "launch.h"

namespace lamk
{
    __global__ void __launch_bounds__(64) k_row_permute(const __grid_constant__ RPParams p)
    {
        extern __shared__ __align__(16) uint32_t rsm[];
        uint32_t* row = rsm + threadIdx.x * p.rowWords;
        uint8_t* rb = reinterpret_cast<uint8_t*>(row);
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        for(uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < p.groups; g += stride)
        {
            const uint64_t e0 = p.begin + g * RP_G;
            // ---- spans -> row (source; destination too when it has holes): every 16-byte vector
            // of the group in flight at once (RP_MAXV at most), then into the row ----
            {
                uint4 x[RP_MAXV];
#pragma unroll
                for(int k = 0; k < RP_MAXV; ++k)
                    if(k < static_cast<int>(p.nvin))
                        x[k] = __ldcs(reinterpret_cast<const uint4*>(p.vin[k].base + (e0 >> p.vin[k].lsh) * p.vin[k].bs
                                                                     + (e0 & p.vin[k].lmask) * p.vin[k].ls));
#pragma unroll
                for(int k = 0; k < RP_MAXV; ++k)
                    if(k < static_cast<int>(p.nvin))
                    {
                        uint32_t* at = row + p.vin[k].row / 4;
                        at[0] = x[k].x;
                        at[1] = x[k].y;
                        at[2] = x[k].z;
                        at[3] = x[k].w;
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
                    else if(L.size >= 4 && (d & 3) == 0)
                    {
                        // word-aligned destination: each word from the (possibly unaligned) source
                        // by one funnel shift of the two words covering it
                        const uint32_t sh = (so & 3) * 8;
                        const uint32_t* sw = row + so / 4;
                        for(uint32_t b = 0; b < L.size / 4; ++b)
                            row[d / 4 + b] = sh ? __funnelshift_r(sw[b], sw[b + 1], sh) : sw[b];
                    }
                    else
                        for(uint32_t b = 0; b < L.size; ++b)
                            rb[d + b] = rb[so + b];
                }
            }
            // ---- destination row -> spans ----
#pragma unroll
            for(int k = 0; k < RP_MAXV; ++k)
                if(k < static_cast<int>(p.nvout))
                {
                    const uint32_t* at = row + p.vout[k].row / 4;
                    __stcs(reinterpret_cast<uint4*>(p.vout[k].base + (e0 >> p.vout[k].lsh) * p.vout[k].bs
                                                    + (e0 & p.vout[k].lmask) * p.vout[k].ls),
                           make_uint4(at[0], at[1], at[2], at[3]));
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
