// Register transpose for uniform physical pairs whose sides are made of several streams with
// different geometries -- Split mappings (mappings.cpp:213-269) such as
// split:Pos:soa-mb:aos-packed, and any mix of SoA / AoSoA<L> leaf runs and AoS-like record
// streams holding a subset of the leaves.  k_vec_transpose (vec_transpose.cu) needs one block
// geometry per side; this kernel resolves every leaf on its own:
//   leaf-contiguous leaf (SoA, or AoSoA with V | L): one 16-byte vector of its V elements,
//     address base_f + (e0 >> lsh_f) * bs_f + (e0 & mask_f) * S
//   record stream (L = 1, record stride rbs = RL * S, leaves at inblock q * S): the V records
//     are RL 16-byte vectors; their words pass through the lane's private smem row, from which
//     each leaf's V values are gathered (source) or into which they are scattered (destination)
// A thread owns V consecutive elements (V * S = 16 bytes per leaf); every global access is a
// 16-byte vector and every byte crosses HBM once.  Rows have an odd word stride, so the per-word
// scatter/gather is conflict-free.  Same semantics as copyView's fieldwise loop (view.cpp:184-188):
// a byte permutation of the leaf bytes; record streams are written whole only when their leaves
// cover every byte of the record (host-checked).
#include "device_common.cuh"
#include "launch.h"

namespace lamk
{
    template<int S>
    __device__ __forceinline__ uint64_t vm_leaf_addr(const VMSide& sd, int f, uint64_t e0)
    {
        return sd.base[f] + (e0 >> sd.lsh[f]) * sd.bs[f] + (e0 & sd.lmask[f]) * S;
    }

    // 5 CTAs/SM (<= 102 registers): ncu showed the kernel latency-bound at 4 (128 registers);
    // 6 spilled the 7- and 8-leaf instantiations
#define VMB 5
    template<int NL, int V>
    __global__ void __launch_bounds__(128, VMB) k_vec_multi(const __grid_constant__ VMParams p)
    {
        constexpr int S = 16 / V;  // leaf bytes
        constexpr int WPE = S / 4; // 32-bit words per value
        using W = typename std::conditional<S == 4, uint32_t, unsigned long long>::type;
        extern __shared__ __align__(16) uint32_t vmsm[];
        uint32_t* row = vmsm + threadIdx.x * p.rowWords; // lane-private (no synchronisation needed)
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        for(uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < p.groups; g += stride)
        {
            const uint64_t e0 = p.begin + g * V;
            W v[NL][V];
            // ---- loads: every 16-byte vector of the source in flight at once ----
            // (record streams are covered by their leaves, so they hold at most NL vectors)
            uint4 rx[NL], lx[NL];
#pragma unroll
            for(int k = 0; k < NL; ++k)
                if(k < static_cast<int>(p.s.nvec))
                    rx[k] = __ldcs(reinterpret_cast<const uint4*>(p.s.vb[k] + e0 * p.s.vs[k]));
#pragma unroll
            for(int f = 0; f < NL; ++f)
                if(p.s.mode[f] == 0)
                    lx[f] = __ldcs(reinterpret_cast<const uint4*>(vm_leaf_addr<S>(p.s, f, e0)));
            if(p.s.full)
            {
                // one record stream holding every leaf in order (AoS): the V records are NL
                // vectors and the AoS -> leaf permutation is compile-time register renaming
#pragma unroll
                for(int k = 0; k < NL; ++k)
                {
                    const W* w = reinterpret_cast<const W*>(&rx[k]);
#pragma unroll
                    for(int j = 0; j < V; ++j)
                    {
                        const int word = k * V + j;
                        v[word % NL][word / NL] = w[j];
                    }
                }
            }
            else
            {
                // record vectors -> the row, word by word
#pragma unroll
                for(int k = 0; k < NL; ++k)
                    if(k < static_cast<int>(p.s.nvec))
                    {
                        uint32_t* at = row + p.s.vrow[k];
                        at[0] = rx[k].x;
                        at[1] = rx[k].y;
                        at[2] = rx[k].z;
                        at[3] = rx[k].w;
                    }
            }
            // ---- gather every leaf ----
#pragma unroll
            for(int f = 0; f < NL; ++f)
            {
                if(p.s.full)
                    break;
                if(p.s.mode[f] == 0)
                {
                    const W* w = reinterpret_cast<const W*>(&lx[f]);
#pragma unroll
                    for(int j = 0; j < V; ++j)
                        v[f][j] = w[j];
                }
                else
                {
                    const uint32_t* at = row + p.s.wpos[f];
                    const uint32_t step = p.s.wstep[f];
#pragma unroll
                    for(int j = 0; j < V; ++j)
                    {
                        if constexpr(S == 4)
                            v[f][j] = at[j * step];
                        else
                            v[f][j] = static_cast<unsigned long long>(at[j * step])
                                | (static_cast<unsigned long long>(at[j * step + 1]) << 32);
                    }
                }
            }
            if(p.d.full)
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
                    __stcs(reinterpret_cast<uint4*>(p.d.vb[k] + e0 * p.d.vs[k]), x);
                }
                continue;
            }
            // ---- scatter every leaf: leaf runs straight out, record leaves into the row ----
#pragma unroll
            for(int f = 0; f < NL; ++f)
            {
                if(p.d.mode[f] == 0)
                {
                    uint4 x;
                    W* w = reinterpret_cast<W*>(&x);
#pragma unroll
                    for(int j = 0; j < V; ++j)
                        w[j] = v[f][j];
                    __stcs(reinterpret_cast<uint4*>(vm_leaf_addr<S>(p.d, f, e0)), x);
                }
                else
                {
                    uint32_t* at = row + p.d.wpos[f];
                    const uint32_t step = p.d.wstep[f];
#pragma unroll
                    for(int j = 0; j < V; ++j)
                    {
                        at[j * step] = static_cast<uint32_t>(v[f][j]);
                        if constexpr(S == 8)
                            at[j * step + 1] = static_cast<uint32_t>(v[f][j] >> 32);
                    }
                }
            }
            // ---- destination record vectors: the row -> 16-byte stores ----
#pragma unroll
            for(int k = 0; k < NL; ++k)
                if(k < static_cast<int>(p.d.nvec))
                {
                    const uint32_t* at = row + p.d.vrow[k];
                    __stcs(reinterpret_cast<uint4*>(p.d.vb[k] + e0 * p.d.vs[k]), make_uint4(at[0], at[1], at[2], at[3]));
                }
        }
    }

    template<int V>
    static bool launch_multi_v(const VMParams& p, cudaStream_t s)
    {
        const size_t smem = static_cast<size_t>(128) * p.rowWords * sizeof(uint32_t);
        const unsigned grid = stream_grid((p.groups + 127) / 128, "LAMB_VEC_CTAS", 0);
        auto go = [&](auto kern)
        {
            lam_cuda_check(opt_in_smem(reinterpret_cast<const void*>(kern), smem), "opt_in_smem");
            kern<<<grid, 128, smem, s>>>(p);
        };
        switch(p.nl)
        {
        case 1: go(k_vec_multi<1, V>); break;
        case 2: go(k_vec_multi<2, V>); break;
        case 3: go(k_vec_multi<3, V>); break;
        case 4: go(k_vec_multi<4, V>); break;
        case 5: go(k_vec_multi<5, V>); break;
        case 6: go(k_vec_multi<6, V>); break;
        case 7: go(k_vec_multi<7, V>); break;
        case 8: go(k_vec_multi<8, V>); break;
        default: return false;
        }
        return true;
    }

    bool vec_multi(const VMParams& p, uint32_t leafSize, cudaStream_t s)
    {
        if(p.groups == 0)
            return false;
        bool ok = false;
        if(leafSize == 4)
            ok = launch_multi_v<4>(p, s);
        else if(leafSize == 8)
            ok = launch_multi_v<2>(p, s);
        if(!ok)
            return false;
        count_launch();
        lam_cuda_check(cudaGetLastError(), "kernel launch");
        return true;
    }
} // namespace lamk
