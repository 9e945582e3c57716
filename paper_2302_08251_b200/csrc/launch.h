// Host-callable launchers implemented in the .cu translation units.
#pragma once

#include "lam_plan.h"

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

// throws (mapped to LAM_ECUDA at the C ABI) on a CUDA error; defined in capi.cpp
void lam_cuda_check(cudaError_t e, const char* what);

namespace lamk
{
    // counts every kernel this library launches (reported as gpu_launches)
    void count_launch(uint64_t n = 1);
    uint64_t launch_count();

    // bit packing for 1/2/8-byte leaves and fields wider than 32 bits (packv.cu)
    struct PackVParams
    {
        unsigned long long vals;   // value stream (element 0's value, SoA) or AoSoA block base
        unsigned long long bits;   // bit stream (word 0 = element 0)
        unsigned long long begin;  // first element (multiple of 32)
        unsigned long long groups; // groups of 32 elements
        uint32_t w;                // field width, 1..64
        uint32_t kind;             // 0 int, 1 float
        uint32_t sgn;              // int: sign-extend on unpack
        uint32_t E, M;             // float format
        uint32_t vbs, vl, vsh, vinb; // value stream geometry: SoA (vl == 1) or AoSoA (vl % 32 == 0)
    };

    struct PackVMulti
    {
        PackVParams base; // shared fields; per-leaf fields below (leaf = blockIdx.y)
        unsigned long long vals[8], bits[8];
        uint32_t vinb[8], sgn[8];
    };
    bool packv(const PackVParams* jobs, uint32_t n, uint32_t vsize, bool pack, cudaStream_t s);

    // register transpose over multi-stream sides (Split mappings), vec_multi.cu
    struct VMSide
    {
        // leaf-contiguous leaves (mode 0): V values at base + (e0 >> lsh) * bs + (e0 & lmask) * S
        unsigned long long base[8];
        uint32_t bs[8], lsh[8], lmask[8], mode[8];
        // record leaves (mode 1): element j's value at row word wpos + j * wstep
        uint32_t wpos[8], wstep[8];
        // record streams as 16-byte vectors k < nvec: address vb + e0 * vs, row words [vrow, vrow + 4)
        unsigned long long vb[8];
        uint32_t vs[8], vrow[8], nvec;
        uint32_t full; // one record stream with every leaf in order (AoS): register renaming, no row
    };
    struct VMParams
    {
        VMSide s, d;
        unsigned long long begin, groups; // groups of V elements
        uint32_t nl, rowWords;            // rowWords: odd (conflict-free lane rows)
    };
    bool vec_multi(const VMParams& p, uint32_t leafSize, cudaStream_t s);

    // bit stream -> bit stream, one leaf (pack.cu k_repack32)
    struct RepackParams
    {
        unsigned long long src, dst;      // bit streams (word 0 = element 0)
        unsigned long long begin, groups; // first element (multiple of 32), groups of 32
        uint32_t ws, wd;                  // field widths 1..32
        uint32_t kind;                    // 0 int, 1 float (E <= 8, M <= 23 on both sides)
        uint32_t sE, sM, dE, dM;
        uint32_t ssgn; // int: sign-extend the source field (signed leaf type)
    };
    bool repack32(const RepackParams& p, cudaStream_t s);
    // minifloat -> minifloat with compile-time formats (e8m10, e5m10, e4m3, e5m2 on both sides)
    bool repack_flt_fast(const RepackParams& p, cudaStream_t s);



    int sm_count(int device);

    // Opt `func` in to `smem` bytes of dynamic shared memory on the CURRENT device.  The
    // attribute is per device, so it is tracked per (kernel, device).
    cudaError_t opt_in_smem(const void* func, size_t smem);

    // Grid for a grid-stride streaming kernel: `want` CTAs (one pass of the data), capped at
    // `perSm` x SMs, with the cap overridable by the environment variable `env`; a cap of 0
    // means uncapped.  Uncapped one-pass grids measured best for streaming copies on B200: the
    // hardware block scheduler keeps the active CTAs on a compact, advancing address window
    // (k_vec_transpose 6.24 -> 6.70 TB/s at 2^26 records).
    unsigned stream_grid(uint64_t want, const char* env, uint64_t perSm);

    // FieldAccessCount closed form: reads[f] += count (src), writes[f] += count (dst), f < nleaves
    cudaError_t fac_add(unsigned long long* srcCounters, unsigned long long* dstCounters, uint32_t nleaves,
                        uint64_t count, cudaStream_t s);

    // generic fieldwise copy over [begin, end): one thread per element, all leaves,
    // plan interpreter on both sides (copy_generic.cu)
    cudaError_t generic_copy(const lamp_view* src, const lamp_view* dst, uint64_t begin, uint64_t end,
                             uint32_t nleaves, bool facSrc, bool facDst, cudaStream_t s, bool countHeat = true);
    // Heatmap accounting when every terminal of the side is a physical byte range
    struct HeatTerm
    {
        uint32_t inblock, ls, size;
    };
    struct HeatStream
    {
        uint64_t base0, bs, lanes;
        uint32_t lshift, nr, t0, t1; // terms [t0, t1) live on this stream
        // closed form, interior blocks: the counts repeat with period P = bs / gcd(g, bs) blocks;
        // pattern[patOff + k] is the count of block pb0 + k (P = 0: no pattern, exact per block)
        int64_t pb0, pLo, pHi;       // pattern origin and the interior block range [pLo, pHi]
        uint32_t period, patOff;
    };
    struct HeatParams
    {
        unsigned long long* heat;
        const uint64_t* heatOff; // device: first counter of blob nr
        uint64_t begin, end, E, gran;
        uint32_t gshift; // log2(gran) when a power of two, else 64
        uint32_t nstreams, maxWindow;
        HeatStream st[64];
        HeatTerm term[256];
        uint32_t pattern[2048];
    };
    cudaError_t heat_phys(const HeatParams& p, cudaStream_t s);

    // Heatmap accounting of a copy over [begin, end) whose data moved through a fast kernel
    cudaError_t heat_account(const lamp_view* v, uint64_t begin, uint64_t end, uint32_t nleaves, cudaStream_t s);
    // byte-exact blob copy (copyView's sameLayout memcpy path)
    cudaError_t blob_copy(void* dst, const void* src, uint64_t bytes, cudaStream_t s);
    cudaError_t blob_copy_multi(void* const* dst, const void* const* src, const uint64_t* bytes, size_t n, cudaStream_t s);
    cudaError_t read_values(const lamp_view* v, const uint64_t* lin, const uint32_t* leaf, uint64_t* out, size_t n,
                            cudaStream_t s);
    cudaError_t write_values(const lamp_view* v, const uint64_t* lin, const uint32_t* leaf, const uint64_t* in,
                             size_t n, cudaStream_t s);
} // namespace lamk
