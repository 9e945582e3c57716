// Tile kernels over the tile-plan form (tile.h):
//   k_warp_tile      the general engine: one warp per tile, 16-byte loads of the source images
//                    into smem, per-leaf transforms from host-resolved descriptors, 16-byte
//                    stores (every plan pair without a specialised kernel)
//   k_uniform_direct uniform pairs outside the register transpose (AoSoA lanes not a multiple
//                    of 16/size or not a power of two): per-element moves through L1
//   k_uniform_warp   warp-tile transpose for uniform pairs (kept behind LAMB_DIRECT=0)
//   k_tile_copy      the first design (below): kept as the last resort for unaligned images.
//
// Tile engine: persistent, double-buffered, TMA-bulk-staged layout copy.
//
// Per CTA, per tile of T elements:
//   load      every source stream image  HBM -> smem   (cp.async.bulk + mbarrier tx count)
//   transform per leaf, per element: read terminal(s) from the source image, convert,
//             write terminal(s) into the destination image (PHYS / byte planes) or into
//             a per-element pattern scratch (bit-packed destinations)
//   pack      bit-packed destinations: each thread owns whole 32-bit words and
//             funnel-shifts them together from the scratch (no RMW, no atomics)
//   store     every destination image smem -> HBM   (cp.async.bulk bulk_group)
// The next tile's loads are in flight during the transform of the current one, and the
// stores of tile k drain while tile k+1 is transformed.  HBM traffic is exactly the
// algorithmic bytes (each source/destination byte moves once); the element-granular
// shuffling happens in shared memory, where AoS strides (7 words for the 28-byte
// record) are bank-conflict free.
#include "device_common.cuh"
#include "launch.h"
#include "tile.h"

namespace lamk
{
    namespace
    {
        __device__ __forceinline__ uint32_t smem_u32(const void* p)
        {
            return static_cast<uint32_t>(__cvta_generic_to_shared(p));
        }

        __device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
        {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
        }

        __device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
        {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                         : "memory");
        }

        __device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
        {
            asm volatile(
                "{\n"
                ".reg .pred p;\n"
                "LAB_WAIT:\n"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                "@!p bra LAB_WAIT;\n"
                "}\n" ::"r"(smem_u32(bar)),
                "r"(parity)
                : "memory");
        }

        __device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar)
        {
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(smem)),
                "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
                : "memory");
        }

        __device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, uint32_t bytes)
        {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem), "r"(smem_u32(smem)),
                         "r"(bytes)
                         : "memory");
        }

        __device__ __forceinline__ void bulk_commit()
        {
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }

        template<int N>
        __device__ __forceinline__ void bulk_wait_read()
        {
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
        }

        __device__ __forceinline__ void bulk_wait_all()
        {
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }

        __device__ __forceinline__ void fence_async_smem()
        {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }

        __device__ __forceinline__ uint64_t tile_global_off(const lamt_stream& s, uint64_t tileStart)
        {
            if(s.kind == 1)
                return (tileStart * s.bs) >> 3; // tileStart*bits is a multiple of 128
            const uint64_t blk = s.lshift != 0xFFFFFFFFu ? (tileStart >> s.lshift) : tileStart / s.lanes;
            return blk * s.bs;
        }

        __device__ __forceinline__ uint32_t image_rel(const lamt_stream& s, uint32_t e, const lamt_term& t)
        {
            if(s.lanes == 1)
                return e * s.bs + t.inblock;
            uint32_t blk, lane;
            if(s.lshift != 0xFFFFFFFFu)
            {
                blk = e >> s.lshift;
                lane = e & (s.lanes - 1);
            }
            else
            {
                blk = e / s.lanes;
                lane = e - blk * s.lanes;
            }
            return blk * s.bs + t.inblock + lane * t.ls;
        }

        __device__ __forceinline__ uint64_t lds_bytes(const uint8_t* p, uint32_t size, bool aligned)
        {
            return lamd::load_bytes(p, size, aligned);
        }

        __device__ __forceinline__ void bulk_wait_read_dyn(uint32_t n)
        {
            if(n == 0)
                bulk_wait_read<0>();
            else if(n == 1)
                bulk_wait_read<1>();
            else if(n == 2)
                bulk_wait_read<2>();
            else
                bulk_wait_read<3>();
        }

        // CTA-cooperative copy for images whose global start is not 16-byte aligned
        __device__ void coop_g2s(uint8_t* smem, const uint8_t* g, uint32_t bytes)
        {
            const uintptr_t a = reinterpret_cast<uintptr_t>(g);
            if((a & 3) == 0 && (bytes & 3) == 0)
            {
                const uint32_t* gs = reinterpret_cast<const uint32_t*>(g);
                uint32_t* ss = reinterpret_cast<uint32_t*>(smem);
                for(uint32_t k = threadIdx.x; k < bytes / 4; k += blockDim.x)
                    ss[k] = __ldg(gs + k);
            }
            else
                for(uint32_t k = threadIdx.x; k < bytes; k += blockDim.x)
                    smem[k] = __ldg(g + k);
        }

        __device__ void coop_s2g(uint8_t* g, const uint8_t* smem, uint32_t bytes)
        {
            const uintptr_t a = reinterpret_cast<uintptr_t>(g);
            if((a & 3) == 0 && (bytes & 3) == 0)
            {
                uint32_t* gd = reinterpret_cast<uint32_t*>(g);
                const uint32_t* ss = reinterpret_cast<const uint32_t*>(smem);
                for(uint32_t k = threadIdx.x; k < bytes / 4; k += blockDim.x)
                    gd[k] = ss[k];
            }
            else
                for(uint32_t k = threadIdx.x; k < bytes; k += blockDim.x)
                    g[k] = smem[k];
        }

        // read the storage value of one leaf for tile-local element e from the source images
        __device__ __forceinline__ uint64_t tile_read(const lamt_params& p, const lamt_leaf& L, const uint8_t* sbuf,
                                                      uint32_t e)
        {
            switch(L.skind)
            {
            case LAMT_K_PHYS:
            {
                const lamt_term& t = L.s[0];
                const lamt_stream& s = p.st[t.stream];
                uint64_t v = lds_bytes(sbuf + s.smem_off + image_rel(s, e, t), t.size, t.aligned);
                return L.stype == lamd::BOOL ? uint64_t(v != 0) : v;
            }
            case LAMT_K_SPLIT:
            {
                uint64_t v = 0;
                for(uint32_t k = 0; k < L.sn; ++k)
                {
                    const lamt_term& t = L.s[k];
                    const lamt_stream& s = p.st[t.stream];
                    v |= uint64_t(sbuf[s.smem_off + image_rel(s, e, t)]) << (8 * k);
                }
                return L.stype == lamd::BOOL ? uint64_t(v != 0) : v;
            }
            case LAMT_K_BITS_INT:
            {
                const lamt_stream& s = p.st[L.s[0].stream];
                uint64_t pat = lamd::read_bits(reinterpret_cast<const uint32_t*>(sbuf + s.smem_off),
                                               uint64_t(e) * L.sE, L.sE);
                if(L.ssigned)
                {
                    const uint64_t sb = 1ull << (L.sE - 1);
                    pat = (pat ^ sb) - sb;
                }
                return pat & lamd::low_mask(8 * lamd::scalar_size(L.stype));
            }
            case LAMT_K_BITS_FLT:
            {
                const lamt_stream& s = p.st[L.s[0].stream];
                const uint32_t w = 1 + L.sE + L.sM;
                const uint64_t pat = lamd::read_bits(reinterpret_cast<const uint32_t*>(sbuf + s.smem_off),
                                                     uint64_t(e) * w, w);
                if(L.stype == lamd::F32 && L.sE == 8 && L.sM == 10)
                {
                    const uint32_t pp = static_cast<uint32_t>(pat);
                    const uint32_t sign = (pp >> 18) << 31;
                    if((pp & 0x3FC00u) == 0x3FC00u && (pp & 0x3FFu))
                        return sign | 0x7FC00000u;
                    return sign | ((pp & 0x3FFFFu) << 13);
                }
                if(L.stype == lamd::F32 && L.sE == 5 && L.sM == 10)
                {
                    const uint32_t pp = static_cast<uint32_t>(pat);
                    if((pp & 0x7C00u) == 0x7C00u && (pp & 0x3FFu))
                        return ((pp >> 15) << 31) | 0x7FC00000u;
                    return __float_as_uint(__half2float(__ushort_as_half(static_cast<unsigned short>(pp))));
                }
                if(L.stype == lamd::F32 && L.sE <= 8 && L.sM <= 23)
                    return lamd::float_decode_f32(static_cast<uint32_t>(pat), L.sE, L.sM);
                const uint64_t d = lamd::float_decode(pat, L.sE, L.sM);
                return L.stype == lamd::F32 ? lamd::f64_to_f32_bits(d) : d;
            }
            default:
                return 0;
            }
        }

        __device__ __forceinline__ void tile_write(const lamt_params& p, const lamt_leaf& L, uint8_t* dbuf, uint32_t e,
                                                   uint64_t v)
        {
            switch(L.dkind)
            {
            case LAMT_K_PHYS:
            {
                const lamt_term& t = L.d[0];
                const lamt_stream& s = p.st[t.stream];
                lamd::store_bytes(dbuf + s.smem_off + image_rel(s, e, t), t.size, t.aligned, v);
                return;
            }
            case LAMT_K_SPLIT:
                for(uint32_t k = 0; k < L.dn; ++k)
                {
                    const lamt_term& t = L.d[k];
                    const lamt_stream& s = p.st[t.stream];
                    dbuf[s.smem_off + image_rel(s, e, t)] = static_cast<uint8_t>(v >> (8 * k));
                }
                return;
            case LAMT_K_BITS_INT:
            {
                const lamt_stream& s = p.st[L.d[0].stream];
                const uint64_t pat = v & lamd::low_mask(L.dE);
                if(s.scratch64)
                    reinterpret_cast<unsigned long long*>(dbuf + s.scratch_off)[e] = pat;
                else
                    reinterpret_cast<uint32_t*>(dbuf + s.scratch_off)[e] = static_cast<uint32_t>(pat);
                return;
            }
            case LAMT_K_BITS_FLT:
            {
                const lamt_stream& s = p.st[L.d[0].stream];
                uint64_t pat;
                if(L.dtype == lamd::F32 && L.dE == 8 && L.dM == 10)
                    pat = lamd::encode_e8m10_f32(static_cast<uint32_t>(v));
                else if(L.dtype == lamd::F32 && L.dE == 5 && L.dM == 10)
                    pat = lamd::encode_e5m10_f32(static_cast<uint32_t>(v));
                else if(L.dtype == lamd::F32)
                    pat = lamd::float_encode_f32(static_cast<uint32_t>(v), L.dE, L.dM);
                else
                    pat = lamd::float_encode(v, L.dE, L.dM);
                if(s.scratch64)
                    reinterpret_cast<unsigned long long*>(dbuf + s.scratch_off)[e] = pat;
                else
                    reinterpret_cast<uint32_t*>(dbuf + s.scratch_off)[e] = static_cast<uint32_t>(pat);
                return;
            }
            default:
                return;
            }
        }

        // whole-word assembly of a bit-packed destination image from its pattern scratch
        __device__ __forceinline__ void pack_words(const lamt_stream& s, uint8_t* dbuf, uint32_t T, uint32_t lane,
                                                   uint32_t nthreads)
        {
            const uint32_t w = s.bs;
            const uint32_t words = T * w / 32;
            uint32_t* out = reinterpret_cast<uint32_t*>(dbuf + s.smem_off);
            if(!s.scratch64)
            {
                const uint32_t* sc = reinterpret_cast<const uint32_t*>(dbuf + s.scratch_off);
                for(uint32_t q = lane; q < words; q += nthreads)
                {
                    const uint32_t bit = q * 32;
                    uint32_t k = bit / w;
                    const uint32_t o = bit - k * w;
                    uint64_t acc = uint64_t(sc[k]) >> o;
                    uint32_t pos = w - o;
                    ++k;
                    while(pos < 32)
                    {
                        acc |= uint64_t(sc[k]) << pos;
                        pos += w;
                        ++k;
                    }
                    out[q] = static_cast<uint32_t>(acc);
                }
            }
            else
            {
                const unsigned long long* sc = reinterpret_cast<const unsigned long long*>(dbuf + s.scratch_off);
                for(uint32_t q = lane; q < words; q += nthreads)
                {
                    const uint64_t bit = uint64_t(q) * 32;
                    uint64_t k = bit / w;
                    const uint32_t o = static_cast<uint32_t>(bit - k * w);
                    uint64_t acc = sc[k] >> o;
                    const uint32_t pos = w - o;
                    if(pos < 32)
                        acc |= sc[k + 1] << pos;
                    out[q] = static_cast<uint32_t>(acc);
                }
            }
        }
    } // namespace

    // CTA-wide pipeline: `stages` source stage buffers (TMA bulk loads in flight ahead of the
    // transform) and `dstages` destination buffers (TMA bulk stores draining behind it).
    // One __syncthreads per tile: after it, thread 0 issues the tile's stores, refills the
    // freed source stage and retires the store that last used the next destination buffer.
    __device__ __forceinline__ uint32_t uni_off(uint32_t e, uint32_t L, uint32_t sh, uint32_t bs, uint32_t ls)
    {
        if(L == 1)
            return e * bs;
        if(sh != 0xFFFFFFFFu)
            return (e >> sh) * bs + (e & (L - 1)) * ls;
        return (e / L) * bs + (e % L) * ls;
    }

    __device__ __forceinline__ void cp_async16(void* smem, const void* g)
    {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(g) : "memory");
    }
    __device__ __forceinline__ void cp_async_commit()
    {
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    template<int N>
    __device__ __forceinline__ void cp_async_wait()
    {
        asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
    }
    __device__ __forceinline__ void cp_async_wait_dyn(uint32_t n)
    {
        switch(n)
        {
        case 0: cp_async_wait<0>(); break;
        case 1: cp_async_wait<1>(); break;
        case 2: cp_async_wait<2>(); break;
        default: cp_async_wait<3>(); break;
        }
    }

    __device__ __forceinline__ void mbar_arrive(uint64_t* bar)
    {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
    }

    __device__ __forceinline__ void named_sync(uint32_t id, uint32_t n)
    {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
    }

    // Warp-specialised pipeline.  Warp 0 (one elected lane) is the producer: it keeps
    // `stages` tiles of TMA bulk loads in flight (mbarrier full[s], tx-counted), issues the
    // TMA bulk stores of each finished tile and recycles destination buffers once the bulk
    // store has read them (dfree[d]).  Warps 1.. (the consumers) only transform: wait full[s]
    // and dfree[d], move the tile through shared memory, fence the async proxy and arrive on
    // tdone[s].  No CTA-wide barrier in the steady state.
    __global__ void __launch_bounds__(544, 1) k_tile_copy(const __grid_constant__ lamt_params p)
    {
        extern __shared__ __align__(128) uint8_t smem[];
        __shared__ __align__(8) uint64_t full[LAMT_MAX_STAGES];
        __shared__ __align__(8) uint64_t tdone[LAMT_MAX_STAGES];
        __shared__ __align__(8) uint64_t dfree[8];
        const uint32_t warp = threadIdx.x >> 5;
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t ncons = blockDim.x - 32; // consumer threads
        const uint32_t nconsWarps = ncons >> 5;
        uint8_t* srcBase = smem;
        uint8_t* dstBase = smem + p.stages * p.src_bytes;
        if(threadIdx.x == 0)
        {
            for(uint32_t s = 0; s < p.stages; ++s)
            {
                mbar_init(&full[s], 1);
                mbar_init(&tdone[s], nconsWarps);
            }
            for(uint32_t d = 0; d < p.dstages; ++d)
                mbar_init(&dfree[d], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();

        if(warp == 0)
        {
            // ================= producer =================
            if(lane != 0)
                return;
            auto load = [&](uint32_t tile, uint32_t s)
            {
                const uint64_t t0 = p.begin + uint64_t(tile) * p.T;
                uint8_t* sb = srcBase + s * p.src_bytes;
                if(p.tma_bytes)
                    mbar_expect_tx(&full[s], p.tma_bytes);
                else
                    mbar_arrive(&full[s]);
                for(uint32_t k = 0; k < p.nsrc; ++k)
                {
                    const lamt_stream& st = p.st[k];
                    if(st.tma && st.tile_bytes)
                        bulk_g2s(sb + st.smem_off, reinterpret_cast<const uint8_t*>(st.gptr) + tile_global_off(st, t0),
                                 st.tile_bytes, &full[s]);
                }
            };
            for(uint32_t d = 0; d < p.dstages; ++d)
                mbar_arrive(&dfree[d]); // every destination buffer starts free
            for(uint32_t s = 0; s < p.stages; ++s)
                if(blockIdx.x + s * gridDim.x < p.ntiles)
                    load(blockIdx.x + s * gridDim.x, s);
            for(uint32_t j = 0;; ++j)
            {
                const uint32_t tile = blockIdx.x + j * gridDim.x;
                if(tile >= p.ntiles)
                    break;
                const uint32_t s = j % p.stages;
                const uint32_t d = j % p.dstages;
                mbar_wait(&tdone[s], (j / p.stages) & 1);
                const uint64_t t0 = p.begin + uint64_t(tile) * p.T;
                uint8_t* db = dstBase + d * p.dst_bytes;
                for(uint32_t k = p.nsrc; k < p.nsrc + p.ndst; ++k)
                {
                    const lamt_stream& st = p.st[k];
                    if(st.tma && st.tile_bytes)
                        bulk_s2g(reinterpret_cast<uint8_t*>(st.gptr) + tile_global_off(st, t0), db + st.smem_off,
                                 st.tile_bytes);
                }
                bulk_commit();
                const uint32_t next = tile + p.stages * gridDim.x;
                if(next < p.ntiles)
                    load(next, s);
                // the store group of tile j-D+1 has left smem -> its buffer serves tile j+1
                bulk_wait_read_dyn(p.dstages - 1);
                if(j + 1 >= p.dstages)
                    mbar_arrive(&dfree[(j + 1) % p.dstages]);
            }
            bulk_wait_all();
            return;
        }

        // ================= consumers =================
        const uint32_t ct = threadIdx.x - 32;
        uint32_t os[LAMT_UNI_LEAVES], od[LAMT_UNI_LEAVES];
#pragma unroll
        for(int f = 0; f < LAMT_UNI_LEAVES; ++f)
        {
            os[f] = p.uoff_s[f];
            od[f] = p.uoff_d[f];
        }
        uint32_t done = 0;
        for(uint32_t k = 0;; ++k)
        {
            const uint32_t tile = blockIdx.x + k * gridDim.x;
            if(tile >= p.ntiles)
                break;
            const uint32_t s = k % p.stages;
            const uint32_t d = k % p.dstages;
            uint8_t* sb = srcBase + s * p.src_bytes;
            uint8_t* db = dstBase + d * p.dst_bytes;
            const uint64_t t0 = p.begin + uint64_t(tile) * p.T;
            mbar_wait(&full[s], (k / p.stages) & 1);
            mbar_wait(&dfree[d], (k / p.dstages) & 1);
            if(p.any_coop)
            {
                for(uint32_t j = 0; j < p.nsrc; ++j)
                {
                    const lamt_stream& st = p.st[j];
                    if(!st.tma && st.tile_bytes)
                        for(uint32_t q = ct; q < st.tile_bytes; q += ncons)
                            sb[st.smem_off + q] = __ldg(reinterpret_cast<const uint8_t*>(st.gptr)
                                                        + tile_global_off(st, t0) + q);
                }
                named_sync(1, ncons);
            }
            // ---- transform ----
            if(p.uni)
            {
                const uint32_t nl = p.nleaves;
                for(uint32_t e = ct; e < p.T; e += ncons)
                {
                    const uint32_t es = uni_off(e, p.ul_s, p.ush_s, p.ubs_s, p.uls_s);
                    const uint32_t ed = uni_off(e, p.ul_d, p.ush_d, p.ubs_d, p.uls_d);
                    if(p.usize == 4)
                    {
                        uint32_t v[LAMT_UNI_LEAVES];
#pragma unroll
                        for(int f = 0; f < LAMT_UNI_LEAVES; ++f)
                            if(f < nl)
                                v[f] = *reinterpret_cast<const uint32_t*>(sb + os[f] + es);
#pragma unroll
                        for(int f = 0; f < LAMT_UNI_LEAVES; ++f)
                            if(f < nl)
                                *reinterpret_cast<uint32_t*>(db + od[f] + ed) = v[f];
                    }
                    else
                    {
#pragma unroll
                        for(int f = 0; f < LAMT_UNI_LEAVES; ++f)
                            if(f < nl)
                                *reinterpret_cast<unsigned long long*>(db + od[f] + ed)
                                    = *reinterpret_cast<const unsigned long long*>(sb + os[f] + es);
                    }
                }
            }
            else
            {
                for(uint32_t f = 0; f < p.nleaves; ++f)
                {
                    const lamt_leaf& L = p.leaf[f];
                    for(uint32_t e = ct; e < p.T; e += ncons)
                    {
                        uint64_t v = tile_read(p, L, sb, e);
                        v = lamd::convert_value(v, L.stype, L.ltype);
                        v = lamd::convert_value(v, L.ltype, L.dtype);
                        tile_write(p, L, db, e, v);
                    }
                }
                if(p.any_bits)
                {
                    named_sync(1, ncons);
                    for(uint32_t j = p.nsrc; j < p.nsrc + p.ndst; ++j)
                        if(p.st[j].kind == 1)
                            pack_words(p.st[j], db, p.T, ct, ncons);
                }
            }
            done += p.T;
            if(p.any_coop)
            {
                named_sync(1, ncons);
                for(uint32_t j = p.nsrc; j < p.nsrc + p.ndst; ++j)
                {
                    const lamt_stream& st = p.st[j];
                    if(!st.tma && st.tile_bytes)
                        for(uint32_t q = ct; q < st.tile_bytes; q += ncons)
                            (reinterpret_cast<uint8_t*>(st.gptr) + tile_global_off(st, t0))[q] = db[st.smem_off + q];
                }
            }
            // make this thread's smem writes visible to the async proxy (the TMA store), then
            // one arrival per consumer warp
            fence_async_smem();
            __syncwarp();
            if(lane == 0)
                mbar_arrive(&tdone[s]);
        }
        // FieldAccessCount: every element of every leaf of a tile is accessed once; one
        // global atomic per CTA per field (instrument.cpp:57-72)
        if((p.facS || p.facD) && done)
        {
            for(uint32_t f = ct; f < p.nleaves; f += ncons)
            {
                if(p.facS)
                    atomicAdd(reinterpret_cast<unsigned long long*>(p.facSrc) + f, static_cast<unsigned long long>(done));
                if(p.facD)
                    atomicAdd(reinterpret_cast<unsigned long long*>(p.facDst) + p.nleaves + f,
                              static_cast<unsigned long long>(done));
            }
        }
    }

    // Direct uniform copy: no shared memory.  Thread = element; per leaf one 4/8-byte load at
    // the source geometry and one store at the destination geometry.  The strided side (AoS
    // 28-byte stride) is served from L1: the 7 leaf loads of a warp touch the same 7 lines.
    template<typename W, int UNROLL>
    __global__ void __launch_bounds__(256) k_uniform_direct(const __grid_constant__ lamt_params p, uint64_t n)
    {
        const uint8_t* sbase[LAMT_UNI_LEAVES];
        uint8_t* dbase[LAMT_UNI_LEAVES];
        const uint32_t nl = p.nleaves;
#pragma unroll
        for(int f = 0; f < LAMT_UNI_LEAVES; ++f)
            if(f < nl)
            {
                sbase[f] = reinterpret_cast<const uint8_t*>(p.st[p.leaf[f].s[0].stream].gptr) + p.leaf[f].s[0].inblock;
                dbase[f] = reinterpret_cast<uint8_t*>(p.st[p.leaf[f].d[0].stream].gptr) + p.leaf[f].d[0].inblock;
            }
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x * UNROLL;
        for(uint64_t i0 = p.begin + static_cast<uint64_t>(blockIdx.x) * blockDim.x * UNROLL + threadIdx.x;
            i0 < p.begin + n; i0 += stride)
        {
            W v[UNROLL][LAMT_UNI_LEAVES];
            uint64_t ed[UNROLL];
#pragma unroll
            for(int u = 0; u < UNROLL; ++u)
            {
                const uint64_t i = i0 + uint64_t(u) * blockDim.x;
                const uint64_t ii = i < p.begin + n ? i : p.begin;
                auto off = [&](uint32_t L, uint32_t sh, uint32_t mag, uint32_t bs, uint32_t ls) -> uint64_t {
                    if(L == 1)
                        return ii * bs;
                    if(sh != 0xFFFFFFFFu)
                        return (ii >> sh) * bs + (ii & (L - 1)) * ls;
                    const uint64_t q = __umulhi(static_cast<uint32_t>(ii), mag); // ii < 2^32 / L (host-checked)
                    return q * bs + (ii - q * L) * ls;
                };
                const uint64_t es = off(p.ul_s, p.ush_s, p.umag_s, p.ubs_s, p.uls_s);
                ed[u] = off(p.ul_d, p.ush_d, p.umag_d, p.ubs_d, p.uls_d);
                // 4-byte gathers from record-strided sources: keep them in L1 so the next
                // leaves' loads of the same lines hit
#pragma unroll
                for(int f = 0; f < LAMT_UNI_LEAVES; ++f)
                    if(f < nl)
                        v[u][f] = __ldg(reinterpret_cast<const W*>(sbase[f] + es));
            }
#pragma unroll
            for(int u = 0; u < UNROLL; ++u)
            {
                const uint64_t i = i0 + uint64_t(u) * blockDim.x;
                if(i < p.begin + n)
                {
#pragma unroll
                    for(int f = 0; f < LAMT_UNI_LEAVES; ++f)
                        if(f < nl)
                            __stcs(reinterpret_cast<W*>(dbase[f] + ed[u]), v[u][f]);
                }
            }
        }
    }

    // Warp-tile transpose for uniform physical pairs: every warp owns a private smem slice and
    // streams warp tiles of WT elements: 16-byte coalesced loads of the source images
    // (registers -> smem), the per-leaf transpose in smem, 16-byte coalesced stores of the
    // destination images.  Only __syncwarp; images of one side all have the same size
    // (one stream per leaf for SoA, one stream for AoS/AoSoA).
    template<typename W, int CH>
    __global__ void __launch_bounds__(256) k_uniform_warp(const __grid_constant__ lamt_params p, uint32_t ntiles)
    {
        extern __shared__ __align__(16) uint8_t wsm[];
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t warp = threadIdx.x >> 5;
        const uint32_t WT = p.T;
        uint8_t* sbuf = wsm + warp * (p.src_bytes + p.dst_bytes);
        uint8_t* dbuf = sbuf + p.src_bytes;
        const uint32_t ns = p.nsrc, nd = p.ndst;
        const uint32_t imgS = p.st[0].tile_bytes, imgD = p.st[ns].tile_bytes;
        const uint32_t cpsS = imgS >> 4, cpsD = imgD >> 4; // 16-byte chunks per image
        const uint32_t chS = ns * cpsS, chD = nd * cpsD;
        uint32_t os[LAMT_UNI_LEAVES], od[LAMT_UNI_LEAVES];
        const uint32_t nl = p.nleaves;
#pragma unroll
        for(int f = 0; f < LAMT_UNI_LEAVES; ++f)
        {
            os[f] = p.uoff_s[f];
            od[f] = p.uoff_d[f];
        }
        const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + warp;
        const uint32_t tw = gridDim.x * (blockDim.x >> 5);
        __shared__ unsigned long long s_done;
        if(threadIdx.x == 0)
            s_done = 0;
        __syncthreads();
        uint32_t done = 0;
        for(uint32_t wt = gw; wt < ntiles; wt += tw)
        {
            done += WT;
            const uint64_t t0 = p.begin + uint64_t(wt) * WT;
            // ---- load: CH chunks per lane in flight ----
            for(uint32_t c0 = 0; c0 < chS; c0 += 32 * CH)
            {
                uint4 v[CH];
#pragma unroll
                for(int u = 0; u < CH; ++u)
                {
                    const uint32_t c = c0 + u * 32 + lane;
                    if(c < chS)
                    {
                        const uint32_t j = c / cpsS, o = c - j * cpsS;
                        const uint4* g = reinterpret_cast<const uint4*>(
                            reinterpret_cast<const uint8_t*>(p.st[j].gptr) + tile_global_off(p.st[j], t0));
                        v[u] = __ldcs(g + o);
                    }
                }
#pragma unroll
                for(int u = 0; u < CH; ++u)
                {
                    const uint32_t c = c0 + u * 32 + lane;
                    if(c < chS)
                        reinterpret_cast<uint4*>(sbuf)[c] = v[u];
                }
            }
            __syncwarp();
            // ---- transpose in smem ----
            for(uint32_t e = lane; e < WT; e += 32)
            {
                const uint32_t es = uni_off(e, p.ul_s, p.ush_s, p.ubs_s, p.uls_s);
                const uint32_t ed = uni_off(e, p.ul_d, p.ush_d, p.ubs_d, p.uls_d);
                W v[LAMT_UNI_LEAVES];
#pragma unroll
                for(int f = 0; f < LAMT_UNI_LEAVES; ++f)
                    if(f < nl)
                        v[f] = *reinterpret_cast<const W*>(sbuf + os[f] + es);
#pragma unroll
                for(int f = 0; f < LAMT_UNI_LEAVES; ++f)
                    if(f < nl)
                        *reinterpret_cast<W*>(dbuf + od[f] + ed) = v[f];
            }
            __syncwarp();
            // ---- store ----
            for(uint32_t c = lane; c < chD; c += 32)
            {
                const uint32_t j = c / cpsD, o = c - j * cpsD;
                uint4* g = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(p.st[ns + j].gptr)
                                                    + tile_global_off(p.st[ns + j], t0));
                __stcs(g + o, reinterpret_cast<const uint4*>(dbuf)[c]);
            }
            __syncwarp();
        }
        // FieldAccessCount: per-warp totals -> shared counter -> one global atomic per CTA per field
        if(p.facS || p.facD)
        {
            if(lane == 0 && done)
                atomicAdd(&s_done, static_cast<unsigned long long>(done));
            __syncthreads();
            for(uint32_t f = threadIdx.x; f < nl && s_done; f += blockDim.x)
            {
                if(p.facS)
                    atomicAdd(reinterpret_cast<unsigned long long*>(p.facSrc) + f, s_done);
                if(p.facD)
                    atomicAdd(reinterpret_cast<unsigned long long*>(p.facDst) + nl + f, s_done);
            }
        }
    }

    // ---- warp-tile fast leaf loops ----------------------------------------------------------
    // One leaf of a warp tile with its terminal addressing resolved into registers once: a
    // term on a lanes == 1 stream (AoS record, SoA array, byte plane) sits at base + e * bs in
    // the smem image.  Handles PHYS <-> PHYS (any sizes, with conversion) and PHYS <-> SPLIT
    // (byte planes; 4 elements per lane so each plane gets one 32-bit smem access when the
    // planes are packed arrays).  Returns false for anything else (the generic loop runs).
    // size | 0x80: the term is not naturally aligned in the smem image (packed AoS of mixed
    // leaf sizes): byte-wise little-endian access
    __device__ __forceinline__ uint64_t wt_ld(const uint8_t* b, uint32_t size)
    {
        if(size & 0x80)
        {
            // two aligned 8-byte smem loads and a funnel shift (the 8 bytes after a source
            // image still lie inside the warp's buffer: the destination images follow it)
            const uint32_t sz = size & 0x7F;
            const uintptr_t a = reinterpret_cast<uintptr_t>(b);
            const unsigned long long* w = reinterpret_cast<const unsigned long long*>(a & ~uintptr_t{7});
            const uint32_t sh = static_cast<uint32_t>(a & 7) * 8;
            uint64_t v = w[0] >> sh;
            if(sh)
                v |= w[1] << (64 - sh);
            return sz == 8 ? v : (v & ((uint64_t{1} << (8 * sz)) - 1));
        }
        switch(size)
        {
        case 1: return *b;
        case 2: return *reinterpret_cast<const uint16_t*>(b);
        case 4: return *reinterpret_cast<const uint32_t*>(b);
        default: return *reinterpret_cast<const unsigned long long*>(b);
        }
    }

    __device__ __forceinline__ void wt_st(uint8_t* b, uint32_t size, uint64_t v)
    {
        if(size & 0x80)
        {
            for(uint32_t k = 0; k < (size & 0x7F); ++k)
                b[k] = static_cast<uint8_t>(v >> (8 * k));
            return;
        }
        switch(size)
        {
        case 1: *b = static_cast<uint8_t>(v); break;
        case 2: *reinterpret_cast<uint16_t*>(b) = static_cast<uint16_t>(v); break;
        case 4: *reinterpret_cast<uint32_t*>(b) = static_cast<uint32_t>(v); break;
        default: *reinterpret_cast<unsigned long long*>(b) = v; break;
        }
    }

    // one leaf of a warp tile through its host-resolved descriptor; false = generic path
    __device__ __forceinline__ bool wt_fast_leaf(const lamt_params& p, const lamt_leaf& L, const lamt_wfast& W,
                                                 const uint8_t* sbuf, uint8_t* dbuf, uint32_t lane)
    {
        const uint32_t T = p.T;
        auto fix = [&](uint64_t v) -> uint64_t
        {
            if(W.boolean)
                v = v != 0;
            if(W.conv)
                v = lamd::convert_value(lamd::convert_value(v, L.stype, L.ltype), L.ltype, L.dtype);
            return v;
        };
        switch(W.mode)
        {
        case LAMT_WF_SKIP:
            return true;
        case LAMT_WF_PP:
            if(W.sL != 1 || W.dL != 1)
            {
                // AoSoA on either side: block / lane split by a magic multiply
                auto addr = [](uint32_t base, uint32_t bs, uint32_t L, uint32_t ls, uint32_t magic, uint32_t e) {
                    if(L == 1)
                        return base + e * bs;
                    const uint32_t q = __umulhi(e, magic);
                    return base + q * bs + (e - q * L) * ls;
                };
                for(uint32_t e = lane; e < T; e += 32)
                    wt_st(dbuf + addr(W.dbase[0], W.dbs[0], W.dL, W.dls, W.dmagic, e), W.dsz,
                          fix(wt_ld(sbuf + addr(W.sbase[0], W.sbs[0], W.sL, W.sls, W.smagic, e), W.ssz)));
                return true;
            }
            if(((W.ssz | W.dsz) & 0x80) == 0)
            {
                // sizes as template parameters: one typed load and store per element
                auto pp = [&](auto ss, auto ds)
                {
                    using TS = decltype(ss);
                    using TD = decltype(ds);
                    if(!W.conv && !W.boolean)
                        for(uint32_t e = lane; e < T; e += 32)
                            *reinterpret_cast<TD*>(dbuf + W.dbase[0] + e * W.dbs[0])
                                = static_cast<TD>(*reinterpret_cast<const TS*>(sbuf + W.sbase[0] + e * W.sbs[0]));
                    else
                        for(uint32_t e = lane; e < T; e += 32)
                            *reinterpret_cast<TD*>(dbuf + W.dbase[0] + e * W.dbs[0]) = static_cast<TD>(
                                fix(*reinterpret_cast<const TS*>(sbuf + W.sbase[0] + e * W.sbs[0])));
                };
                auto dst = [&](auto ss)
                {
                    switch(W.dsz)
                    {
                    case 1: pp(ss, uint8_t{}); break;
                    case 2: pp(ss, uint16_t{}); break;
                    case 4: pp(ss, uint32_t{}); break;
                    default: pp(ss, static_cast<unsigned long long>(0)); break;
                    }
                };
                switch(W.ssz)
                {
                case 1: dst(uint8_t{}); break;
                case 2: dst(uint16_t{}); break;
                case 4: dst(uint32_t{}); break;
                default: dst(static_cast<unsigned long long>(0)); break;
                }
                return true;
            }
            for(uint32_t e = lane; e < T; e += 32)
                wt_st(dbuf + W.dbase[0] + e * W.dbs[0], W.dsz, fix(wt_ld(sbuf + W.sbase[0] + e * W.sbs[0], W.ssz)));
            return true;
        case LAMT_WF_PS_PLANES:
            for(uint32_t e4 = 4 * lane; e4 < T; e4 += 128)
            {
                uint64_t v[4];
#pragma unroll
                for(int q = 0; q < 4; ++q)
                    v[q] = fix(wt_ld(sbuf + W.sbase[0] + (e4 + q) * W.sbs[0], W.ssz));
#pragma unroll
                for(uint32_t k = 0; k < 8; ++k)
                {
                    if(k >= W.dn)
                        break;
                    const uint32_t sh = 8 * k;
                    const uint32_t w = static_cast<uint32_t>((v[0] >> sh) & 0xFF)
                        | static_cast<uint32_t>(((v[1] >> sh) & 0xFF) << 8) | static_cast<uint32_t>(((v[2] >> sh) & 0xFF) << 16)
                        | static_cast<uint32_t>(((v[3] >> sh) & 0xFF) << 24);
                    *reinterpret_cast<uint32_t*>(dbuf + W.dbase[k] + e4) = w;
                }
            }
            return true;
        case LAMT_WF_PS_BYTES:
            for(uint32_t e = lane; e < T; e += 32)
            {
                const uint64_t v = fix(wt_ld(sbuf + W.sbase[0] + e * W.sbs[0], W.ssz));
#pragma unroll
                for(uint32_t k = 0; k < 8; ++k)
                    if(k < W.dn)
                        dbuf[W.dbase[k] + e * W.dbs[k]] = static_cast<uint8_t>(v >> (8 * k));
            }
            return true;
        case LAMT_WF_SP_PLANES:
            for(uint32_t e4 = 4 * lane; e4 < T; e4 += 128)
            {
                uint64_t v[4] = {0, 0, 0, 0};
#pragma unroll
                for(uint32_t k = 0; k < 8; ++k)
                {
                    if(k >= W.sn)
                        break;
                    const uint32_t w = *reinterpret_cast<const uint32_t*>(sbuf + W.sbase[k] + e4);
#pragma unroll
                    for(int q = 0; q < 4; ++q)
                        v[q] |= uint64_t((w >> (8 * q)) & 0xFF) << (8 * k);
                }
#pragma unroll
                for(int q = 0; q < 4; ++q)
                    wt_st(dbuf + W.dbase[0] + (e4 + q) * W.dbs[0], W.dsz, fix(v[q]));
            }
            return true;
        case LAMT_WF_SP_BYTES:
            for(uint32_t e = lane; e < T; e += 32)
            {
                uint64_t v = 0;
#pragma unroll
                for(uint32_t k = 0; k < 8; ++k)
                    if(k < W.sn)
                        v |= uint64_t(sbuf[W.sbase[k] + e * W.sbs[k]]) << (8 * k);
                wt_st(dbuf + W.dbase[0] + e * W.dbs[0], W.dsz, fix(v));
            }
            return true;
        default:
            return false;
        }
    }

    // General warp-tile engine: any pair of tile plans (byte splits, type conversions, mixed
    // leaf sizes, bit-packed sides, non-power-of-two AoSoA, Null).  One warp owns one tile of
    // p.T elements: every stream image of the tile is one contiguous, 16-byte aligned byte
    // range, moved HBM -> smem with 16-byte loads (CH per lane in flight before the first smem
    // store), transformed leaf by leaf in smem (read terminal(s) -> convert -> write
    // terminal(s), the reference's dst.write(src.read), view.cpp:186-188), bit-packed
    // destinations assembled as whole words, then smem -> HBM with 16-byte stores.  One tile
    // per warp and a one-pass grid (the block scheduler walks the address space in order).
    // Chunk c of the source images lives at sbuf + 16 c; p.st[j].pad holds stream j's first
    // chunk index (prefix over the source, and separately over the destination, images).
    template<int CH>
    __global__ void __launch_bounds__(256, 4) k_warp_tile(const __grid_constant__ lamt_params p, uint32_t ntiles)
    {
        extern __shared__ __align__(16) uint8_t wsm[];
        // chunk -> stream table (host-built, shared by the CTA's warps)
        __shared__ __align__(16) uint8_t cst[1024];
        __shared__ uint16_t s_pad[LAMT_WT_MAX_STREAMS];
        __shared__ unsigned long long s_base[8][LAMT_WT_MAX_STREAMS];
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t warp = threadIdx.x >> 5;
        const uint32_t ns = p.nsrc, nd = p.ndst;
        const uint32_t chS = p.wt_chs, chD = p.wt_chd;
        for(uint32_t k = threadIdx.x; k < (chS + chD + 15) / 16; k += blockDim.x)
            reinterpret_cast<uint4*>(cst)[k] = reinterpret_cast<const uint4*>(p.wt_cst)[k];
        for(uint32_t j = threadIdx.x; j < ns + nd; j += blockDim.x)
            s_pad[j] = static_cast<uint16_t>(p.st[j].pad);
        const uint8_t* s_cst = cst;
        const uint8_t* d_cst = cst + chS;
        __syncthreads();
        uint8_t* sbuf = wsm + warp * (p.src_bytes + p.dst_bytes);
        uint8_t* dbuf = sbuf + p.src_bytes;
        unsigned long long* base = s_base[warp];
        // tiles in warp order: at any moment the active warps work on adjacent tiles
        const uint32_t tw = gridDim.x * (blockDim.x >> 5);
        for(uint32_t wt = blockIdx.x * (blockDim.x >> 5) + warp; wt < ntiles; wt += tw)
        {
            const uint64_t t0 = p.begin + uint64_t(wt) * p.T;
            for(uint32_t j = lane; j < ns + nd; j += 32)
                base[j] = p.st[j].gptr + tile_global_off(p.st[j], t0);
            __syncwarp();
            // ---- load: source images, CH 16-byte chunks per lane in flight ----
            for(uint32_t c0 = 0; c0 < chS; c0 += 32 * CH)
            {
                uint4 v[CH];
    #pragma unroll
                for(int u = 0; u < CH; ++u)
                {
                    const uint32_t c = c0 + u * 32 + lane;
                    if(c < chS)
                    {
                        const uint32_t j = s_cst[c];
                        v[u] = __ldcs(reinterpret_cast<const uint4*>(base[j]) + (c - s_pad[j]));
                    }
                }
    #pragma unroll
                for(int u = 0; u < CH; ++u)
                {
                    const uint32_t c = c0 + u * 32 + lane;
                    if(c < chS)
                        reinterpret_cast<uint4*>(sbuf)[c] = v[u];
                }
            }
            if(p.dst_holes) // destination images with padding: start from their current bytes
                for(uint32_t j = ns; j < ns + nd; ++j)
                    if(p.st[j].preload)
                    {
                        const uint4* g = reinterpret_cast<const uint4*>(base[j]);
                        uint4* sm = reinterpret_cast<uint4*>(dbuf + p.st[j].smem_off);
                        for(uint32_t c = lane; c < (p.st[j].tile_bytes >> 4); c += 32)
                            sm[c] = __ldcs(g + c);
                    }
            __syncwarp();
            // ---- transform ----
            for(uint32_t f = 0; f < p.nleaves; ++f)
            {
                const lamt_leaf& L = p.leaf[f];
                if(L.dkind == LAMT_K_NULL)
                    continue;
                if(wt_fast_leaf(p, L, p.wf[f], sbuf, dbuf, lane))
                    continue;
                for(uint32_t e = lane; e < p.T; e += 32)
                {
                    uint64_t v = tile_read(p, L, sbuf, e);
                    v = lamd::convert_value(v, L.stype, L.ltype);
                    v = lamd::convert_value(v, L.ltype, L.dtype);
                    tile_write(p, L, dbuf, e, v);
                }
            }
            __syncwarp();
            if(p.any_bits)
            {
                for(uint32_t j = ns; j < ns + nd; ++j)
                    if(p.st[j].kind == 1)
                        pack_words(p.st[j], dbuf, p.T, lane, 32);
                __syncwarp();
            }
            // ---- store: destination images (contiguous in dbuf, chunk c at dbuf + 16 c) ----
            for(uint32_t c = lane; c < chD; c += 32)
            {
                const uint32_t j = d_cst[c];
                __stcs(reinterpret_cast<uint4*>(base[j]) + (c - s_pad[j]), reinterpret_cast<const uint4*>(dbuf)[c]);
            }
            __syncwarp();
        }
    }

    cudaError_t warp_tile(const lamt_params& p, uint32_t ntiles, cudaStream_t s)
    {
        const uint32_t warps = 8;
        const size_t smem = static_cast<size_t>(warps) * (p.src_bytes + p.dst_bytes);
        if(cudaError_t e = opt_in_smem(reinterpret_cast<const void*>(k_warp_tile<8>), smem); e != cudaSuccess)
            return e;
        const unsigned grid = stream_grid((uint64_t(ntiles) + warps - 1) / warps, "LAMB_WT_CTAS", 8);
        k_warp_tile<8><<<grid, warps * 32, smem, s>>>(p, ntiles);
        count_launch();
        return cudaGetLastError();
    }

    cudaError_t uniform_warp(const lamt_params& p, uint32_t ntiles, cudaStream_t s)
    {
        int dev = 0;
        cudaGetDevice(&dev);
        const uint32_t perWarp = p.src_bytes + p.dst_bytes;
        const uint32_t warps = 8;
        const size_t smem = static_cast<size_t>(warps) * perWarp;
        auto kern = p.usize == 4 ? k_uniform_warp<uint32_t, 4> : k_uniform_warp<unsigned long long, 4>;
        if(cudaError_t e = opt_in_smem(reinterpret_cast<const void*>(kern), smem); e != cudaSuccess)
            return e;
        int occ = 0;
        if(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, warps * 32, smem) != cudaSuccess || occ < 1)
            occ = 1;
        uint64_t grid = static_cast<uint64_t>(sm_count(dev)) * occ;
        const uint64_t need = (ntiles + warps - 1) / warps;
        if(grid > need)
            grid = need;
        kern<<<static_cast<unsigned>(grid), warps * 32, smem, s>>>(p, ntiles);
        count_launch();
        return cudaGetLastError();
    }

    cudaError_t uniform_direct(const lamt_params& p, uint64_t n, cudaStream_t s)
    {
        int dev = 0;
        cudaGetDevice(&dev);
        const unsigned grid = stream_grid((n + 511) / 512, "LAMB_UDIRECT_CTAS", 32); // grid-stride keeps L1 reuse; one-pass loses 28%
        if(p.usize == 4)
            k_uniform_direct<uint32_t, 2><<<grid, 256, 0, s>>>(p, n);
        else
            k_uniform_direct<unsigned long long, 2><<<grid, 256, 0, s>>>(p, n);
        count_launch();
        return cudaGetLastError();
    }

    cudaError_t tile_copy(const lamt_params& p, uint32_t smemBytes, uint32_t ctasPerSm, cudaStream_t s)
    {
        if(p.ntiles == 0)
            return cudaSuccess;
        int dev = 0;
        cudaGetDevice(&dev);
        if(cudaError_t e = opt_in_smem(reinterpret_cast<const void*>(k_tile_copy), smemBytes); e != cudaSuccess)
            return e;
        const uint32_t sms = static_cast<uint32_t>(sm_count(dev));
        // persistent grid: exactly the CTAs that are co-resident (a second wave would serialise)
        int occ = 0;
        cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tile_copy, static_cast<int>(p.threads + 32),
                                                                       smemBytes);
        if(oe != cudaSuccess || occ < 1)
            occ = 1;
        const uint32_t perSm = ctasPerSm < static_cast<uint32_t>(occ) ? ctasPerSm : static_cast<uint32_t>(occ);
        uint64_t grid = static_cast<uint64_t>(sms) * perSm;
        if(grid > p.ntiles)
            grid = p.ntiles;
        k_tile_copy<<<static_cast<unsigned>(grid), p.threads + 32, smemBytes, s>>>(p);
        count_launch();
        return cudaGetLastError();
    }
} // namespace lamk
