/* lamina_b200 device API: View / RecordRef-style access from USER kernels (sm_100a).
 *
 * The GPU analogue of lamina::View::read/write/load/store (core/include/lamina/view.hpp:144-181),
 * of the batched leaf transfers loadLeafLanes/loadSimd (core/include/lamina/simd.hpp:198-236,
 * core/src/simd.cpp:48-76) and of the n-body runner's accessors (tools/nbody/accessors.hpp:26-93).
 * A user kernel receives the device plan of a view (lam_view_device_plan, include/lamina_b200.h)
 * and reads / writes elements through ANY mapping the grammar can express, with the same value
 * semantics as the reference (bit packing, minifloats, ChangeType conversions, byte splits, Null)
 * and the same instrumentation (a FieldAccessCount counts every read()/write(); a Heatmap counts the
 * access ranges).
 *
 *   __global__ void k(lamina_b200::DeviceView v) {
 *       uint64_t i = ...;
 *       float m = v.load<float>(i, 6);                       // any mapping, counted
 *       lamina_b200::PhysLeaf<float> px(v, 0);                // direct accessor (physical leaf)
 *       px[i] += 1.0f;                                        // not counted (like a raw pointer)
 *   }
 *
 * Types: load<T>/store<T> require T to match the leaf's scalar kind (the reference throws "type
 * mismatch", view.hpp:154-181; on the device a mismatch traps).  Element indices are linear
 * (row-major, extents.cpp:94-103).
 *
 * SmemRecordTile<T, NL, N> is a shared-memory view with compile-time extents: N records x NL
 * leaves of type T in SoA order, filled / drained cooperatively by a CTA through the mapping.
 * The library's own n-body kernels (csrc/nbody.cu) stage their j-tiles in the same shape
 * (compile-time extents, filled through resolved leaf accessors) but as hand-packed float4 /
 * negated FP32x2-pair arrays that the packed-FMA inner loop consumes directly, not through this
 * type; SmemRecordTile is exercised by user kernels (examples/device_view_demo.cu,
 * tests/test_gpu_device_api.py).
 */
#pragma once

#include "../paper_2302_08251_b200/csrc/device_common.cuh"
#include "../paper_2302_08251_b200/csrc/lam_plan.h"

namespace lamina_b200
{
    template<typename T>
    struct ScalarKind;
#define LAMB_KIND(T, K)                                                                                                 \
    template<>                                                                                                         \
    struct ScalarKind<T>                                                                                               \
    {                                                                                                                  \
        static constexpr int value = K;                                                                                \
    };
    LAMB_KIND(int8_t, lamd::I8)
    LAMB_KIND(int16_t, lamd::I16)
    LAMB_KIND(int32_t, lamd::I32)
    LAMB_KIND(long long, lamd::I64)
    LAMB_KIND(uint8_t, lamd::U8)
    LAMB_KIND(uint16_t, lamd::U16)
    LAMB_KIND(uint32_t, lamd::U32)
    LAMB_KIND(unsigned long long, lamd::U64)
    LAMB_KIND(float, lamd::F32)
    LAMB_KIND(double, lamd::F64)
    LAMB_KIND(bool, lamd::BOOL)
#undef LAMB_KIND

    template<typename T>
    __device__ __forceinline__ T from_bits(uint64_t b)
    {
        T v;
        if constexpr(sizeof(T) == 8)
            memcpy(&v, &b, 8);
        else if constexpr(sizeof(T) == 4)
        {
            const uint32_t w = static_cast<uint32_t>(b);
            memcpy(&v, &w, 4);
        }
        else if constexpr(sizeof(T) == 2)
        {
            const uint16_t w = static_cast<uint16_t>(b);
            memcpy(&v, &w, 2);
        }
        else
        {
            const uint8_t w = static_cast<uint8_t>(b);
            memcpy(&v, &w, 1);
        }
        return v;
    }

    template<typename T>
    __device__ __forceinline__ uint64_t to_bits(T v)
    {
        if constexpr(sizeof(T) == 8)
        {
            uint64_t b;
            memcpy(&b, &v, 8);
            return b;
        }
        else if constexpr(sizeof(T) == 4)
        {
            uint32_t b;
            memcpy(&b, &v, 4);
            return b;
        }
        else if constexpr(sizeof(T) == 2)
        {
            uint16_t b;
            memcpy(&b, &v, 2);
            return b;
        }
        else
        {
            uint8_t b;
            memcpy(&b, &v, 1);
            return b;
        }
    }

    /// A view inside a kernel: the lowered mapping plan of a lam_view (pass by value).
    struct DeviceView
    {
        const lamp_view* plan;

        __device__ uint64_t elementCount() const
        {
            return plan->n;
        }
        __device__ uint32_t leafCount() const
        {
            return plan->nleaves;
        }
        /// scalar kind of the leaf's logical value (lamd::F32 == LAM_F32, ...)
        __device__ int leafKind(uint32_t leaf) const
        {
            return plan->nodes[plan->roots[leaf]].type;
        }

        /// View::read(i, f) as storage bits of the leaf's kind (ScalarValue::storageBits)
        __device__ uint64_t readBits(uint64_t i, uint32_t leaf) const
        {
            const lamd::ViewCtx c = lamd::make_ctx(plan);
            if(plan->fac)
                atomicAdd(plan->fac_counters + leaf, 1ull);
            return lamd::read_node<LAMP_MAX_DEPTH>(c, plan->roots[leaf], i);
        }

        /// View::write(i, f, value) from storage bits of the leaf's kind
        __device__ void writeBits(uint64_t i, uint32_t leaf, uint64_t bits) const
        {
            const lamd::ViewCtx c = lamd::make_ctx(plan);
            if(plan->fac)
                atomicAdd(plan->fac_counters + plan->nleaves + leaf, 1ull);
            lamd::write_node<LAMP_MAX_DEPTH>(c, plan->roots[leaf], i, bits);
        }

        /// View::load<T>(i, f): T must be the leaf's type (traps otherwise: "type mismatch")
        template<typename T>
        __device__ T load(uint64_t i, uint32_t leaf) const
        {
            if(leafKind(leaf) != ScalarKind<T>::value)
                __trap();
            return from_bits<T>(readBits(i, leaf));
        }

        /// View::store<T>(i, f, v)
        template<typename T>
        __device__ void store(uint64_t i, uint32_t leaf, T v) const
        {
            if(leafKind(leaf) != ScalarKind<T>::value)
                __trap();
            writeBits(i, leaf, to_bits<T>(v));
        }

        /// true when the leaf is stored physically and naturally aligned (PhysLeaf is usable)
        __device__ bool isPhysical(uint32_t leaf) const
        {
            const lamp_node nd = plan->nodes[plan->roots[leaf]];
            return nd.kind == LAMP_PHYS && (nd.flags & LAMP_FLAG_ALIGNED);
        }
    };

    /// Direct accessor of one physical leaf: the mapping's offset function resolved into
    /// registers once (AoS: base + i*recordSize; SoA: base + i*size; AoSoA<L>: block/lane),
    /// like the reference's AffineAccessor / AoSoAAccessor (tools/nbody/accessors.hpp:26-93).
    /// Accesses through it are raw memory accesses: not instrumented.
    template<typename T>
    struct PhysLeaf
    {
        uint8_t* base;
        uint64_t stride;
        uint32_t shift, mask, ls, div;

        __device__ PhysLeaf(const DeviceView& v, uint32_t leaf)
        {
            const lamp_node nd = v.plan->nodes[v.plan->roots[leaf]];
            if(nd.kind != LAMP_PHYS || !(nd.flags & LAMP_FLAG_ALIGNED) || lamd::scalar_size(nd.type) != sizeof(T))
                __trap(); // "computed leaf has no physical offset" (mapping.cpp:10)
            const lamp_stream st = v.plan->streams[nd.stream];
            base = v.plan->stream_ptr[nd.stream] + nd.a;
            stride = st.block_stride;
            shift = 0;
            mask = 0;
            ls = 0;
            div = 0;
            if(st.lanes != 1)
            {
                ls = nd.b;
                if(st.lane_shift != 0xFFFFFFFFu)
                {
                    shift = st.lane_shift;
                    mask = static_cast<uint32_t>(st.lanes - 1);
                }
                else
                    div = static_cast<uint32_t>(st.lanes);
            }
        }

        __device__ __forceinline__ T* ptr(uint64_t i) const
        {
            uint64_t blk, lane;
            if(div)
            {
                blk = i / div;
                lane = i - blk * div;
            }
            else
            {
                blk = i >> shift;
                lane = i & mask;
            }
            return reinterpret_cast<T*>(base + blk * stride + lane * ls);
        }

        __device__ __forceinline__ T& operator[](uint64_t i) const
        {
            return *ptr(i);
        }
    };

    /// Shared-memory record tile with compile-time extents (N records x NL leaves of T, SoA).
    /// load/store move records [i0, i0 + count) between the view (through its mapping, counted
    /// like View::read/write) and the tile, cooperatively over the CTA; call __syncthreads()
    /// between a load and the first use of the tile.
    template<typename T, int NL, int N>
    struct SmemRecordTile
    {
        T v[NL][N];

        __device__ void load(const DeviceView& view, uint64_t i0, uint32_t count, const uint32_t (&leaves)[NL])
        {
            for(uint32_t k = threadIdx.x; k < static_cast<uint32_t>(N) * NL; k += blockDim.x)
            {
                const uint32_t r = k % N, f = k / N;
                v[f][r] = r < count ? view.load<T>(i0 + r, leaves[f]) : T(0);
            }
        }

        __device__ void store(const DeviceView& view, uint64_t i0, uint32_t count,
                              const uint32_t (&leaves)[NL]) const
        {
            for(uint32_t k = threadIdx.x; k < static_cast<uint32_t>(N) * NL; k += blockDim.x)
            {
                const uint32_t r = k % N, f = k / N;
                if(r < count)
                    view.store<T>(i0 + r, leaves[f], v[f][r]);
            }
        }
    };
} // namespace lamina_b200
