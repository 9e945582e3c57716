// The reference's hand-written n-body baselines (tools/nbody/steps.hpp:124-230,
// runner.cpp:239-323) written for the device the way a CUDA programmer would write them
// without the library: a fixed C++ struct (ManualParticle, AoS) or seven plain arrays
// (ManualSoA), one thread per particle i, j-tiles staged through shared memory, no mapping,
// no accessor, no plan.  They exist to measure what the mapping abstraction costs (or
// gains) on the device -- paper Fig. 3's library-vs-hand-written ratio -- and, in exact
// mode, their checksum text must equal the library layouts' (acceptance.cpp:744-766).
//   EXACT: IEEE-rounded sub/add/mul, __fsqrt_rn and an IEEE division (kernel.hpp:31-40), j in
//          order: bit-identical to the x86 reference built without FMA.
//   FAST : the textbook GPU kernel (FMA, rsqrt, m*dt folded into the tile).
#include "launch.h"

#include <cuda_runtime.h>
#include <stdint.h>

namespace lamk
{
    namespace
    {
        template<typename T>
        struct ManualParticle
        {
            T posX, posY, posZ;
            T velX, velY, velZ;
            T mass;
        };

        __device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
        __device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
        __device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
        __device__ __forceinline__ float inv_sqrt_rn(float a) { return __fdiv_rn(1.0f, __fsqrt_rn(a)); }
        __device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
        __device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
        __device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
        __device__ __forceinline__ double inv_sqrt_rn(double a) { return __ddiv_rn(1.0, __dsqrt_rn(a)); }
        __device__ __forceinline__ float fma_(float a, float b, float c) { return fmaf(a, b, c); }
        __device__ __forceinline__ double fma_(double a, double b, double c) { return fma(a, b, c); }
        __device__ __forceinline__ float rsqrt_(float a) { return rsqrtf(a); }
        __device__ __forceinline__ double rsqrt_(double a) { return rsqrt(a); }

        // pPInteraction (kernel.hpp:15-41) in the reference's operation order
        template<typename T, bool EXACT>
        __device__ __forceinline__ void interact(T pix, T piy, T piz, T& vx, T& vy, T& vz, T qx, T qy, T qz, T qm)
        {
            const T eps2 = static_cast<T>(0.01);
            const T dt = static_cast<T>(0.0001);
            const T dx = sub_rn(pix, qx), dy = sub_rn(piy, qy), dz = sub_rn(piz, qz);
            if constexpr(EXACT)
            {
                const T d2 = add_rn(add_rn(add_rn(eps2, mul_rn(dx, dx)), mul_rn(dy, dy)), mul_rn(dz, dz));
                const T inv = inv_sqrt_rn(mul_rn(mul_rn(d2, d2), d2));
                const T sts = mul_rn(mul_rn(qm, inv), dt);
                vx = add_rn(vx, mul_rn(dx, sts));
                vy = add_rn(vy, mul_rn(dy, sts));
                vz = add_rn(vz, mul_rn(dz, sts));
            }
            else
            {
                const T d2 = fma_(dz, dz, fma_(dy, dy, fma_(dx, dx, eps2)));
                const T ri = rsqrt_(d2);
                const T s = qm * (ri * ri * ri); // qm = m * dt (staged)
                vx = fma_(dx, s, vx);
                vy = fma_(dy, s, vy);
                vz = fma_(dz, s, vz);
            }
        }

        // manualAoSUpdate / manualSoAUpdate (steps.hpp:132-212): the AoS and SoA kernels differ
        // only in where a particle's fields live (Get = struct member / array element)
        template<typename T, bool EXACT, int NT, typename Get, typename Put>
        __device__ __forceinline__ void update_body(uint64_t n, Get get, Put put)
        {
            __shared__ T sx[NT], sy[NT], sz[NT], sm[NT];
            const T dt = static_cast<T>(0.0001);
            const uint64_t i = static_cast<uint64_t>(blockIdx.x) * NT + threadIdx.x;
            const bool live = i < n;
            T pix = 0, piy = 0, piz = 0, vx = 0, vy = 0, vz = 0;
            if(live)
                get(i, pix, piy, piz, vx, vy, vz);
            for(uint64_t j0 = 0; j0 < n; j0 += NT)
            {
                const uint64_t j = j0 + threadIdx.x;
                if(j < n)
                {
                    T a, b, c, d, e, f, m;
                    get(j, a, b, c, d, e, f, &m);
                    sx[threadIdx.x] = a;
                    sy[threadIdx.x] = b;
                    sz[threadIdx.x] = c;
                    sm[threadIdx.x] = EXACT ? m : m * dt;
                }
                __syncthreads();
                const int cnt = n - j0 < static_cast<uint64_t>(NT) ? static_cast<int>(n - j0) : NT;
                if(cnt == NT)
                {
#pragma unroll 8
                    for(int k = 0; k < NT; ++k)
                        interact<T, EXACT>(pix, piy, piz, vx, vy, vz, sx[k], sy[k], sz[k], sm[k]);
                }
                else
                    for(int k = 0; k < cnt; ++k)
                        interact<T, EXACT>(pix, piy, piz, vx, vy, vz, sx[k], sy[k], sz[k], sm[k]);
                __syncthreads();
            }
            if(live)
                put(i, vx, vy, vz);
        }

        template<typename T, bool EXACT, int NT>
        __global__ void __launch_bounds__(NT) k_manual_aos_update(ManualParticle<T>* __restrict__ ps, uint64_t n)
        {
            update_body<T, EXACT, NT>(
                n,
                [&](uint64_t k, T& x, T& y, T& z, T& u, T& v, T& w, T* m = nullptr)
                {
                    const ManualParticle<T>& p = ps[k];
                    x = p.posX;
                    y = p.posY;
                    z = p.posZ;
                    if(m)
                        *m = p.mass;
                    else
                    {
                        u = p.velX;
                        v = p.velY;
                        w = p.velZ;
                    }
                },
                [&](uint64_t k, T u, T v, T w)
                {
                    ps[k].velX = u;
                    ps[k].velY = v;
                    ps[k].velZ = w;
                });
        }

        template<typename T>
        struct SoAPtrs
        {
            T *posX, *posY, *posZ, *velX, *velY, *velZ, *mass;
        };

        template<typename T, bool EXACT, int NT>
        __global__ void __launch_bounds__(NT) k_manual_soa_update(const SoAPtrs<T> ps, uint64_t n)
        {
            update_body<T, EXACT, NT>(
                n,
                [&](uint64_t k, T& x, T& y, T& z, T& u, T& v, T& w, T* m = nullptr)
                {
                    x = ps.posX[k];
                    y = ps.posY[k];
                    z = ps.posZ[k];
                    if(m)
                        *m = ps.mass[k];
                    else
                    {
                        u = ps.velX[k];
                        v = ps.velY[k];
                        w = ps.velZ[k];
                    }
                },
                [&](uint64_t k, T u, T v, T w)
                {
                    ps.velX[k] = u;
                    ps.velY[k] = v;
                    ps.velZ[k] = w;
                });
        }

        // manualAoSMove / manualSoAMove (steps.hpp:167-177, 214-229): p += v * dt, no contraction
        template<typename T>
        __global__ void __launch_bounds__(256) k_manual_aos_move(ManualParticle<T>* __restrict__ ps, uint64_t n)
        {
            const T dt = static_cast<T>(0.0001);
            for(uint64_t i = static_cast<uint64_t>(blockIdx.x) * 256 + threadIdx.x; i < n;
                i += static_cast<uint64_t>(gridDim.x) * 256)
            {
                ManualParticle<T>& p = ps[i];
                p.posX = add_rn(p.posX, mul_rn(p.velX, dt));
                p.posY = add_rn(p.posY, mul_rn(p.velY, dt));
                p.posZ = add_rn(p.posZ, mul_rn(p.velZ, dt));
            }
        }

        template<typename T>
        __global__ void __launch_bounds__(256) k_manual_soa_move(const SoAPtrs<T> ps, uint64_t n)
        {
            const T dt = static_cast<T>(0.0001);
            for(uint64_t i = static_cast<uint64_t>(blockIdx.x) * 256 + threadIdx.x; i < n;
                i += static_cast<uint64_t>(gridDim.x) * 256)
            {
                ps.posX[i] = add_rn(ps.posX[i], mul_rn(ps.velX[i], dt));
                ps.posY[i] = add_rn(ps.posY[i], mul_rn(ps.velY[i], dt));
                ps.posZ[i] = add_rn(ps.posZ[i], mul_rn(ps.velZ[i], dt));
            }
        }

        template<typename T>
        SoAPtrs<T> soa_ptrs(void* base, uint64_t n)
        {
            T* p = static_cast<T*>(base);
            return SoAPtrs<T>{p, p + n, p + 2 * n, p + 3 * n, p + 4 * n, p + 5 * n, p + 6 * n};
        }

        template<typename T>
        void launch_update(bool soa, bool exact, void* base, uint64_t n, cudaStream_t s)
        {
            constexpr int NT = 128;
            const unsigned grid = static_cast<unsigned>((n + NT - 1) / NT);
            if(soa)
                exact ? k_manual_soa_update<T, true, NT><<<grid, NT, 0, s>>>(soa_ptrs<T>(base, n), n)
                      : k_manual_soa_update<T, false, NT><<<grid, NT, 0, s>>>(soa_ptrs<T>(base, n), n);
            else
                exact ? k_manual_aos_update<T, true, NT><<<grid, NT, 0, s>>>(static_cast<ManualParticle<T>*>(base), n)
                      : k_manual_aos_update<T, false, NT><<<grid, NT, 0, s>>>(static_cast<ManualParticle<T>*>(base), n);
        }

        template<typename T>
        void launch_move(bool soa, void* base, uint64_t n, cudaStream_t s)
        {
            int dev = 0;
            cudaGetDevice(&dev);
            const uint64_t want = (n + 255) / 256, cap = static_cast<uint64_t>(sm_count(dev)) * 8;
            const unsigned grid = static_cast<unsigned>(want < cap ? want : cap);
            if(soa)
                k_manual_soa_move<T><<<grid, 256, 0, s>>>(soa_ptrs<T>(base, n), n);
            else
                k_manual_aos_move<T><<<grid, 256, 0, s>>>(static_cast<ManualParticle<T>*>(base), n);
        }
    } // namespace

    // base: n particles, AoS records {pos xyz, vel xyz, mass} or 7 consecutive arrays of n
    cudaError_t nbody_manual_update(bool soa, bool f64, bool exact, void* base, uint64_t n, cudaStream_t s)
    {
        if(n == 0)
            return cudaSuccess;
        f64 ? launch_update<double>(soa, exact, base, n, s) : launch_update<float>(soa, exact, base, n, s);
        count_launch();
        return cudaGetLastError();
    }

    cudaError_t nbody_manual_move(bool soa, bool f64, void* base, uint64_t n, cudaStream_t s)
    {
        if(n == 0)
            return cudaSuccess;
        f64 ? launch_move<double>(soa, base, n, s) : launch_move<float>(soa, base, n, s);
        count_launch();
        return cudaGetLastError();
    }
} // namespace lamk
