// Example user kernels on the device API (include/lamina_b200_device.cuh), built into
// _lib/liblamina_b200_demo.so and exercised by tests/test_gpu_device_api.py.  They take the
// device plan of a lam_view (lam_view_device_plan) and work through any mapping.
#include "../../include/lamina_b200_device.cuh"

#include <cuda_runtime.h>

using namespace lamina_b200;

namespace
{
    // v[i].leaf *= factor through View::load/store semantics (any mapping, instrumented)
    __global__ void k_scale(DeviceView v, uint32_t leaf, float factor)
    {
        for(uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < v.elementCount();
            i += uint64_t(gridDim.x) * blockDim.x)
            v.store<float>(i, leaf, v.load<float>(i, leaf) * factor);
    }

    // v[i].leaf += add through the direct physical accessor (not instrumented)
    __global__ void k_phys_add(DeviceView v, uint32_t leaf, float add)
    {
        const PhysLeaf<float> a(v, leaf);
        for(uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < v.elementCount();
            i += uint64_t(gridDim.x) * blockDim.x)
            a[i] += add;
    }

    // record-tile copy of the 7-leaf f32 particle record: src -> smem tile -> dst
    __global__ void k_tile_copy7(DeviceView src, DeviceView dst)
    {
        constexpr int N = 64;
        __shared__ SmemRecordTile<float, 7, N> tile;
        const uint32_t leaves[7] = {0, 1, 2, 3, 4, 5, 6};
        for(uint64_t i0 = blockIdx.x * uint64_t(N); i0 < src.elementCount(); i0 += uint64_t(gridDim.x) * N)
        {
            const uint64_t left = src.elementCount() - i0;
            const uint32_t count = left < N ? static_cast<uint32_t>(left) : N;
            tile.load(src, i0, count, leaves);
            __syncthreads();
            tile.store(dst, i0, count, leaves);
            __syncthreads();
        }
    }

    unsigned grid_for(uint64_t n)
    {
        const uint64_t g = (n + 255) / 256;
        return static_cast<unsigned>(g == 0 ? 1 : (g > 4096 ? 4096 : g));
    }
} // namespace

extern "C"
{
    int lam_demo_scale(const void* plan, uint64_t n, uint32_t leaf, float factor, void* stream)
    {
        k_scale<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
            DeviceView{static_cast<const lamp_view*>(plan)}, leaf, factor);
        return static_cast<int>(cudaGetLastError());
    }

    int lam_demo_phys_add(const void* plan, uint64_t n, uint32_t leaf, float add, void* stream)
    {
        k_phys_add<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
            DeviceView{static_cast<const lamp_view*>(plan)}, leaf, add);
        return static_cast<int>(cudaGetLastError());
    }

    int lam_demo_tile_copy7(const void* src, const void* dst, uint64_t n, void* stream)
    {
        const uint64_t g = (n + 63) / 64;
        k_tile_copy7<<<static_cast<unsigned>(g == 0 ? 1 : (g > 4096 ? 4096 : g)), 128, 0,
                       static_cast<cudaStream_t>(stream)>>>(DeviceView{static_cast<const lamp_view*>(src)},
                                                            DeviceView{static_cast<const lamp_view*>(dst)});
        return static_cast<int>(cudaGetLastError());
    }
}
