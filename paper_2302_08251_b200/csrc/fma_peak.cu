// FP32 CUDA-core peak microkernel (the n-body roofline denominator):
// independent FFMA chains at full occupancy, timed with CUDA events on the device.
#include "launch.h"

#include "../../include/lamina_b200.h"

namespace lamk
{
    __global__ void __launch_bounds__(256) k_fma_peak(float* out, int iters, float a, float b)
    {
        float x[8];
#pragma unroll
        for(int k = 0; k < 8; ++k)
            x[k] = threadIdx.x * 1e-7f + k;
        for(int i = 0; i < iters; ++i)
        {
#pragma unroll
            for(int k = 0; k < 8; ++k)
                x[k] = fmaf(x[k], a, b); // a ~ 1, b ~ 0: values stay finite
        }
        float s = 0.f;
#pragma unroll
        for(int k = 0; k < 8; ++k)
            s += x[k];
        if(s == 12345.678f)
            out[0] = s;
    }
} // namespace lamk

extern "C" int lam_bench_fma_peak(int device, double seconds, double* tflops)
{
    if(cudaSetDevice(device) != cudaSuccess)
        return LAM_ECUDA;
    int sms = lamk::sm_count(device);
    float* out = nullptr;
    if(cudaMalloc(&out, 16) != cudaSuccess)
        return LAM_ECUDA;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    lamk::k_fma_peak<<<blocks, threads>>>(out, iters, 0.9999999f, 1e-7f); // warm-up
    cudaDeviceSynchronize();
    double flop = 0, ms = 0;
    int reps = 0;
    cudaEventRecord(e0);
    do
    {
        lamk::k_fma_peak<<<blocks, threads>>>(out, iters, 0.9999999f, 1e-7f);
        flop += 2.0 * 8 * iters * double(blocks) * threads;
        ++reps;
        if(reps % 8 == 0)
        {
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float t = 0;
            cudaEventElapsedTime(&t, e0, e1);
            ms = t;
        }
    } while(ms < seconds * 1e3 || reps % 8 != 0);
    lamk::count_launch(reps + 1);
    *tflops = flop / (ms * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? LAM_OK : LAM_ECUDA;
}
