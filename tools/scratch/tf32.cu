// Does cvt.rn.tf32.f32 (RNE to e8m10 in the top 19 bits) equal the reference's floatEncode(f, 8, 10)
// (= lamd::encode_e8m10_f32) on every non-NaN f32?  Exhaustive over 2^32 inputs.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t enc_ref(uint32_t b)
{
    const uint32_t s = (b >> 31) << 18;
    const uint32_t a = b & 0x7FFFFFFFu;
    const uint32_t r = (a + 0xFFFu + ((a >> 13) & 1u)) >> 13;
    return s | (a > 0x7F800000u ? 0x3FE00u : r);
}
__device__ __forceinline__ uint32_t enc_cvt(uint32_t b)
{
    uint32_t t;
    asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(t) : "f"(__uint_as_float(b)));
    const uint32_t a = b & 0x7FFFFFFFu;
    return a > 0x7F800000u ? (((b >> 31) << 18) | 0x3FE00u) : (t >> 13);
}
__global__ void k(unsigned long long* bad)
{
    for(uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < (1ull << 32); b += (uint64_t)gridDim.x * blockDim.x)
        if(enc_ref((uint32_t)b) != enc_cvt((uint32_t)b))
            atomicAdd(bad, 1ull);
}
int main()
{
    unsigned long long* bad;
    cudaMallocManaged(&bad, 8);
    *bad = 0;
    k<<<148 * 16, 256>>>(bad);
    cudaError_t e = cudaDeviceSynchronize();
    printf("err %d mismatches %llu\n", (int)e, *bad);
}
