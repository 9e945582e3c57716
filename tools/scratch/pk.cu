#include <cstdio>
#include <cstdlib>
#include <cstring>
__global__ void k(const float* a, const float* b, unsigned* bad, int n)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if(2 * i + 1 >= n) return;
    float2 x = make_float2(a[2*i], a[2*i+1]), y = make_float2(b[2*i], b[2*i+1]);
    float2 s = __fadd2_rn(x, y), m = __fmul2_rn(x, y);
    float s0 = __fadd_rn(x.x, y.x), s1 = __fadd_rn(x.y, y.y), m0 = __fmul_rn(x.x, y.x), m1 = __fmul_rn(x.y, y.y);
    if(__float_as_uint(s.x) != __float_as_uint(s0) || __float_as_uint(s.y) != __float_as_uint(s1)) atomicAdd(bad, 1);
    if(__float_as_uint(m.x) != __float_as_uint(m0) || __float_as_uint(m.y) != __float_as_uint(m1)) atomicAdd(bad + 1, 1);
    // chained like the kernel
    float2 d = __fmul2_rn(__fmul2_rn(x, x), x);
    float d0 = __fmul_rn(__fmul_rn(x.x, x.x), x.x);
    if(__float_as_uint(d.x) != __float_as_uint(d0)) atomicAdd(bad + 2, 1);
}
int main()
{
    const int n = 1 << 22;
    float *a, *b; unsigned* bad;
    cudaMallocManaged(&a, n * 4); cudaMallocManaged(&b, n * 4); cudaMallocManaged(&bad, 12);
    srand(1);
    for(int i = 0; i < n; ++i) { a[i] = (rand() / (float)RAND_MAX - 0.5f) * 3; b[i] = (rand() / (float)RAND_MAX - 0.5f) * 1e-3f; }
    memset(bad, 0, 12);
    k<<<n / 512, 256>>>(a, b, bad, n);
    cudaDeviceSynchronize();
    printf("add mismatches %u mul mismatches %u chain %u\n", bad[0], bad[1], bad[2]);
}
