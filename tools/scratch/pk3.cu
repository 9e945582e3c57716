#include <cstdio>
#include <cstdlib>
__global__ void k(const float* a, unsigned* bad, int n)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if(i >= n) return;
    const float* q = a + 8 * i;
    float px = q[0], qx = q[3], qx2 = q[7];
    // scalar
    const float dxs = __fsub_rn(px, qx);
    const float d2s = __fadd_rn(0.01f, __fmul_rn(dxs, dxs));
    const float d6s = __fmul_rn(__fmul_rn(d2s, d2s), d2s);
    const float invs = __frcp_rn(__fsqrt_rn(d6s));
    const float stss = __fmul_rn(__fmul_rn(q[6], invs), 0.0001f);
    const float cxs = __fmul_rn(dxs, stss);
    // packed
    const float2 dx = __fadd2_rn(make_float2(px, px), make_float2(-qx, -qx2));
    const float2 d2 = __fadd2_rn(make_float2(0.01f, 0.01f), __fmul2_rn(dx, dx));
    const float2 d6 = __fmul2_rn(__fmul2_rn(d2, d2), d2);
    const float2 inv = make_float2(__frcp_rn(__fsqrt_rn(d6.x)), __frcp_rn(__fsqrt_rn(d6.y)));
    const float2 sts = __fmul2_rn(__fmul2_rn(make_float2(q[6], q[5]), inv), make_float2(0.0001f, 0.0001f));
    const float2 cx = __fmul2_rn(dx, sts);
    if(__float_as_uint(dx.x) != __float_as_uint(dxs)) atomicAdd(bad + 0, 1);
    if(__float_as_uint(d2.x) != __float_as_uint(d2s)) atomicAdd(bad + 1, 1);
    if(__float_as_uint(d6.x) != __float_as_uint(d6s)) atomicAdd(bad + 2, 1);
    if(__float_as_uint(inv.x) != __float_as_uint(invs)) atomicAdd(bad + 3, 1);
    if(__float_as_uint(sts.x) != __float_as_uint(stss)) atomicAdd(bad + 4, 1);
    if(__float_as_uint(cx.x) != __float_as_uint(cxs)) atomicAdd(bad + 5, 1);
}
int main()
{
    const int n = 1 << 20;
    float* a; unsigned* bad;
    cudaMallocManaged(&a, n * 32); cudaMallocManaged(&bad, 32);
    srand(2);
    for(int i = 0; i < 8 * n; ++i) a[i] = rand() / (float)RAND_MAX;
    for(int i = 0; i < 8; ++i) bad[i] = 0;
    k<<<n / 256, 256>>>(a, bad, n);
    cudaDeviceSynchronize();
    printf("dx %u d2 %u d6 %u inv %u sts %u cx %u\n", bad[0], bad[1], bad[2], bad[3], bad[4], bad[5]);
}
