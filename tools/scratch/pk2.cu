#include <cstdio>
#include <cstdlib>
#include <cstring>
__device__ void one(float px, float qx, float qy, float qz, float py, float pz, float w, float& vx)
{
    const float dx = __fsub_rn(px, qx), dy = __fsub_rn(py, qy), dz = __fsub_rn(pz, qz);
    const float d2 = __fadd_rn(__fadd_rn(__fadd_rn(0.01f, __fmul_rn(dx, dx)), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
    const float d6 = __fmul_rn(__fmul_rn(d2, d2), d2);
    const float inv = __frcp_rn(__fsqrt_rn(d6));
    const float sts = __fmul_rn(__fmul_rn(w, inv), 0.0001f);
    vx = __fadd_rn(vx, __fmul_rn(dx, sts));
}
__global__ void k(const float* a, unsigned* bad, int n)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if(i >= n) return;
    const float* q = a + 8 * i;
    float px = q[0], py = q[1], pz = q[2];
    float v1 = 0, v2 = 0;
    one(px, q[3], q[4], q[5], py, pz, q[6], v1);
    one(px, q[7], q[3], q[4], py, pz, q[5], v1);
    // packed
    const float2 dx = __fadd2_rn(make_float2(px, px), make_float2(-q[3], -q[7]));
    const float2 dy = __fadd2_rn(make_float2(py, py), make_float2(-q[4], -q[3]));
    const float2 dz = __fadd2_rn(make_float2(pz, pz), make_float2(-q[5], -q[4]));
    const float2 d2 = __fadd2_rn(__fadd2_rn(__fadd2_rn(make_float2(0.01f, 0.01f), __fmul2_rn(dx, dx)), __fmul2_rn(dy, dy)), __fmul2_rn(dz, dz));
    const float2 d6 = __fmul2_rn(__fmul2_rn(d2, d2), d2);
    const float2 inv = make_float2(__frcp_rn(__fsqrt_rn(d6.x)), __frcp_rn(__fsqrt_rn(d6.y)));
    const float2 sts = __fmul2_rn(__fmul2_rn(make_float2(q[6], q[5]), inv), make_float2(0.0001f, 0.0001f));
    const float2 cx = __fmul2_rn(dx, sts);
    v2 = __fadd_rn(__fadd_rn(v2, cx.x), cx.y);
    if(__float_as_uint(v1) != __float_as_uint(v2)) { unsigned k = atomicAdd(bad, 1); if (k < 4) printf("%d: %a %a dx %a %a\n", i, v1, v2, dx.x, dx.y); }
}
int main()
{
    const int n = 1 << 20;
    float* a; unsigned* bad;
    cudaMallocManaged(&a, n * 32); cudaMallocManaged(&bad, 4);
    srand(2);
    for(int i = 0; i < 8 * n; ++i) a[i] = rand() / (float)RAND_MAX;
    *bad = 0;
    k<<<n / 256, 256>>>(a, bad, n);
    cudaDeviceSynchronize();
    printf("mismatches %u / %d\n", *bad, n);
}
