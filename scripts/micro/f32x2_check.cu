// Compare packed fp32x2 intrinsics with their scalar IEEE counterparts.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
__global__ void k(const float* a, const float* b, const float* c, int n, int* bad) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * i + 1 >= n) return;
    float2 A = make_float2(a[2*i], a[2*i+1]), B = make_float2(b[2*i], b[2*i+1]), C = make_float2(c[2*i], c[2*i+1]);
    float2 m = __fmul2_rn(A, B), s = __fadd2_rn(A, B), f = __ffma2_rn(A, B, C);
    if (__float_as_uint(m.x) != __float_as_uint(__fmul_rn(A.x, B.x)) || __float_as_uint(m.y) != __float_as_uint(__fmul_rn(A.y, B.y))) atomicAdd(bad, 1);
    if (__float_as_uint(s.x) != __float_as_uint(__fadd_rn(A.x, B.x)) || __float_as_uint(s.y) != __float_as_uint(__fadd_rn(A.y, B.y))) atomicAdd(bad + 1, 1);
    if (__float_as_uint(f.x) != __float_as_uint(__fmaf_rn(A.x, B.x, C.x)) || __float_as_uint(f.y) != __float_as_uint(__fmaf_rn(A.y, B.y, C.y))) atomicAdd(bad + 2, 1);
}
int main() {
    const int n = 1 << 22;
    float *a, *b, *c; int* bad;
    cudaMallocManaged(&a, n * 4); cudaMallocManaged(&b, n * 4); cudaMallocManaged(&c, n * 4); cudaMallocManaged(&bad, 12);
    srand(1);
    for (int i = 0; i < n; ++i) {
        unsigned r1 = (unsigned)rand() * 2654435761u ^ rand(), r2 = (unsigned)rand() * 40503u ^ rand(), r3 = rand() * 7919u ^ rand();
        // mixture: normal values, tiny values (denormal products), exact denormals
        int kind = i % 4;
        a[i] = kind == 3 ? __builtin_bit_cast(float, r1 & 0x807fffffu) : (float)((int)(r1 % 2000001) - 1000000) * 1e-6f * (kind == 2 ? 1e-20f : 1.f);
        b[i] = (float)((int)(r2 % 2000001) - 1000000) * 1e-6f * (kind == 2 ? 1e-20f : 1.f);
        c[i] = (float)((int)(r3 % 2000001) - 1000000) * 1e-6f * (kind >= 2 ? 1e-38f : 1.f);
    }
    memset(bad, 0, 12);
    k<<<(n / 2 + 255) / 256, 256>>>(a, b, c, n, bad);
    cudaDeviceSynchronize();
    printf("mismatch pairs: fmul2 %d  fadd2 %d  ffma2 %d  (of %d)\n", bad[0], bad[1], bad[2], n / 2);
    // which kinds?
    return 0;
}
