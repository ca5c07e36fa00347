#include <cuda_runtime.h>
__global__ void k(float2* o, const float2* a, const float2* b, const float2* c) {
    int i = threadIdx.x;
    o[i] = __fadd2_rn(__fmul2_rn(a[i], b[i]), c[i]);
}
// the workaround used in k_update.cu: product as FFMA2 with a -0 addend
__global__ void k2(float2* o, const float2* a, const float2* b, const float2* c) {
    int i = threadIdx.x;
    o[i] = __fadd2_rn(__ffma2_rn(a[i], b[i], make_float2(-0.0f, -0.0f)), c[i]);
}
