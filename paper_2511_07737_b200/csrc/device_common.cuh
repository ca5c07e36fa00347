// device_common.cuh - device helpers shared by the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tsat_internal.h"

namespace tsat {

// Philox4x32-10 (Salmon et al., SC'11), 10 rounds, in place.
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
        uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
        uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
__device__ __forceinline__ float warp_maxf(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

// Block-wide int64 sum + float max (blockDim multiple of 32, <= 1024).
__device__ __forceinline__ void block_sum_max(long long& s, float& mx, long long* sh_s, float* sh_m) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    s = warp_sum(s);
    mx = warp_maxf(mx);
    if (lane == 0) { sh_s[warp] = s; sh_m[warp] = mx; }
    __syncthreads();
    if (warp == 0) {
        long long a = lane < nw ? sh_s[lane] : 0;
        float b = lane < nw ? sh_m[lane] : 0.0f;
        a = warp_sum(a);
        b = warp_maxf(b);
        if (lane == 0) { sh_s[0] = a; sh_m[0] = b; }
    }
    __syncthreads();
    s = sh_s[0];
    mx = sh_m[0];
    __syncthreads();
}

// Named barrier over `nthreads` threads (a warp group); id 1..15.
__device__ __forceinline__ void group_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ceil(log2(x)) for finite x > 0, exactly.
__device__ __forceinline__ int ceil_log2(double x) {
    int e;
    double f = frexp(x, &e);
    return (f == 0.5) ? e - 1 : e;
}

// Eq. 5 row statistics from the exact fixed-point row sum Q (R3, R10).
__device__ __forceinline__ void row_finish(long long Q, const MethodConsts& mc, double* d, double* rho,
                                           unsigned char* guard) {
    if (!mc.normalize) { *d = 1.0; *rho = 1.0; *guard = 1; return; }
    double mu = ((double)Q * 2.3283064365386963e-10) / (double)mc.Nglobal;
    double a = fabs(mu);
    double mag = a > mc.eps_norm ? a : mc.eps_norm;
    double dd = mu >= 0.0 ? mag : -mag;
    *d = dd;
    *rho = 1.0 / dd;
    *guard = (a <= mc.eps_norm) ? 1 : 0;
}

// In-register 32x32 bit-matrix transpose: afterwards bit j of A[i] equals
// bit i of the original A[j] (bit 0 = least significant).
__device__ __forceinline__ void transpose32(uint32_t (&A)[32]) {
    uint32_t m = 0x0000FFFFu;
#pragma unroll
    for (int j = 16; j != 0; j >>= 1, m ^= (m << j)) {
#pragma unroll
        for (int k = 0; k < 32; k = (k + j + 1) & ~j) {
            uint32_t t = ((A[k] >> j) ^ A[k + j]) & m;
            A[k] ^= (t << j);
            A[k + j] ^= t;
        }
    }
}

// Bit-sliced signed counters (B planes, two's complement): add / subtract a
// 0/1 mask (one bit per candidate of a 32-candidate word).
template <int B>
__device__ __forceinline__ void vc_inc(uint32_t (&c)[B], uint32_t m) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
        uint32_t t = c[b] & m;
        c[b] ^= m;
        m = t;
    }
}
template <int B>
__device__ __forceinline__ void vc_dec(uint32_t (&c)[B], uint32_t m) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
        uint32_t t = ~c[b] & m;
        c[b] ^= m;
        m = t;
    }
}

// Bit-sliced addition of a 0/1 mask into an NP-plane unsigned count.
template <int NP>
__device__ __forceinline__ void bs_add(uint32_t (&s)[NP], uint32_t x) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        uint32_t t = s[p] & x;
        s[p] ^= x;
        x = t;
    }
}

// Mask of candidates whose NP-plane count equals r.
template <int NP>
__device__ __forceinline__ uint32_t bs_eq(const uint32_t (&s)[NP], int r) {
    uint32_t m = 0xffffffffu;
#pragma unroll
    for (int p = 0; p < NP; ++p) m &= ((r >> p) & 1) ? s[p] : ~s[p];
    return m;
}

}  // namespace tsat
