// upd_common.cuh - helpers of the fused update kernels (k_update.cu, k_update_blk.cu):
// rows (a7) STE backward fold, (a8) Eq. 5 Jacobian terms, (a9) AdamW streams
// (§3.2 l.189-191, l.226; §4.1 l.255-269).
#pragma once
#include <cstdio>
#include <cstdlib>

#include "device_common.cuh"

#ifndef TSAT_UNI3
#define TSAT_UNI3 2
#endif
#ifndef TSAT_3B_UNROLL
#define TSAT_3B_UNROLL 1
#endif
constexpr int kUnroll3b = TSAT_3B_UNROLL;
#ifndef TSAT_UPD_THREADS8
#define TSAT_UPD_THREADS8 512        // KB = 8 block size bound
#endif
#ifndef TSAT_UPD_THREADS4P
#define TSAT_UPD_THREADS4P 768      // KB = 4 block size bound of the peer-exchange kernel (MODE 2)
#endif
#ifndef TSAT_UPD_THREADS4
#define TSAT_UPD_THREADS4 768       // KB = 4 block size bound (register budget)
#endif
#ifndef TSAT_UPD_THREADS4C6
#define TSAT_UPD_THREADS4C6 896     // KB = 4 with 6-plane counters (c2: k_update -2.5 % vs 8 planes at 768)
#endif

#ifndef TSAT_ANEXT_CS
#define TSAT_ANEXT_CS 1            // next-state bit planes stored streaming (c3: k_update -2 %)
#endif
#ifndef TSAT_BLK_PIPE
#define TSAT_BLK_PIPE 0
#endif
#ifndef TSAT_FOLD_I2F
#define TSAT_FOLD_I2F 1            // counts -> float by I2F.S8 (one op) instead of PRMT + FADD: c4 k_update -1.9 %, c3 -1.4 %, c2 -0.8 %
#endif
#ifndef TSAT_FOLD_DP4A
#define TSAT_FOLD_DP4A 1           // KB = 8: derived bin of the fold by byte dot products (c4 -1.8 %; KB = 4 +3 % at c3, not used)
#endif
#ifndef TSAT_HINTS
#define TSAT_HINTS 1
#endif

namespace tsat {

// Pass 3b's last reads and writes of theta, m, v: with TSAT_HINTS, streaming
// (evict-first) so the bit planes and records keep their L2 lines.
__device__ __forceinline__ float4 ld_last(const float* p) {
#if TSAT_HINTS
    return __ldcs(reinterpret_cast<const float4*>(p));
#else
    return *reinterpret_cast<const float4*>(p);
#endif
}
__device__ __forceinline__ void st_stream(float* p, float4 x) {
#if TSAT_HINTS
    __stcs(reinterpret_cast<float4*>(p), x);
#else
    *reinterpret_cast<float4*>(p) = x;
#endif
}

namespace {
constexpr int kCtr = 8;        // counter planes (int8) in the fused kernel
constexpr int kHubCtrPlain = 11;    // counter planes (int11) in k_hub (kHubSlab = 1023 occurrences)
// planes of a signed count of up to x occurrences: the smallest B with 2^(B-1) - 1 >= x
__host__ __device__ constexpr int signed_planes(int x, int b = 1) { return ((1 << (b - 1)) - 1 >= x) ? b : signed_planes(x, b + 1); }
constexpr int kHubCtrBatched = signed_planes(kHubSlabBatches * 4);  // batched super-chunks: <= kHubSlabBatches * 4 occurrences

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) / 16 * 16; }
}  // namespace

// Raise a kernel's dynamic shared-memory limit to at least `need` bytes.  The
// limit is a process-wide per-function attribute: it only ever grows, so a
// context configured later with a smaller geometry cannot lower it below
// another context's launch.  (TSAT_ATTR_OPTIN: always the opt-in maximum.)
#ifndef TSAT_ATTR_OPTIN
#define TSAT_ATTR_OPTIN 0
#endif
template <typename Kern>
inline cudaError_t set_max_dyn_smem(Kern* k, int need, int optin) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k);
    if (e != cudaSuccess) return e;
    const int target = TSAT_ATTR_OPTIN ? optin - (int)fa.sharedSizeBytes : need;
    if (!TSAT_ATTR_OPTIN && fa.maxDynamicSharedSizeBytes >= target) return cudaSuccess;
    return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, target);
}

// Shared-memory geometry of k_update (host and device agree through this).
__host__ __device__ inline size_t upd_gs_bytes(int KB, int N) { return align16((size_t)KB * N * 4); }
__host__ __device__ inline size_t upd_dpk_words(int N) { return (size_t)N + (N >> 5); }
// nbufs: 2 record buffers (the next row's records land during this row's
// streams), or 1 (staged after this row's gather) when that buys a warp group:
// KB = 8 (shared-memory bound), a compile-time choice (a runtime one costs
// the instruction-cache-bound KB = 8 kernel ~7 %).
__host__ __device__ constexpr int upd_recbufs(int KB) { return KB == 8 ? 1 : 2; }
// parities: 2 for the peer kernel (MODE 2 finishes a row one row late), else 1
// xslots: cluster-split rows (MODE 3) add the group's DSMEM exchange slots
// [2 kinds][kMaxCluster = 16 ranks][2 words] (cluster.cuh) below the scratch.
__host__ __device__ inline size_t upd_group_bytes(int KB, int N, int rec_cap, int nbufs, int parities = 2,
                                                  bool xslots = false) {
    const int NDW = KB == 4 ? 1 : 2;
    // dpk | nbufs record buffers | sign planes [parities][pos, neg][NW] | (slots) | 128 B scratch
    return align16((size_t)NDW * upd_dpk_words(N) * 4) + nbufs * align16((size_t)rec_cap * 4) +
           align16((size_t)2 * parities * (N >> 5) * 4) + (xslots ? 512 : 0) + 128;
}
constexpr int kClusterSlotBytes = 512;

// x * 2^s, exact (== scalbn) when 2^s is a normal double.
__device__ __forceinline__ double times_pow2(double x, int s) {
    if (s >= -1000 && s <= 1000) return x * __longlong_as_double((long long)(1023 + s) << 52);
    return scalbn(x, s);
}

// Signed byte r of u (counts stored as int8) -> exact float: the byte, biased
// by 128, goes into the mantissa of 2^23 (PRMT) and the bias is subtracted.
__device__ __forceinline__ float sbyte_to_float(uint32_t ub, int r) {
    return __uint_as_float(__byte_perm(ub, 0x4B000000u, 0x7540u + (unsigned)r)) - 8388736.0f;
}

// a * b per lane, correctly rounded, never contracted with a following add:
// ptxas fuses FMUL2 + FADD2 into FFMA2 even with --fmad=false (and folds an
// FFMA2 with a -0 addend the same way; scripts/micro/fuse_check.cu), so
// products that feed an add are two scalar __fmul_rn (which ptxas respects).
__device__ __forceinline__ float2 mul2_unfused(float2 a, float2 b) {
    return make_float2(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y));
}

// Per-bin counts of one candidate as exact floats (bytes + derived last bin).
template <int KB>
__device__ __forceinline__ void fold_counts(float (&d)[KB], uint32_t p0, uint32_t p1, int dsum) {
#if TSAT_FOLD_I2F
    // I2F.S8 with a byte selector: one conversion per bin (exact; +0 for 0)
#pragma unroll
    for (int r = 0; r < KB - 1; ++r) d[r] = (float)(int8_t)((r < 4 ? p0 : p1) >> (8 * (r & 3)));
#else
    const uint32_t u0 = p0 ^ 0x80808080u, u1 = p1 ^ 0x80808080u;
#pragma unroll
    for (int r = 0; r < KB - 1; ++r) d[r] = sbyte_to_float(r < 4 ? u0 : u1, r & 3);
#endif
    // derived bin: dsum - sum_r d_r as an integer (byte dot products with -1;
    // the unused top byte is 0), made an exact float through the mantissa of
    // 1.5 * 2^23 (|x| < 2^22); +0 for x = 0, as the fp32 subtraction gave
    if (TSAT_FOLD_DP4A == 2) {                       // every KB, I2F conversion (exact: |x| < 2^24)
        int x = __dp4a((int)p0, -1, dsum);
        if (KB == 8) x = __dp4a((int)p1, -1, x);
        d[KB - 1] = (float)x;
    } else if (TSAT_FOLD_DP4A && KB == 8) {
        int x = __dp4a((int)p0, -1, dsum);
        x = __dp4a((int)p1, -1, x);
        d[KB - 1] = __int_as_float(0x4B400000 + x) - 12582912.0f;
    } else {
        float acc = d[0];
#pragma unroll
        for (int r = 1; r < KB - 1; ++r) acc = acc + d[r];     // exact: small integers (never -0)
        d[KB - 1] = (float)dsum - acc;
    }
}

template <int KB>
__device__ __forceinline__ float fold_ints(const int* hubrow, int N, int n, int dsum, const float (&gq)[KB]) {
    float d[KB];
    int acc = 0;
#pragma unroll
    for (int r = 0; r < KB - 1; ++r) { const int x = hubrow[(size_t)r * N + n]; acc += x; d[r] = (float)x; }
    d[KB - 1] = (float)(dsum - acc);
    float G = 0.0f;
#pragma unroll
    for (int r = 0; r < KB; ++r) G = __fmaf_rn(d[r], gq[r], G);
    return G;
}

// Pass 3a of one row: G for every candidate (stored over its counts in dpk),
// and the int64 fixed-point partial sum of J_v = sum_n G theta (R13).
template <int KB, bool HUB>
__device__ __forceinline__ long long pass_fold(const float* __restrict__ trow, uint32_t* dpk, size_t dpkw,
                                               const float* gs, int* hubrow, int N, int Nst, int GT, int tg, int dsum,
                                               bool jvalid, float p2, float* __restrict__ gout, int Ngs) {
    // N candidates from the pointers' origin; Nst = row stride of hubrow, Ngs of gs
    long long I = 0;
    float4 th_nx = (4 * tg < N) ? *reinterpret_cast<const float4*>(trow + 4 * tg) : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int n = 4 * tg; n < N; n += 4 * GT) {
        const float4 th4 = th_nx;
        if (n + 4 * GT < N) th_nx = *reinterpret_cast<const float4*>(trow + n + 4 * GT);
        const float th[4] = {th4.x, th4.y, th4.z, th4.w};
        float4 g4[KB];
#pragma unroll
        for (int r = 0; r < KB; ++r) g4[r] = *reinterpret_cast<const float4*>(gs + (size_t)r * Ngs + n);
        uint32_t* dp = dpk + n + (n >> 5);
        float Gq[4];
        if (HUB) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float gq[KB];
#pragma unroll
                for (int r = 0; r < KB; ++r) gq[r] = q == 0 ? g4[r].x : q == 1 ? g4[r].y : q == 2 ? g4[r].z : g4[r].w;
                Gq[q] = fold_ints<KB>(hubrow, Nst, n + q, dsum, gq);
            }
        } else {
            // candidate pairs: d_r as floats (exact small integers), then the
            // r-ascending FMA chain with packed fp32x2 FMAs (per-lane exact FMA)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float dA[KB], dB[KB];
                fold_counts<KB>(dA, dp[2 * h], KB == 8 ? dp[dpkw + 2 * h] : 0u, dsum);
                fold_counts<KB>(dB, dp[2 * h + 1], KB == 8 ? dp[dpkw + 2 * h + 1] : 0u, dsum);
                float2 G2 = make_float2(0.0f, 0.0f);
#pragma unroll
                for (int r = 0; r < KB; ++r)
                    G2 = __ffma2_rn(make_float2(dA[r], dB[r]),
                                    h == 0 ? make_float2(g4[r].x, g4[r].y) : make_float2(g4[r].z, g4[r].w), G2);
                Gq[2 * h] = G2.x;
                Gq[2 * h + 1] = G2.y;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float G = Gq[q];
            dp[q] = __float_as_uint(G);
            if (jvalid) I += jterm(G, th[q], p2);
        }
        if (gout) *reinterpret_cast<float4*>(gout + n) = make_float4(Gq[0], Gq[1], Gq[2], Gq[3]);
        if (HUB) {
#pragma unroll
            for (int r = 0; r < KB - 1; ++r) *reinterpret_cast<int4*>(hubrow + (size_t)r * Nst + n) = make_int4(0, 0, 0, 0);
        }
    }
    return I;
}

// Bulk prefetch of [p, p + bytes) into L2 (TMA engine; bytes % 16 == 0).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Optional update noise (R17): xi = (x >> 8) 2^-24 - 1/2 with
// x = Philox(key = seed, ctr = (n>>2, v, 1+t, 0))[n & 3].  Out of line: it is
// off by default and would otherwise bloat the hot loop's instruction footprint.
static __device__ __noinline__ float noise_xi(unsigned long long seed, long long ng, int v, long long t) {
    uint32_t xr[4] = {(uint32_t)(ng >> 2), (uint32_t)v, (uint32_t)(1 + t), 0u};
    philox4x32_10(xr, (uint32_t)seed, (uint32_t)(seed >> 32));
    return (float)(xr[ng & 3] >> 8) * 5.9604644775390625e-08f - 0.5f;
}

// 4-byte asynchronous global -> shared copy (LDGSTS) and its group fences.
__device__ __forceinline__ void cp_async4(uint32_t* smem_dst, const uint32_t* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Barrier over one warp group: a warp-sized group only needs __syncwarp, so
// more than 15 groups (the named-barrier limit) can share a CTA.
__device__ __forceinline__ void gsync(int bar, int GT) {
    if (GT == 32) __syncwarp();
    else group_bar(bar, GT);
}

}  // namespace tsat
