// device_common.cuh - device helpers shared by the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tsat_internal.h"

#ifndef TSAT_PLANE_KEEP_BYTES
#define TSAT_PLANE_KEEP_BYTES 48.0e6     // both plane buffers below this: evict-last gathers
#endif

namespace tsat {

// L2 cache policy for the bit-plane gathers (created once per kernel):
// evict-last when both plane buffers fit comfortably in L2 (they are re-read
// by every occurrence), evict-normal otherwise.
#ifndef TSAT_BIN_SKIP
#define TSAT_BIN_SKIP 1              // batched records: skip bins above the batch's clause length
#endif
#ifndef TSAT_ODD_STEP
#define TSAT_ODD_STEP 0              // 1: an odd last literal step skips the absent half (measured c4 k_update +4 %, k_hub +9 %)
#endif
#ifndef TSAT_PLANE_FRAC
#define TSAT_PLANE_FRAC 0            // planes larger than L2: evict-last on this fraction of the lines (0: normal)
#endif
__device__ __forceinline__ unsigned long long plane_policy(bool keep) {
    unsigned long long pol;
    if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#if TSAT_PLANE_FRAC
    else asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(pol) : "f"((float)TSAT_PLANE_FRAC / 100.0f));
#else
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
#endif
    return pol;
}
// Eq. 5 gradient addend (R27b): grad = fmaf(G, rho, addend) with addend = -c;
// normalize 3 (R28, d = mean |theta|): -sign(theta) c, and -0 at theta = 0.
__device__ __forceinline__ float jac_addend(float ncf, float th, bool mag) {
    if (!mag) return ncf;
    return th > 0.0f ? ncf : (th < 0.0f ? -ncf : -0.0f);
}

// Whether both bit-plane buffers ((V + 1) x NW words each) fit comfortably in L2.
__host__ __device__ __forceinline__ bool planes_fit_l2(int V, int NW) {
    return 2.0 * 4.0 * ((double)V + 1.0) * (double)NW <= TSAT_PLANE_KEEP_BYTES;
}
__device__ __forceinline__ uint32_t ld_plane(const uint32_t* p, unsigned long long pol) {
    uint32_t x;
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(x) : "l"(p), "l"(pol));
    return x;
}

// Programmatic dependent launch: wait for the preceding kernel in the stream
// (complete, memory visible) and let the next one be scheduled.  Both are
// no-ops for a kernel launched without the PDL attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

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

// R13 fixed-point scale of J_v: s = 61 - ceil(log2(N occ gmax thmax)),
// clamped to the fp32 exponent range [-126, 127]; p2 = 2^s as fp32.
// Returns false (J_v = 0) when the row has no occurrences or x = 0.
__device__ __forceinline__ bool jscale(long long Nnorm, int occ, double gmax, float thmax, int* s, float* p2) {
    double x = (double)Nnorm * (double)occ;
    x = x * gmax;
    x = x * (double)thmax;
    *s = 0;
    *p2 = 1.0f;
    if (!(occ > 0 && x > 0.0)) return false;
    int e = 61 - ceil_log2(x);
    e = e > 127 ? 127 : (e < -126 ? -126 : e);
    *s = e;
    *p2 = __uint_as_float((uint32_t)(127 + e) << 23);
    return true;
}

// One term of J_v's fixed-point sum (R13): llrintf(G (x) (theta (x) 2^s)),
// both products fp32 round-to-nearest-even.
__device__ __forceinline__ long long jterm(float G, float th, float p2) {
    return __float2ll_rn(__fmul_rn(G, __fmul_rn(th, p2)));
}

// Eq. 5 row statistics from the exact fixed-point row sum Q (R3, R10).
__device__ __forceinline__ void row_finish(long long Q, const MethodConsts& mc, double* d, double* rho,
                                           unsigned char* guard) {
    if (!mc.normalize) { *d = 1.0; *rho = 1.0; *guard = 1; return; }
    double mu = ((double)Q * 2.3283064365386963e-10) / (double)mc.Nnorm;
    double a = fabs(mu);
    double mag = a > mc.eps_norm ? a : mc.eps_norm;
    double dd = mu >= 0.0 ? mag : -mag;
    *d = dd;
    *rho = 1.0 / dd;
    *guard = (a <= mc.eps_norm) ? 1 : 0;
}

// Bitwise select m ? x : y in one LOP3 (ptxas otherwise emits two).
__device__ __forceinline__ uint32_t bsel(uint32_t m, uint32_t x, uint32_t y) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(r) : "r"(m), "r"(x), "r"(y));
    return r;
}

// In-register 32x32 bit-matrix transpose: afterwards bit j of A[i] equals
// bit i of the original A[j] (bit 0 = least significant).
// TSAT_TRANSPOSE_V 1 (2): the 16- and 8-bit stages as byte permutes (2 PRMT
// per pair) and (or not) the 4/2/1-bit stages as shift + one-LOP3 select: ~256
// instead of ~410 operations, yet measured slower on the same box (c3 k_update
// +6 %, c5 N = 8192 k_clause +9 %; c2 -0.5 %), so the shift-xor form stays.
#ifndef TSAT_TRANSPOSE_V
#define TSAT_TRANSPOSE_V 0
#endif
__device__ __forceinline__ void transpose32(uint32_t (&A)[32]) {
#if TSAT_TRANSPOSE_V == 0
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
#else
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const uint32_t a = A[k], b = A[k + 16];
        A[k] = __byte_perm(a, b, 0x5410u);
        A[k + 16] = __byte_perm(a, b, 0x7632u);
    }
#pragma unroll
    for (int k = 0; k < 32; k = (k + 9) & ~8) {
        const uint32_t a = A[k], b = A[k + 8];
        A[k] = __byte_perm(a, b, 0x6240u);
        A[k + 8] = __byte_perm(a, b, 0x7351u);
    }
    uint32_t m = 0x0F0F0F0Fu;
#pragma unroll
    for (int j = 4; j != 0; j >>= 1, m ^= (m << j)) {
#pragma unroll
        for (int k = 0; k < 32; k = (k + j + 1) & ~j) {
#if TSAT_TRANSPOSE_V == 1
            const uint32_t a = A[k], b = A[k + j];
            A[k] = bsel(m, a, b << j);
            A[k + j] = bsel(m, a >> j, b);
#else
            uint32_t t = ((A[k] >> j) ^ A[k + j]) & m;
            A[k] ^= (t << j);
            A[k + j] ^= t;
#endif
        }
    }
#endif
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

// 4 one-bit masks -> their 3-bit bit-sliced sum (s0 + 2 s1 + 4 s2), carry-save.
__device__ __forceinline__ void sum4(uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3, uint32_t& s0, uint32_t& s1,
                                     uint32_t& s2) {
    const uint32_t sa = m0 ^ m1 ^ m2;
    const uint32_t ca = (m0 & m1) | (m2 & (m0 ^ m1));
    s0 = sa ^ m3;
    const uint32_t cb = sa & m3;
    s1 = ca ^ cb;
    s2 = ca & cb;
}

// Signed B-plane counters (two's complement): c += S / c -= S for a bit-sliced
// 3-bit S (ripple of full adders; subtraction adds ~S with carry-in 1).
template <int B>
__device__ __forceinline__ void vc_add3(uint32_t (&c)[B], uint32_t s0, uint32_t s1, uint32_t s2) {
    uint32_t carry = c[0] & s0;
    c[0] ^= s0;
    uint32_t x = c[1];
    c[1] = x ^ s1 ^ carry;
    carry = (x & s1) | (carry & (x ^ s1));
    x = c[2];
    c[2] = x ^ s2 ^ carry;
    carry = (x & s2) | (carry & (x ^ s2));
#pragma unroll
    for (int b = 3; b < B; ++b) {
        const uint32_t t = c[b] & carry;
        c[b] ^= carry;
        carry = t;
    }
}
template <int B>
__device__ __forceinline__ void vc_sub3(uint32_t (&c)[B], uint32_t s0, uint32_t s1, uint32_t s2) {
    uint32_t carry = 0xffffffffu;
    const uint32_t ns[3] = {~s0, ~s1, ~s2};
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        const uint32_t x = c[b];
        c[b] = x ^ ns[b] ^ carry;
        carry = (x & ns[b]) | (carry & (x ^ ns[b]));
    }
#pragma unroll
    for (int b = 3; b < B; ++b) {           // operand bits are all 1 here
        const uint32_t x = c[b];
        c[b] = ~(x ^ carry);
        carry = x | carry;
    }
}

// c += (x0 + 2 x1 + 4 x2 + hi (2^3 + ... + 2^(B-1))) + cin, B-plane ripple of
// full adders; with x = ~S, hi = cin = all ones this is c -= S.
template <int B>
__device__ __forceinline__ void vc_addc(uint32_t (&c)[B], uint32_t x0, uint32_t x1, uint32_t x2, uint32_t hi) {
    uint32_t carry = hi;
    const uint32_t x[3] = {x0, x1, x2};
#pragma unroll
    for (int b = 0; b < B; ++b) {
        const uint32_t y = b < 3 ? x[b] : hi, cb = c[b];
        c[b] = cb ^ y ^ carry;
        carry = (cb & y) | (carry & (cb ^ y));
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

// One record's literal values for one 32-candidate word: own literal plus the
// clause's other literals (codes), as NP count planes.
template <int NP, typename RecFn>
__device__ __forceinline__ void rec_planes(uint32_t (&sp)[NP], RecFn rec, unsigned p, uint32_t hdr, uint32_t own,
                                           const uint32_t* __restrict__ Acur, unsigned NW, unsigned w,
                                           unsigned long long pol) {
    const uint32_t len = hdr >> 1;
    sp[0] = own ^ (0u - (hdr & 1u));
#pragma unroll
    for (int q = 1; q < NP; ++q) sp[q] = 0u;
    for (uint32_t i = 1; i < len; ++i) {
        const uint32_t code = rec(p + i);
        bs_add<NP>(sp, ld_plane(Acur + ((code >> 1) * NW + w), pol) ^ (0u - (code & 1u)));
    }
}

// Signed per-bin counts d_r = cneg[r] - cpos[r], r < NCTR, of one variable's
// occurrence records [0, nrec) for one 32-candidate word w, as B-plane
// two's-complement counters.  Records are sign-sorted (negated first, host
// side), so runs of 4 same-sign records are summed by carry-save adders and
// added (negated) or subtracted (positive) once.  UNI3: every record has 3
// words (uniform 3-SAT), so a group's 8 gathers are issued together.  GROUP
// false: one record at a time (smaller code, for I-cache-bound callers).
template <int NP, int NCTR, int B, bool UNI3, bool GROUP, typename RecFn>
__device__ __forceinline__ void count_occurrences(uint32_t (&cnt)[NCTR][B], RecFn rec, unsigned nrec, uint32_t own,
                                                  const uint32_t* __restrict__ Acur, unsigned NW, unsigned w, unsigned long long pol) {
#pragma unroll
    for (int r = 0; r < NCTR; ++r)
#pragma unroll
        for (int b = 0; b < B; ++b) cnt[r][b] = 0u;
    auto ld = [&](uint32_t code) { return ld_plane(Acur + ((code >> 1) * NW + w), pol) ^ (0u - (code & 1u)); };
    unsigned p = 0;
    while (p < nrec) {
        const uint32_t h0 = rec(p);
        unsigned p4 = 0;
        bool grp = false;
        uint32_t h[4];
        unsigned pp[4];
        h[0] = h0;
        pp[0] = p;
        if (!GROUP) {
        } else if (UNI3) {
            if (p + 12 <= nrec) {
                h[1] = rec(p + 3); h[2] = rec(p + 6); h[3] = rec(p + 9);
                pp[1] = p + 3; pp[2] = p + 6; pp[3] = p + 9;
                p4 = p + 12;
                grp = ((h0 ^ h[3]) & 1u) == 0u;          // signs are monotone in the row
            }
        } else {
            unsigned q = p + (h0 >> 1);
            grp = true;
#pragma unroll
            for (int k = 1; k < 4; ++k) {
                if (q >= nrec) { grp = false; break; }
                h[k] = rec(q);
                pp[k] = q;
                q += h[k] >> 1;
            }
            if (grp) { p4 = q; grp = ((h0 ^ h[3]) & 1u) == 0u; }
        }
        if (grp) {
            uint32_t sp[4][NP];
            if (UNI3) {
                uint32_t x[4][2];
#pragma unroll
                for (int k = 0; k < 4; ++k) { x[k][0] = ld(rec(pp[k] + 1)); x[k][1] = ld(rec(pp[k] + 2)); }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    sp[k][0] = own ^ (0u - (h[k] & 1u));
#pragma unroll
                    for (int q = 1; q < NP; ++q) sp[k][q] = 0u;
                    bs_add<NP>(sp[k], x[k][0]);
                    bs_add<NP>(sp[k], x[k][1]);
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) rec_planes<NP>(sp[k], rec, pp[k], h[k], own, Acur, NW, w, pol);
            }
#pragma unroll
            for (int r = 0; r < NCTR; ++r) {
                uint32_t s0, s1, s2;
                sum4(bs_eq<NP>(sp[0], r), bs_eq<NP>(sp[1], r), bs_eq<NP>(sp[2], r), bs_eq<NP>(sp[3], r), s0, s1, s2);
                if (h0 & 1u) vc_add3<B>(cnt[r], s0, s1, s2);
                else vc_sub3<B>(cnt[r], s0, s1, s2);
            }
            p = p4;
        } else {
            uint32_t sp[NP];
            rec_planes<NP>(sp, rec, p, h0, own, Acur, NW, w, pol);
            if (h0 & 1u) {
#pragma unroll
                for (int r = 0; r < NCTR; ++r) vc_inc<B>(cnt[r], bs_eq<NP>(sp, r));
            } else {
#pragma unroll
                for (int r = 0; r < NCTR; ++r) vc_dec<B>(cnt[r], bs_eq<NP>(sp, r));
            }
            p += h0 >> 1;
        }
    }
}

// count_occurrences for uniform 3-SAT rows (3-word records: header + two
// literal codes), nneg negated records first, then npos positive ones.  Each
// sign section is cut into batches of 4 records (the last one masked), so
// every batch is one carry-save sum4 + one 3-bit counter update, and the next
// batch's 8 gathers are issued before the current batch is counted: a row
// costs ~ceil(nneg/4) + ceil(npos/4) overlapped L2 round trips instead of one
// per leftover record.
template <int NCTR, int B, bool PIPE, typename RecFn>
__device__ __forceinline__ void count_uni3(uint32_t (&cnt)[NCTR][B], RecFn rec, unsigned nneg, unsigned npos,
                                           uint32_t own, const uint32_t* __restrict__ Acur, unsigned NW, unsigned w, unsigned long long pol) {
#pragma unroll
    for (int r = 0; r < NCTR; ++r)
#pragma unroll
        for (int b = 0; b < B; ++b) cnt[r][b] = 0u;
    const unsigned nbn = (nneg + 3) >> 2, nb = nbn + ((npos + 3) >> 2);
    if (nb == 0) return;
    const unsigned nrec = nneg + npos;
    auto ld = [&](uint32_t code) { return ld_plane(Acur + ((code >> 1) * NW + w), pol) ^ (0u - (code & 1u)); };
    // batch b: records [first, first + count), all of one sign
    auto batch = [&](unsigned b, unsigned& first, unsigned& count) {
        if (b < nbn) { first = 4 * b; count = min(4u, nneg - 4 * b); }
        else { first = nneg + 4 * (b - nbn); count = min(4u, nrec - first); }
    };
    uint32_t xn[4][2];
    auto load = [&](unsigned b) {
        unsigned first, count;
        batch(b, first, count);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned i = 3 * (first + min((unsigned)k, count - 1));   // masked lanes re-read a valid record
            xn[k][0] = ld(rec(i + 1));
            xn[k][1] = ld(rec(i + 2));
        }
    };
    if (PIPE) load(0);
    for (unsigned b = 0; b < nb; ++b) {
        uint32_t x[4][2];
        if (!PIPE) load(b);
#pragma unroll
        for (int k = 0; k < 4; ++k) { x[k][0] = xn[k][0]; x[k][1] = xn[k][1]; }
        if (PIPE && b + 1 < nb) load(b + 1);
        unsigned first, count;
        batch(b, first, count);
        const bool neg = b < nbn;
        const uint32_t os = neg ? ~own : own;               // own literal's value in this section
        uint32_t p0[4], p1[4], mk[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            p0[k] = os ^ x[k][0] ^ x[k][1];                 // 2-plane count of true literals
            p1[k] = (os & x[k][0]) | (x[k][1] & (os ^ x[k][0]));
            mk[k] = (unsigned)k < count ? 0xffffffffu : 0u;
        }
#pragma unroll
        for (int r = 0; r < NCTR; ++r) {
            uint32_t e[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                e[k] = ((r & 1) ? p0[k] : ~p0[k]) & ((r & 2) ? p1[k] : ~p1[k]) & mk[k];
            uint32_t s0, s1, s2;
            sum4(e[0], e[1], e[2], e[3], s0, s1, s2);
            if (neg) vc_add3<B>(cnt[r], s0, s1, s2);
            else vc_sub3<B>(cnt[r], s0, s1, s2);
        }
    }
}

// count_occurrences over batched records (host_cnf.cpp build_batched): every
// instance except uniform 3-SAT.  A batch holds up to 4 same-sign records
// padded to the longest; its gathers are issued two literal steps (8 loads)
// at a time, absent records start at the all-ones count KB - 1 = 2^NP - 1
// (the derived bin, never counted), and each bin takes one carry-save sum4
// and one counter update per batch.
// R0: the counters hold bins R0 .. R0 + NCTR - 1 (KB = 16 counts its 15 bins
// in two passes of at most 8, k_hub).
template <int NP, int NCTR, int B, int R0 = 0, typename RecFn>
__device__ __forceinline__ void count_batched(uint32_t (&cnt)[NCTR][B], RecFn rec, unsigned nwords, uint32_t own,
                                              const uint32_t* __restrict__ Acur, unsigned NW, unsigned w, unsigned long long pol) {
    static_assert(R0 + NCTR <= (1 << NP) - 1, "absent records rely on bin 2^NP - 1 being derived (never counted)");
#pragma unroll
    for (int r = 0; r < NCTR; ++r)
#pragma unroll
        for (int b = 0; b < B; ++b) cnt[r][b] = 0u;
    auto ld = [&](uint32_t code) { return ld_plane(Acur + ((code >> 1) * NW + w), pol) ^ (0u - (code & 1u)); };
    unsigned p = 0;
    while (p < nwords) {
        const uint32_t hdr = rec(p);
        const unsigned J = hdr >> 4, nk = (hdr >> 1) & 7u;
        const bool neg = (hdr & 1u) != 0u;
        const uint32_t os = neg ? ~own : own;              // own literal's value in this section
        uint32_t sp[4][NP];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool on = (unsigned)k < nk;
            sp[k][0] = on ? os : 0xffffffffu;
#pragma unroll
            for (int q = 1; q < NP; ++q) sp[k][q] = on ? 0u : 0xffffffffu;
        }
        for (unsigned j = 0; j < J; j += 2) {
            const unsigned q0 = p + 1 + 4 * j;
            const bool two = j + 1 < J;
            uint32_t x[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) x[k] = ld(rec(q0 + k));
#if TSAT_ODD_STEP
            if (two) {                                   // warp-uniform: an odd last step adds nothing more
#pragma unroll
                for (int k = 0; k < 4; ++k) x[4 + k] = ld(rec(q0 + 4 + k));
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    bs_add<NP>(sp[k], x[k]);
                    bs_add<NP>(sp[k], x[4 + k]);
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) bs_add<NP>(sp[k], x[k]);
            }
#else
#pragma unroll
            for (int k = 0; k < 4; ++k) x[4 + k] = two ? ld(rec(q0 + 4 + k)) : 0u;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                bs_add<NP>(sp[k], x[k]);
                bs_add<NP>(sp[k], x[4 + k]);
            }
#endif
        }
        // one code path for both signs: c - S = c + ~S + 1 (two's complement)
        const uint32_t cm = neg ? 0u : 0xffffffffu;
#pragma unroll
        for (int r = 0; r < NCTR; ++r) {
#if TSAT_BIN_SKIP
            // R <= clause length <= J + 1 (records are padded to the batch's
            // longest): higher bins get nothing from this batch (warp-uniform)
            if (R0 + r > (int)J + 1) break;
#endif
            uint32_t s0, s1, s2;
            sum4(bs_eq<NP>(sp[0], R0 + r), bs_eq<NP>(sp[1], R0 + r), bs_eq<NP>(sp[2], R0 + r), bs_eq<NP>(sp[3], R0 + r),
                 s0, s1, s2);
            vc_addc<B>(cnt[r], s0 ^ cm, s1 ^ cm, s2 ^ cm, cm);
        }
        p += 1 + 4 * J;
    }
}

}  // namespace tsat
