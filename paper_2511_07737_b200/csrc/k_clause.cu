// k_clause.cu - rows (a4) R = P A and (a5) the per-candidate histogram
// h_n[r] = #{c : R_cn = r} (Eq. 1, §3.1.3-3.1.4).
//
// Bit-sliced design: lane = one 32-candidate word of the batch, warp = 32
// consecutive words (1024 candidates), so every literal gather is one
// 128-byte coalesced load of the bit plane.  R_cn is accumulated as NP
// bit-planes; the one-hot masks [R = r] of 4 clauses are combined by a
// carry-save tree (ones, twos planes) before one ripple into the 7-bit
// vertical counters of each bin.  After CH <= 127 clauses each lane extracts
// per-candidate counts into a shared histogram (bank-rotated), and the CTA
// adds it to the global one.  A warp first stages its chunk's literals in
// shared memory as pre-multiplied bit-plane word offsets (one coalesced read
// of the CSR), then evaluates 4 clauses at a time so 4 * KMAXC independent
// gathers are in flight.
#include "device_common.cuh"

#ifndef TSAT_CL_CH3
#define TSAT_CL_CH3 64             // clauses per warp chunk, K <= 3
#endif
#ifndef TSAT_CL_G3
#define TSAT_CL_G3 2               // carry-save groups of 4 clauses per iteration, K <= 3
#endif

namespace tsat {

namespace {
constexpr int kWarps = 8;
// clauses per warp chunk (<= 127: 7-bit counters); K = 7 halves it to keep
// the staged literals within the 48 KB static shared memory
__host__ __device__ constexpr int chunk_clauses(int kmaxc, int wide = 0) { return kmaxc > 3 ? 32 : (wide ? 96 : TSAT_CL_CH3); }
// K <= 3 variants: WIDE = 0 (3 CTAs / SM, 64-clause chunks) for batches of
// >= 2048 candidates per GPU; WIDE = 1 (4 CTAs / SM at 64 registers, 96-clause
// chunks) below, where fewer word blocks leave the warps latency-bound (c3
// N = 1024: k_clause -7 %, N = 128: -21 %; c2 N = 4096: +5 %, so not there)
constexpr int kUnr = 4;        // clauses evaluated together (carry-save group)
constexpr uint32_t kNone = 0xffffffffu;

// full adder on bit planes: (a + b + c) = s + 2 * carry
__device__ __forceinline__ void fa(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& carry) {
    s = a ^ b ^ c;
    carry = (a & b) | (c & (a ^ b));
}
}  // namespace

// Counter of one bin: planes[0] = ones, planes[1] = twos, planes[2..6] weight 4..64.
template <int CB>
__device__ __forceinline__ void csa_add4(uint32_t (&c)[CB], uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3) {
    uint32_t s, c1, c2, c4;
    fa(c[0], m0, m1, s, c1);
    fa(s, m2, m3, c[0], c2);
    fa(c[1], c1, c2, c[1], c4);
    uint32_t carry = c4;
#pragma unroll
    for (int b = 2; b < CB; ++b) {
        uint32_t t = c[b] & carry;
        c[b] ^= carry;
        carry = t;
    }
}

#ifndef TSAT_SEG_SHORT_CTAS
#define TSAT_SEG_SHORT_CTAS 4        // k_clause_seg L <= 3: CTAs (256 threads) per SM it is compiled and sized for
#endif
#ifndef TSAT_SEG_LONG_CTAS
#define TSAT_SEG_LONG_CTAS 2         // k_clause_seg L = 4..7
#endif
#ifndef TSAT_CL_WIDE_FROM
#define TSAT_CL_WIDE_FROM 8192     // the wide K <= 3 variant also from this many candidates per GPU (c5 N = 8192: k_clause 0.54 -> 0.35 ms; c2 N = 4096: +5 %)
#endif
#ifndef TSAT_CL_PERSM3
#define TSAT_CL_PERSM3 3           // K <= 3: CTAs per SM the grid is sized for
#endif
#ifndef TSAT_CL_MINB8
#define TSAT_CL_MINB8 2            // CTAs per SM the K <= 7 kernel is compiled for
#endif
template <int KB, int KMAXC, int WIDE = 0>
__global__ void __launch_bounds__(256, KB == 4 ? (WIDE ? 4 : TSAT_CL_PERSM3) : TSAT_CL_MINB8) k_clause(const uint32_t* __restrict__ A, int NW, int V,
                                                                const uint32_t* __restrict__ cptr,
                                                                const uint32_t* __restrict__ clit, long long C,
                                                                int* __restrict__ hist, int N, int uniform,
                                                                DevScalars* __restrict__ ds,
                                                                const StepScalars* __restrict__ sc, int nsub) {
    constexpr int NP = (KB == 4) ? 2 : 3;
    constexpr int CB = 7;
    __shared__ int sh[(KB - 1) * 1024];
    // staged literals: {element offset var * NW, sign mask}; empty slots and
    // padding clauses read the all-zero row V with mask 0 (literal false)
    __shared__ uint2 soff[kWarps][chunk_clauses(KMAXC, WIDE) * KMAXC];
    constexpr int kCH = chunk_clauses(KMAXC, WIDE);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // nsub > 1 (fewer than 32 words, N < 1024 per GPU): the warp's lanes are
    // nsub sub-groups of NW lanes; sub-group `sub` evaluates every nsub-th
    // carry-save group of the chunk for word w, so no lane idles
    const int sub = nsub > 1 ? lane / NW : 0;
    const int w = nsub > 1 ? lane - sub * NW : blockIdx.x * 32 + lane;
    const bool valid = w < NW && sub < nsub;
    const int wl = nsub > 1 ? w : lane;                 // word within the CTA's 32-word block
    pdl_wait();
    pdl_trigger();
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
        // the iteration's accumulators (the previous k_update consumed them):
        // best key and gmax (k_gtable), row scheduler and max|theta_{t+1}| (k_update)
        const long long t = sc->t;
        ds->best_key = ~0ull;
        ds->gmax_bits = 0ull;
        ds->row_counter = 0;
        ds->thmax_bits[(t + 1) & 1] = 0u;
        ds->loss_fx = 0;
    }
    for (int i = threadIdx.x; i < (KB - 1) * 1024; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    uint2* my = soff[warp];
    const uint32_t unw = (uint32_t)NW;
    const uint2 zero_lit = make_uint2((uint32_t)V * unw, 0u);
    const uint32_t* Aw = A + (valid ? w : 0);          // lanes past NW read a valid word, results unused
    const unsigned long long pol = plane_policy(planes_fit_l2(V, NW));
    const long long nchunks = (C + kCH - 1) / kCH;
    constexpr int kG0 = KMAXC <= 3 ? TSAT_CL_G3 : 1;
    // with sub-groups a lane sees kCH / nsub clauses per chunk: its counters
    // (<= 127 per bin) are carried over nsub chunks before one extraction
    uint32_t cnt[KB - 1][CB];
#pragma unroll
    for (int r = 0; r < KB - 1; ++r)
#pragma unroll
        for (int b = 0; b < CB; ++b) cnt[r][b] = 0u;
    int pend = 0;
    // grid-sized: warps stride over the clause chunks of this word block
    for (long long chunk = (long long)blockIdx.y * kWarps + warp; chunk < nchunks;
         chunk += (long long)gridDim.y * kWarps) {
        const long long c0 = chunk * kCH;
        const long long c1 = c0 + kCH < C ? c0 + kCH : C;
        const int nc = (int)(c1 - c0);
        __syncwarp();
        if (uniform) {
            const uint32_t* src = clit + (size_t)c0 * KMAXC;
            for (int i = lane; i < kCH * KMAXC; i += 32) {
                const uint32_t code = (i < nc * KMAXC) ? src[i] : kNone;
                my[i] = code == kNone ? zero_lit : make_uint2((code >> 1) * unw, 0u - (code & 1u));
            }
        } else {
            for (int i = lane; i < kCH * KMAXC; i += 32) {
                const int c = i / KMAXC, l = i - c * KMAXC;
                uint2 o = zero_lit;
                if (c < nc) {
                    const uint32_t b = cptr[c0 + c], e = cptr[c0 + c + 1];
                    if (b + l < e) {
                        const uint32_t code = clit[b + l];
                        o = make_uint2((code >> 1) * unw, 0u - (code & 1u));
                    }
                }
                my[i] = o;
            }
        }
        __syncwarp();
        constexpr int kG = kG0;                         // carry-save groups per iteration (gathers in flight)
        for (int cb0 = sub * kUnr * kG; cb0 < nc; cb0 += kUnr * kG * nsub) {
            uint32_t xx[kG][kUnr][KMAXC];
#pragma unroll
            for (int gq = 0; gq < kG; ++gq)
#pragma unroll
                for (int u = 0; u < kUnr; ++u)
#pragma unroll
                    for (int l = 0; l < KMAXC; ++l) {
                        const int c = cb0 + gq * kUnr + u;      // < kCH: the chunk is padded
                        const uint2 o = my[c * KMAXC + l];
                        xx[gq][u][l] = ld_plane(Aw + o.x, pol) ^ o.y;
                    }
#pragma unroll
          for (int gq = 0; gq < kG; ++gq) {
            const int cb = cb0 + gq * kUnr;
            uint32_t (&x)[kUnr][KMAXC] = xx[gq];
            // one-hot masks [R = r] per clause (padding clauses past nc have all
            // literals 0 -> R = 0, so their bin-0 mask is cleared)
            uint32_t m[kUnr][KB - 1];
#pragma unroll
            for (int u = 0; u < kUnr; ++u) {
                const uint32_t live = (cb + u < nc) ? 0xffffffffu : 0u;
                if (KMAXC == 3 && KB == 4) {
                    const uint32_t a = x[u][0], b = x[u][1], c = x[u][2];
                    m[u][0] = ~(a | b | c) & live;                     // R = 0
                    const uint32_t s0 = a ^ b ^ c, s1 = (a & b) | (c & (a ^ b));
                    m[u][1] = s0 & ~s1;                                 // R = 1
                    m[u][2] = ~s0 & s1;                                 // R = 2
                } else {
                    uint32_t sp[NP];
#pragma unroll
                    for (int p = 0; p < NP; ++p) sp[p] = 0u;
#pragma unroll
                    for (int l = 0; l < KMAXC; ++l) bs_add<NP>(sp, x[u][l]);
#pragma unroll
                    for (int r = 0; r < KB - 1; ++r) m[u][r] = bs_eq<NP>(sp, r) & (r == 0 ? live : 0xffffffffu);
                }
            }
#pragma unroll
            for (int r = 0; r < KB - 1; ++r) csa_add4<CB>(cnt[r], m[0][r], m[1][r], m[2][r], m[3][r]);
          }
        }
        ++pend;
        const bool last = chunk + (long long)gridDim.y * kWarps >= nchunks;
        if (pend < nsub && !last) continue;             // keep counting into the same counters
        pend = 0;
        if (valid) {
            if (KB == 4) {
                // one 32x32 transpose packs the three 7-bit counts of each
                // candidate into 10-bit fields of one word; they are widened to
                // 21-bit fields of a 64-bit CTA accumulator (< 2^21 clauses per
                // CTA and word block, see launch_clause)
                uint32_t T[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) T[i] = (i % 10 < CB && i / 10 < KB - 1) ? cnt[i / 10][i % 10] : 0u;
                transpose32(T);
                unsigned long long* shp = reinterpret_cast<unsigned long long*>(sh);
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (T[j]) {
                        const unsigned long long pk = T[j];
                        const unsigned long long wide = (pk & 0x3FFull) | ((pk & 0xFFC00ull) << 11) | ((pk & 0x3FF00000ull) << 22);
                        atomicAdd(&shp[33 * wl + j], wide);               // padded layout
                    }
            } else {
                // two 32x32 transposes (bins 0-3, 4-6) give each candidate's
                // 7-bit counts as bytes; they are widened into 21-bit fields of
                // three 64-bit CTA accumulators per candidate:
                // [0] = bins 0, 1, 2   [1] = bins 3, 4, 5   [2] = bin 6
                unsigned long long* shp = reinterpret_cast<unsigned long long*>(sh);
                constexpr int kAcc = 33 * 32;                // one padded accumulator plane
#pragma unroll 1
                for (int blk = 0; blk < 2; ++blk) {
                    uint32_t T[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int r = i / 8, b = i % 8;
                        const uint32_t lo = (b < CB) ? cnt[r][b] : 0u;
                        const uint32_t hi = (b < CB && 4 + r < KB - 1) ? cnt[4 + r][b] : 0u;
                        T[i] = blk ? hi : lo;
                    }
                    transpose32(T);
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const unsigned long long x = T[j];
                        if (!x) continue;
                        const int o = 33 * wl + j;
                        if (blk == 0) {
                            const unsigned long long w0 = (x & 0xFFull) | ((x & 0xFF00ull) << 13) | ((x & 0xFF0000ull) << 26);
                            if (w0) atomicAdd(&shp[o], w0);
                            if (x >> 24) atomicAdd(&shp[kAcc + o], x >> 24);
                        } else {
                            const unsigned long long w1 = ((x & 0xFFull) << 21) | ((x & 0xFF00ull) << 34);
                            if (w1) atomicAdd(&shp[kAcc + o], w1);
                            if (x & 0xFF0000ull) atomicAdd(&shp[2 * kAcc + o], (x >> 16) & 0xFFull);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < KB - 1; ++r)
#pragma unroll
            for (int b = 0; b < CB; ++b) cnt[r][b] = 0u;
    }
    __syncthreads();
    if (KB == 4) {
        const unsigned long long* shp = reinterpret_cast<const unsigned long long*>(sh);
        for (int cl = threadIdx.x; cl < 1024; cl += blockDim.x) {
            const int n = blockIdx.x * 1024 + cl;
            const unsigned long long pk = shp[33 * (cl >> 5) + (cl & 31)];
            if (n < N && pk) {
#pragma unroll
                for (int r = 0; r < KB - 1; ++r) {
                    const int val = (int)((pk >> (21 * r)) & 0x1FFFFFull);
                    if (val) atomicAdd(&hist[(size_t)n * KB + r], val);
                }
            }
        }
    } else {
        const unsigned long long* shp = reinterpret_cast<const unsigned long long*>(sh);
        constexpr int kAcc = 33 * 32;
        for (int cl = threadIdx.x; cl < 1024; cl += blockDim.x) {
            const int n = blockIdx.x * 1024 + cl;
            if (n >= N) continue;
            const int o = 33 * (cl >> 5) + (cl & 31);
#pragma unroll
            for (int r = 0; r < KB - 1; ++r) {
                const unsigned long long pk = shp[(r / 3) * kAcc + o];
                const int val = (int)((pk >> (21 * (r % 3))) & 0x1FFFFFull);
                if (val) atomicAdd(&hist[(size_t)n * KB + r], val);
            }
        }
    }
}

// K > 7 (KB = 16: long clauses such as at-least-one constraints):
// R needs 4 bit-planes and 15 counted bins.  Lane = one 32-candidate word; a
// warp evaluates chunks of 64 clauses one at a time (literal codes read through
// L1, broadcast to the lanes), adds the one-hot masks [R = r] to 7-bit
// vertical counters and, per chunk, extracts per-candidate counts with four
// 32x32 transposes (4 bins as bytes each) into global int32 atomics.
// Correctness-first: this layout is not tuned (no long-clause workload in BASELINE).
__global__ void __launch_bounds__(256, 1) k_clause_wide(const uint32_t* __restrict__ A, int NW, int V,
                                                      const uint32_t* __restrict__ cptr,
                                                      const uint32_t* __restrict__ clit, long long C,
                                                      int* __restrict__ hist, int N, DevScalars* __restrict__ ds,
                                                      const StepScalars* __restrict__ sc) {
    constexpr int KB = 16, NP = 4, CB = 7, kCHW = 64;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int w = blockIdx.x * 32 + lane;
    const bool valid = w < NW;
    pdl_wait();
    pdl_trigger();
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
        const long long t = sc->t;
        ds->best_key = ~0ull;
        ds->gmax_bits = 0ull;
        ds->row_counter = 0;
        ds->thmax_bits[(t + 1) & 1] = 0u;
        ds->loss_fx = 0;
    }
    const uint32_t* Aw = A + (valid ? w : 0);
    const unsigned long long pol = plane_policy(planes_fit_l2(V, NW));
    const long long nchunks = (C + kCHW - 1) / kCHW;
    for (long long chunk = (long long)blockIdx.y * kWarps + warp; chunk < nchunks;
         chunk += (long long)gridDim.y * kWarps) {
        const long long c0 = chunk * kCHW, c1 = c0 + kCHW < C ? c0 + kCHW : C;
        uint32_t cnt[KB - 1][CB];
#pragma unroll
        for (int r = 0; r < KB - 1; ++r)
#pragma unroll
            for (int b = 0; b < CB; ++b) cnt[r][b] = 0u;
        for (long long c = c0; c < c1; ++c) {
            const uint32_t b = __ldg(cptr + c), e = __ldg(cptr + c + 1);
            uint32_t sp[NP] = {0u, 0u, 0u, 0u};
            for (uint32_t i = b; i < e; ++i) {
                const uint32_t code = __ldg(clit + i);
                bs_add<NP>(sp, ld_plane(Aw + (size_t)(code >> 1) * NW, pol) ^ (0u - (code & 1u)));
            }
#pragma unroll
            for (int r = 0; r < KB - 1; ++r) vc_inc<CB>(cnt[r], bs_eq<NP>(sp, r));
        }
        if (!valid) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {                       // bins 4q .. 4q + 3 as bytes
            uint32_t T[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int r = 4 * q + i / 8, bb = i % 8;
                T[i] = (r < KB - 1 && bb < CB) ? cnt[r < KB - 1 ? r : 0][bb < CB ? bb : 0] : 0u;
            }
            transpose32(T);
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
                const int n = 32 * w + j;
                if (n >= N || !T[j]) continue;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int r = 4 * q + k;
                    const int val = (int)((T[j] >> (8 * k)) & 0xffu);
                    if (r < KB - 1 && val) atomicAdd(&hist[(size_t)n * KB + r], val);
                }
            }
        }
    }
}

__global__ void k_reset_accumulators(DevScalars* __restrict__ ds, const StepScalars* __restrict__ sc) {
    const long long t = sc->t;
    ds->best_key = ~0ull;
    ds->gmax_bits = 0ull;
    ds->row_counter = 0;
    ds->thmax_bits[(t + 1) & 1] = 0u;
    ds->loss_fx = 0;
}

// ---------------------------------------------------------------- length segments
// k_clause_seg: every K <= 7 instance except uniform 3-SAT, >= 1024 candidates
// per GPU.  Clauses come grouped by length (host_cnf.cpp build_segments); a
// warp chunk of the length-L segment gathers exactly L literals per clause and
// counts L + 1 one-hot bins (NP = 1, 2 or 3 count planes), where the padded
// kernel above gathers K literals and counts KB - 1 bins for every clause
// (industrial mix, mean length 3.2 of K = 7).  Two instantiations: L <= 3 (4
// CTAs per SM) and L = 4..7 (2 CTAs per SM), so the short clauses do not
// run at the long ones' register budget.  Counters are 7-bit carry-save
// planes per bin as above; each chunk (<= 112 clauses) is extracted by one
// (NB <= 4 bins) or two byte transposes into 21-bit fields of three 64-bit
// CTA accumulators per candidate: [0] bins 0, 1, 2  [1] bins 3, 4, 5  [2] bin 6.
struct SegArgs {
    long long off[8];          // word offset of segment L in seg_lit
    long long C[8];            // clauses of length L
    long long ch0[9];          // first chunk of segment L in this kernel's chunk range (ch0[LMAX + 1] = total)
};
__host__ __device__ constexpr int seg_chunk(int L) {
    return L <= 2 ? 112 : (L == 3 ? 72 : (L == 4 ? 56 : (L == 5 ? 44 : (L == 6 ? 36 : 32))));
}
constexpr int kSegStage = 224;     // staged literal slots per warp: max over L of seg_chunk(L) * L
constexpr int kSegAcc = 33 * 32;   // one padded accumulator plane (u64 per candidate of the block)

template <int KB, int L>
__device__ __forceinline__ void seg_eval(const uint32_t* __restrict__ Aw, const uint32_t* __restrict__ lit, int nc,
                                         uint2* my, uint32_t unw, uint2 zero_lit, unsigned long long pol,
                                         unsigned long long* acc, int lane, bool valid) {
    constexpr int NB = (L + 1 < KB - 1) ? L + 1 : KB - 1;     // counted bins (bin KB - 1 is derived)
    constexpr int NP = L <= 1 ? 1 : (L <= 3 ? 2 : 3);
    constexpr int kCH = seg_chunk(L);
    constexpr int CB = 7;
    constexpr int kG = L <= 3 ? 2 : 1;                         // carry-save groups of 4 clauses in flight
    static_assert(kCH * L <= kSegStage && kCH % (kUnr * kG) == 0 && kCH <= 127, "segment chunk geometry");
    __syncwarp();
    for (int i = lane; i < kCH * L; i += 32) {
        const uint32_t code = i < nc * L ? __ldg(lit + i) : kNone;
        my[i] = code == kNone ? zero_lit : make_uint2((code >> 1) * unw, 0u - (code & 1u));
    }
    __syncwarp();
    uint32_t cnt[NB][CB];
#pragma unroll
    for (int r = 0; r < NB; ++r)
#pragma unroll
        for (int b = 0; b < CB; ++b) cnt[r][b] = 0u;
    for (int cb0 = 0; cb0 < nc; cb0 += kUnr * kG) {
        uint32_t xx[kG][kUnr][L];
#pragma unroll
        for (int gq = 0; gq < kG; ++gq)
#pragma unroll
            for (int u = 0; u < kUnr; ++u)
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    const uint2 o = my[(cb0 + gq * kUnr + u) * L + l];     // < kCH: the chunk is padded
                    xx[gq][u][l] = ld_plane(Aw + o.x, pol) ^ o.y;
                }
#pragma unroll
        for (int gq = 0; gq < kG; ++gq) {
            uint32_t m[kUnr][NB];
#pragma unroll
            for (int u = 0; u < kUnr; ++u) {
                // padding clauses past nc read literal-false rows: R = 0, bin 0 cleared
                const uint32_t live = (cb0 + gq * kUnr + u < nc) ? 0xffffffffu : 0u;
                const uint32_t* x = xx[gq][u];
                if constexpr (L == 1) {
                    m[u][0] = ~x[0] & live;
                    m[u][1] = x[0];
                } else if constexpr (L == 2) {
                    m[u][0] = ~(x[0] | x[1]) & live;
                    m[u][1] = x[0] ^ x[1];
                    if constexpr (NB > 2) m[u][2] = x[0] & x[1];
                } else if constexpr (L == 3) {
                    const uint32_t s0 = x[0] ^ x[1] ^ x[2], s1 = (x[0] & x[1]) | (x[2] & (x[0] ^ x[1]));
                    m[u][0] = ~(x[0] | x[1] | x[2]) & live;
                    m[u][1] = s0 & ~s1;
                    m[u][2] = ~s0 & s1;
                    if constexpr (NB > 3) m[u][3] = s0 & s1;
                } else {
                    uint32_t sp[NP];
#pragma unroll
                    for (int p = 0; p < NP; ++p) sp[p] = 0u;
#pragma unroll
                    for (int l = 0; l < L; ++l) bs_add<NP>(sp, x[l]);
#pragma unroll
                    for (int r = 0; r < NB; ++r) m[u][r] = bs_eq<NP>(sp, r) & (r == 0 ? live : 0xffffffffu);
                }
            }
#pragma unroll
            for (int r = 0; r < NB; ++r) csa_add4<CB>(cnt[r], m[0][r], m[1][r], m[2][r], m[3][r]);
        }
    }
    if (!valid) return;
    // bins 4 blk .. 4 blk + 3 as bytes per candidate, into the 21-bit fields
#pragma unroll 1
    for (int blk = 0; blk < (NB > 4 ? 2 : 1); ++blk) {
        uint32_t T[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const int r = i / 8, b = i % 8;
            const uint32_t lo = (b < CB && r < NB) ? cnt[r < NB ? r : 0][b < CB ? b : 0] : 0u;
            const uint32_t hi = (b < CB && 4 + r < NB) ? cnt[4 + r < NB ? 4 + r : 0][b < CB ? b : 0] : 0u;
            T[i] = blk ? hi : lo;
        }
        transpose32(T);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const unsigned long long x = T[j];
            if (!x) continue;
            const int o = 33 * lane + j;
            if (blk == 0) {
                const unsigned long long w0 = (x & 0xFFull) | ((x & 0xFF00ull) << 13) | ((x & 0xFF0000ull) << 26);
                if (w0) atomicAdd(&acc[o], w0);
                if (NB > 3 && (x >> 24)) atomicAdd(&acc[kSegAcc + o], x >> 24);
            } else {
                const unsigned long long w1 = ((x & 0xFFull) << 21) | ((x & 0xFF00ull) << 34);
                if (w1) atomicAdd(&acc[kSegAcc + o], w1);
                if (NB > 6 && (x & 0xFF0000ull)) atomicAdd(&acc[2 * kSegAcc + o], (x >> 16) & 0xFFull);
            }
        }
    }
}

template <int KB, int LMIN, int LMAX>
__global__ void __launch_bounds__(256, LMAX <= 3 ? TSAT_SEG_SHORT_CTAS : TSAT_SEG_LONG_CTAS)
    k_clause_seg(const uint32_t* __restrict__ A, int NW, int V, const uint32_t* __restrict__ seg_lit, SegArgs sa,
                 int* __restrict__ hist, int N, DevScalars* __restrict__ ds, const StepScalars* __restrict__ sc,
                 int reset) {
    constexpr int NBK = (LMAX + 1 < KB - 1) ? LMAX + 1 : KB - 1;    // bins this kernel counts
    constexpr int NACC = NBK > 6 ? 3 : (NBK > 3 ? 2 : 1);
    __shared__ unsigned long long acc[NACC * kSegAcc];
    __shared__ uint2 stage[kWarps][kSegStage];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int w = blockIdx.x * 32 + lane;
    const bool valid = w < NW;
    pdl_wait();
    pdl_trigger();
    if (reset && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
        const long long t = sc->t;               // the iteration's accumulators (see k_clause)
        ds->best_key = ~0ull;
        ds->gmax_bits = 0ull;
        ds->row_counter = 0;
        ds->thmax_bits[(t + 1) & 1] = 0u;
        ds->loss_fx = 0;
    }
    for (int i = threadIdx.x; i < NACC * kSegAcc; i += blockDim.x) acc[i] = 0ull;
    __syncthreads();
    uint2* my = stage[warp];
    const uint32_t unw = (uint32_t)NW;
    const uint2 zero_lit = make_uint2((uint32_t)V * unw, 0u);
    const uint32_t* Aw = A + (valid ? w : 0);
    const unsigned long long pol = plane_policy(planes_fit_l2(V, NW));
    const long long nchunks = sa.ch0[LMAX + 1];
    for (long long chunk = (long long)blockIdx.y * kWarps + warp; chunk < nchunks;
         chunk += (long long)gridDim.y * kWarps) {
        int L = LMIN;
        while (L < LMAX && chunk >= sa.ch0[L + 1]) ++L;      // warp-uniform
        const long long c0 = (chunk - sa.ch0[L]) * seg_chunk(L);
        const int nc = (int)min((long long)seg_chunk(L), sa.C[L] - c0);
        const uint32_t* lit = seg_lit + sa.off[L] + c0 * L;
#define TSAT_SEG_CASE(LL)                                                                                    \
    case LL:                                                                                                 \
        if constexpr (LMIN <= LL && LL <= LMAX) seg_eval<KB, LL>(Aw, lit, nc, my, unw, zero_lit, pol, acc, lane, valid); \
        break;
        switch (L) {
            TSAT_SEG_CASE(1) TSAT_SEG_CASE(2) TSAT_SEG_CASE(3) TSAT_SEG_CASE(4) TSAT_SEG_CASE(5) TSAT_SEG_CASE(6)
            TSAT_SEG_CASE(7)
            default: break;
        }
#undef TSAT_SEG_CASE
    }
    __syncthreads();
    for (int cl = threadIdx.x; cl < 1024; cl += blockDim.x) {
        const int n = blockIdx.x * 1024 + cl;
        if (n >= N) continue;
        const int o = 33 * (cl >> 5) + (cl & 31);
#pragma unroll
        for (int r = 0; r < NBK; ++r) {
            const unsigned long long pk = acc[(r / 3) * kSegAcc + o];
            const int val = (int)((pk >> (21 * (r % 3))) & 0x1FFFFFull);
            if (val) atomicAdd(&hist[(size_t)n * KB + r], val);
        }
    }
}

// Launch the short (L <= 3) and long (L = 4..7) segment kernels, in that order
// on the stream (the first resets the iteration's accumulators).
template <int KB>
static cudaError_t launch_clause_seg(const StepArgs& a, const uint32_t* Acur, const StepScalars* sc, cudaStream_t st) {
    const int NW = a.N >> 5, nwb = (NW + 31) / 32;
    bool first = true;
    for (int part = 0; part < 2; ++part) {
        const int lmin = part ? 4 : 1, lmax = part ? (KB == 4 ? 3 : 7) : 3;
        if (lmin > lmax) continue;
        SegArgs sa{};
        long long ch = 0, ncl = 0;
        for (int L = 0; L < 8; ++L) { sa.off[L] = a.seg_off[L]; sa.C[L] = a.seg_C[L]; }
        for (int L = 0; L <= 8; ++L) {
            sa.ch0[L] = ch;
            if (L >= lmin && L <= lmax) { ch += (a.seg_C[L] + seg_chunk(L) - 1) / seg_chunk(L); ncl += a.seg_C[L]; }
        }
        if (ch == 0) continue;
        const int per_sm = part ? TSAT_SEG_LONG_CTAS : TSAT_SEG_SHORT_CTAS;
        long long gy = ((long long)a.num_sms * per_sm + nwb - 1) / nwb;
        const long long need = (ch + kWarps - 1) / kWarps;
        if (gy > need) gy = need;
        // 21-bit CTA accumulator fields: < 2^20 clauses per CTA and word block (2x margin)
        const long long gy_min = (ncl + (1LL << 20) - 1) >> 20;
        if (gy < gy_min) gy = gy_min;
        if (gy < 1) gy = 1;
        const dim3 grid(nwb, (unsigned)gy);
        const int rs = first ? 1 : 0;
        cudaError_t e;
        if (part == 0)
            e = launch_maybe_pdl(a.pdl, k_clause_seg<KB, 1, 3>, grid, dim3(256), 0, st, Acur, NW, a.V, a.seg_lit, sa, a.hist,
                                 a.N, a.ds, sc, rs);
        else if constexpr (KB == 8)
            e = launch_maybe_pdl(a.pdl, k_clause_seg<KB, 4, 7>, grid, dim3(256), 0, st, Acur, NW, a.V, a.seg_lit, sa,
                                 a.hist, a.N, a.ds, sc, rs);
        else
            e = cudaErrorInvalidValue;
        if (e != cudaSuccess) return e;
        first = false;
    }
    if (first) k_reset_accumulators<<<1, 1, 0, st>>>(a.ds, sc);    // no clause at all
    return cudaGetLastError();
}

cudaError_t launch_clause(const StepArgs& a, const uint32_t* Acur, const StepScalars* sc, cudaStream_t st) {
    if (a.C == 0) {
        k_reset_accumulators<<<1, 1, 0, st>>>(a.ds, sc);
        return cudaGetLastError();
    }
    if (a.use_seg) return a.KB == 4 ? launch_clause_seg<4>(a, Acur, sc, st) : launch_clause_seg<8>(a, Acur, sc, st);
    const int NW = a.N >> 5;
    const int nwb = (NW + 31) / 32;
    // sub-groups of NW lanes when a warp would leave lanes idle (N < 1024 per GPU);
    // a chunk (kCH clauses) must split evenly into carry-save groups per sub-group
    const int wide = (a.mc.K <= 3 && (a.N < 2048 || a.N >= TSAT_CL_WIDE_FROM)) ? 1 : 0;
    const int kCH = chunk_clauses(a.mc.K <= 3 ? 3 : 7, wide);
    const int kGrp = 4 * (a.mc.K <= 3 ? TSAT_CL_G3 : 1);
    int nsub = NW < 32 ? 32 / NW : 1;
    while (nsub > 1 && kCH % (kGrp * nsub)) --nsub;
    const long long nchunks = (a.C + kCH - 1) / kCH;
    const long long ctas_needed = (nchunks + kWarps - 1) / kWarps;
    const int K = a.mc.K;
    // grid-sized: (CTAs resident per SM) x SMs, split over the word blocks
    const int per_sm = K <= 3 ? (wide ? 4 : TSAT_CL_PERSM3) : TSAT_CL_MINB8;
    long long gy = ((long long)a.num_sms * per_sm + nwb - 1) / nwb;
    if (gy > ctas_needed) gy = ctas_needed;
    // packed 21-bit CTA histogram fields (KB = 4): < 2^21 clauses per CTA
    const long long gy_min = (a.C + (1LL << 20) - 1) >> 20;
    if (gy < gy_min) gy = gy_min;
    if (gy < 1) gy = 1;
    dim3 grid(nwb, (unsigned)gy);
    const int uni = a.uniform_len;
    if (K <= 2)
        return wide ? launch_maybe_pdl(a.pdl, k_clause<4, 2, 1>, grid, dim3(256), 0, st, Acur, NW, a.V, a.cptr, a.clit,
                                       a.C, a.hist, a.N, (int)(uni && K == 2), a.ds, sc, nsub)
                    : launch_maybe_pdl(a.pdl, k_clause<4, 2, 0>, grid, dim3(256), 0, st, Acur, NW, a.V, a.cptr, a.clit,
                                       a.C, a.hist, a.N, (int)(uni && K == 2), a.ds, sc, nsub);
    else if (K == 3)
        return wide ? launch_maybe_pdl(a.pdl, k_clause<4, 3, 1>, grid, dim3(256), 0, st, Acur, NW, a.V, a.cptr, a.clit,
                                       a.C, a.hist, a.N, uni, a.ds, sc, nsub)
                    : launch_maybe_pdl(a.pdl, k_clause<4, 3, 0>, grid, dim3(256), 0, st, Acur, NW, a.V, a.cptr, a.clit,
                                       a.C, a.hist, a.N, uni, a.ds, sc, nsub);
    else if (K <= 7)
        return launch_maybe_pdl(a.pdl, k_clause<8, 7>, grid, dim3(256), 0, st, Acur, NW, a.V, a.cptr, a.clit, a.C, a.hist,
                                a.N, (int)(uni && K == 7), a.ds, sc, nsub);
    else {
        const long long chunks_w = (a.C + 63) / 64;
        long long gyw = ((long long)a.num_sms * 2 + nwb - 1) / nwb;
        const long long need = (chunks_w + kWarps - 1) / kWarps;
        if (gyw > need) gyw = need;
        if (gyw < 1) gyw = 1;
        return launch_maybe_pdl(a.pdl, k_clause_wide, dim3(nwb, (unsigned)gyw), dim3(256), 0, st, Acur, NW, a.V, a.cptr,
                                a.clit, a.C, a.hist, a.N, a.ds, sc);
    }
    return cudaGetLastError();
}

}  // namespace tsat
