// k_clause.cu - rows (a4) R = P A and (a5) the per-candidate histogram
// h_n[r] = #{c : R_cn = r} (Eq. 1, §3.1.3-3.1.4).
//
// Bit-sliced design: lane = one 32-candidate word of the batch, warp = 32
// consecutive words (1024 candidates), so every literal gather is one
// 128-byte coalesced load of the bit plane.  R_cn is accumulated as NP
// bit-planes; the one-hot masks [R = r] feed 7-bit vertical counters per bin;
// after CH <= 127 clauses each lane extracts per-candidate counts into a
// shared histogram (bank-rotated), and the CTA adds it to the global one.
// A warp first stages its chunk's literal codes in shared memory (one
// coalesced read of the CSR), then evaluates UNR clauses at a time so
// UNR * KMAXC independent gathers are in flight.
#include "device_common.cuh"

namespace tsat {

namespace {
constexpr int kWarps = 8;
constexpr int kCH = 64;        // clauses per warp chunk (<= 127: 7-bit counters)
constexpr int kUnr = 4;        // clauses evaluated together
constexpr uint32_t kNone = 0xffffffffu;
}  // namespace

template <int KB, int KMAXC>
__global__ void __launch_bounds__(256) k_clause(const uint32_t* __restrict__ A, int NW, const uint32_t* __restrict__ cptr,
                                                const uint32_t* __restrict__ clit, long long C, int* __restrict__ hist,
                                                int N, int uniform) {
    constexpr int NP = (KB == 4) ? 2 : 3;
    constexpr int CB = 7;
    __shared__ int sh[(KB - 1) * 1024];
    __shared__ uint32_t scode[kWarps][kCH * KMAXC];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int w = blockIdx.x * 32 + lane;
    const bool valid = w < NW;
    for (int i = threadIdx.x; i < (KB - 1) * 1024; i += blockDim.x) sh[i] = 0;
    const long long c0 = ((long long)blockIdx.y * kWarps + warp) * kCH;
    const long long c1 = c0 + kCH < C ? c0 + kCH : C;
    const int nc = c1 > c0 ? (int)(c1 - c0) : 0;
    // stage codes: slot (c, l) of the chunk, kNone where clause c has < l+1 literals
    uint32_t* my = scode[warp];
    if (uniform) {
        const uint32_t* src = clit + (size_t)c0 * KMAXC;
        for (int i = lane; i < kCH * KMAXC; i += 32) my[i] = (i < nc * KMAXC) ? src[i] : kNone;
    } else {
        for (int i = lane; i < kCH * KMAXC; i += 32) {
            const int c = i / KMAXC, l = i - c * KMAXC;
            uint32_t code = kNone;
            if (c < nc) {
                const uint32_t b = cptr[c0 + c], e = cptr[c0 + c + 1];
                if (b + l < e) code = clit[b + l];
            }
            my[i] = code;
        }
    }
    __syncthreads();
    uint32_t cnt[KB - 1][CB];
#pragma unroll
    for (int r = 0; r < KB - 1; ++r)
#pragma unroll
        for (int b = 0; b < CB; ++b) cnt[r][b] = 0u;
    const size_t wofs = valid ? (size_t)w : 0;
    for (int cb = 0; cb < nc; cb += kUnr) {
        uint32_t x[kUnr][KMAXC];
#pragma unroll
        for (int u = 0; u < kUnr; ++u)
#pragma unroll
            for (int l = 0; l < KMAXC; ++l) {
                const uint32_t code = (cb + u < nc) ? my[(cb + u) * KMAXC + l] : kNone;
                uint32_t val = 0u;
                if (code != kNone && valid) val = __ldg(A + (size_t)(code >> 1) * NW + wofs) ^ (0u - (code & 1u));
                x[u][l] = val;
            }
#pragma unroll
        for (int u = 0; u < kUnr; ++u) {
            if (cb + u >= nc) break;
            uint32_t s[NP];
#pragma unroll
            for (int p = 0; p < NP; ++p) s[p] = 0u;
#pragma unroll
            for (int l = 0; l < KMAXC; ++l) bs_add<NP>(s, x[u][l]);
#pragma unroll
            for (int r = 0; r < KB - 1; ++r) {
                uint32_t carry = bs_eq<NP>(s, r);
#pragma unroll
                for (int b = 0; b < CB; ++b) {
                    uint32_t t = cnt[r][b] & carry;
                    cnt[r][b] ^= carry;
                    carry = t;
                }
            }
        }
    }
    if (valid) {
#pragma unroll
        for (int r = 0; r < KB - 1; ++r)
            for (int j0 = 0; j0 < 32; ++j0) {
                int j = (j0 + lane) & 31;            // rotate: conflict-free smem banks
                int val = 0;
#pragma unroll
                for (int b = 0; b < CB; ++b) val |= (int)((cnt[r][b] >> j) & 1u) << b;
                if (val) atomicAdd(&sh[r * 1024 + lane * 32 + j], val);
            }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < (KB - 1) * 1024; i += blockDim.x) {
        int r = i >> 10, cl = i & 1023;
        int n = blockIdx.x * 1024 + cl;
        int val = sh[i];
        if (n < N && val) atomicAdd(&hist[(size_t)n * KB + r], val);
    }
}

cudaError_t launch_clause(const StepArgs& a, const uint32_t* Acur, cudaStream_t st) {
    if (a.C == 0) return cudaGetLastError();
    const int NW = a.N >> 5;
    dim3 grid((NW + 31) / 32, (unsigned)((a.C + (long long)kWarps * kCH - 1) / ((long long)kWarps * kCH)));
    const int K = a.mc.K;
    const int uni = a.uniform_len;
    if (K <= 2)
        k_clause<4, 2><<<grid, 256, 0, st>>>(Acur, NW, a.cptr, a.clit, a.C, a.hist, a.N, uni && K == 2);
    else if (K == 3)
        k_clause<4, 3><<<grid, 256, 0, st>>>(Acur, NW, a.cptr, a.clit, a.C, a.hist, a.N, uni);
    else
        k_clause<8, 7><<<grid, 256, 0, st>>>(Acur, NW, a.cptr, a.clit, a.C, a.hist, a.N, uni && K == 7);
    return cudaGetLastError();
}

}  // namespace tsat
