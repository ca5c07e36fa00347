// k_dense.cu - SURVEY §8(f) f4: rows (a4) R = P A and (a5) the histogram as a
// DENSE tensor-core product, the paper's literal "GEMM" framing (PAPER.md
// l.131: "leveraging GPU-accelerated GEMM"; Eq. 1 l.185-188).
//
// P is the C x 2V binary problem matrix (row c: the literals of clause c,
// column l = 2v + negated) and A the 2V x N binary assignment matrix (A[2v][n]
// = b_vn, A[2v+1][n] = 1 - b_vn), both stored as uint8 0/1, K-major (a
// clause's / a candidate's 2V literal bytes contiguous).  One CTA computes a
// 128-clause x 256-candidate tile of R with tcgen05.mma.kind::i8 (uint8 x
// uint8 -> int32 in TMEM; exact: R <= 15), operands staged in shared memory
// in the canonical no-swizzle K-major layout (8-row x 16-byte core matrices),
// K in chunks of 64 bytes (2 MMAs of K = 32), double-buffered (the next
// chunk's cp.async loads overlap the current MMAs).  The epilogue reads R with
// tcgen05.ld (one clause row per thread), turns each candidate column into
// 4 bit planes with warp ballots and adds popcount(bin masks) to the
// CTA's shared histogram, then one global atomic per (candidate, bin) per CTA
// (bins 0 .. KB-2; k_gtable derives the top bin).
//
// This is an experiment (config.clause_eval = 1): the sparse bit-sliced
// k_clause moves 1 bit per literal occurrence and candidate; the dense form
// does C x 2V x N MACs, so it can only win on small clause-dense instances
// (measured in profiles/).
#include <cstdint>

#include "device_common.cuh"

namespace tsat {

namespace {
constexpr int kDM = 128, kDN = 256, kDKC = 64;         // tile M (clauses), N (candidates), K chunk (bytes)
constexpr int kAStep = kDM / 8 * 256, kBStep = kDN / 8 * 256;   // bytes per 32-byte k-step (A, B)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Shared-memory matrix descriptor (sm100): start >> 4 [0,14), LBO >> 4
// [16,30), SBO >> 4 [32,46), version 1 [46,48), layout SWIZZLE_NONE (0) [61,64).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// Instruction descriptor, kind::i8: D s32 (bits 4-5 = 2), A/B uint8 (0), both
// K-major, N >> 3 at bit 17, M >> 4 at bit 24.
constexpr uint32_t kIdesc = (2u << 4) | ((uint32_t)(kDN >> 3) << 17) | ((uint32_t)(kDM >> 4) << 24);

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(a), "r"(phase) : "memory");
    } while (!done);
}
}  // namespace

// A (K-major) from the bit planes: AL[n][2v] = b_vn, AL[n][2v+1] = 1 - b_vn.
// Thread per (candidate, 8 variables): 16 bytes stored.
__global__ void k_dense_pack(const uint32_t* __restrict__ A, int V, int NW, int N, int Kp, uint8_t* __restrict__ AL) {
    const int groups = (V + 7) >> 3;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)N * groups) return;
    const int n = (int)(i / groups), g = (int)(i % groups);
    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int v = 8 * g + j;
        if (v >= V) break;
        const uint32_t b = (__ldg(A + (size_t)v * NW + (n >> 5)) >> (n & 31)) & 1u;
        const uint32_t pair = b | ((b ^ 1u) << 8);          // bytes (2v, 2v + 1)
        w[j >> 1] |= pair << (16 * (j & 1));
    }
    *reinterpret_cast<uint4*>(AL + (size_t)n * Kp + 16 * g) = make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void __launch_bounds__(128, 2) k_dense_clause(const uint8_t* __restrict__ P, const uint8_t* __restrict__ AL,
                                                          long long C, int Kp, int N, int KB, int* __restrict__ hist,
                                                          DevScalars* __restrict__ ds, const StepScalars* __restrict__ sc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    constexpr int kStage = (kDKC / 32) * (kAStep + kBStep);      // one K chunk of both operands
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ uint32_t tmem_base;
    __shared__ int shist[16 * kDN];                               // the CTA's counts: [bin][column]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long m0 = (long long)blockIdx.y * kDM;
    const int n0 = blockIdx.x * kDN;
    pdl_wait();
    pdl_trigger();
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) {      // the iteration's accumulators (as k_clause)
        const long long t = sc->t;
        ds->best_key = ~0ull;
        ds->gmax_bits = 0ull;
        ds->row_counter = 0;
        ds->thmax_bits[(t + 1) & 1] = 0u;
        ds->loss_fx = 0;
    }
    for (int i = tid; i < kDN * 16; i += 128) shist[i] = 0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(kDN) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;
    // operand chunk -> canonical K-major layout of stage `st`: core matrix
    // (8 rows x 16 B) at ks * step + (row / 8) * 256 + half * 128 (LBO 128, SBO 256)
    auto load_chunk = [&](int kc, int st) {
        const int kb = Kp - kc < kDKC ? Kp - kc : kDKC, nch = kb / 16;
        uint8_t* sA = sm + st * kStage;
        uint8_t* sB = sA + (kDKC / 32) * kAStep;
        for (int idx = tid; idx < kDM * nch; idx += 128) {
            const int row = idx / nch, ch = idx % nch;
            const uint32_t dst = smem_u32(sA) + (ch >> 1) * kAStep + (row >> 3) * 256 + (ch & 1) * 128 + (row & 7) * 16;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(P + (size_t)(m0 + row) * Kp + kc + ch * 16)
                         : "memory");
        }
        for (int idx = tid; idx < kDN * nch; idx += 128) {
            const int row = idx / nch, ch = idx % nch;
            const uint32_t dst = smem_u32(sB) + (ch >> 1) * kBStep + (row >> 3) * 256 + (ch & 1) * 128 + (row & 7) * 16;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(AL + (size_t)(n0 + row) * Kp + kc + ch * 16)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // 2-stage pipeline: chunk i+1 loads while the tensor core consumes chunk i
    const int nk = (Kp + kDKC - 1) / kDKC;
    uint32_t ph[2] = {0u, 0u};
    load_chunk(0, 0);
    for (int i = 0; i < nk; ++i) {
        const int st = i & 1, kc = i * kDKC;
        if (i + 1 < nk) {
            if (i >= 1) { mbar_wait(&mbar[st ^ 1], ph[st ^ 1]); ph[st ^ 1] ^= 1u; }   // MMAs of chunk i-1 done
            load_chunk(kc + kDKC, st ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");                      // chunk i landed
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic-proxy writes -> tensor core
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int kb = Kp - kc < kDKC ? Kp - kc : kDKC;
            const uint32_t sA = smem_u32(sm + st * kStage), sB = sA + (kDKC / 32) * kAStep;
            for (int ks = 0; ks < kb / 32; ++ks) {
                const uint64_t ad = sdesc(sA + ks * kAStep, 128, 256);
                const uint64_t bd = sdesc(sB + ks * kBStep, 128, 256);
                const uint32_t acc = (kc > 0 || ks > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                    ::"r"(tmem), "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc) : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                         ::"r"(smem_u32(&mbar[st])) : "memory");
        }
    }
    {   // the last chunk's MMAs (and, in issue order, all earlier ones) complete
        const int st = (nk - 1) & 1;
        mbar_wait(&mbar[st], ph[st]);
        if (nk >= 2) mbar_wait(&mbar[st ^ 1], ph[st ^ 1]);
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: thread = clause row m0 + 32 warp + lane; 32 candidate columns at a time
    const bool vrow = m0 + 32 * warp + lane < C;
    const uint32_t vmask = __ballot_sync(0xffffffffu, vrow);
    for (int c0 = 0; c0 < kDN; c0 += 32) {
        uint32_t r[32];
        const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // column c0 + j's four bit planes over the warp's 32 clauses -> lane j
        uint32_t q0 = 0u, q1 = 0u, q2 = 0u, q3 = 0u;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const uint32_t b0 = __ballot_sync(0xffffffffu, r[j] & 1u), b1 = __ballot_sync(0xffffffffu, r[j] & 2u);
            const uint32_t b2 = __ballot_sync(0xffffffffu, r[j] & 4u), b3 = __ballot_sync(0xffffffffu, r[j] & 8u);
            if (lane == j) { q0 = b0; q1 = b1; q2 = b2; q3 = b3; }
        }
        for (int rr = 0; rr < KB - 1; ++rr) {
            const uint32_t m = vmask & ((rr & 1) ? q0 : ~q0) & ((rr & 2) ? q1 : ~q1) & ((rr & 4) ? q2 : ~q2) &
                               ((rr & 8) ? q3 : ~q3);
            const int cnt = __popc(m);
            if (cnt) atomicAdd(&shist[rr * kDN + c0 + lane], cnt);     // consecutive lanes: no bank conflict
        }
    }
    __syncthreads();
    for (int i = tid; i < kDN * 16; i += 128) {           // one global atomic per (column, bin) per CTA
        const int col = i % kDN, rr = i / kDN, n = n0 + col;
        const int x = shist[i];
        if (x && n < N && rr < KB - 1) atomicAdd(&hist[(size_t)n * KB + rr], x);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kDN) : "memory");
}

size_t dense_smem_bytes() { return 2 * (size_t)(kDKC / 32) * (kAStep + kBStep); }   // 2 stages
cudaError_t configure_dense() {
    return cudaFuncSetAttribute(k_dense_clause, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dense_smem_bytes());
}
int dense_tile_m() { return kDM; }
int dense_tile_n() { return kDN; }

cudaError_t launch_dense_clause(const StepArgs& a, const uint32_t* Acur, const StepScalars* sc, cudaStream_t st) {
    const int NW = a.N >> 5;
    const long long packs = (long long)a.N * ((a.V + 7) >> 3);
    if (packs > 0)
        k_dense_pack<<<(unsigned)((packs + 255) / 256), 256, 0, st>>>(Acur, a.V, NW, a.N, a.dKp, a.dAL);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const dim3 grid((unsigned)((a.N + kDN - 1) / kDN), (unsigned)(a.dCp / kDM));
    k_dense_clause<<<grid, 128, dense_smem_bytes(), st>>>(a.dP, a.dAL, a.C, a.dKp, a.N, a.KB, a.hist, a.ds, sc);
    return cudaGetLastError();
}

}  // namespace tsat
