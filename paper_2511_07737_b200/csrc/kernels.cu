// kernels.cu - sm_100a kernels of the TurboSAT step.
//
// Compiled with -fmad=false: every floating operation is a separate IEEE
// round-to-nearest op unless written as an explicit fmaf().  Together with
// integer / fixed-point cross-candidate sums this makes the GPU step
// bit-identical to the canonical step.
//
// Layouts (candidate fastest, "batch-contiguous"):
//   theta, m, v : fp32 [V][N]
//   A (bits)    : u32  [V][N/32], bit j of word w = candidate 32w + j
//   hist        : i32  [N][KB]  (bins 0..KB-2 accumulated, top bin derived)
//   gtab        : f64  [N][KB]
#include <cuda_runtime.h>
#include <stdint.h>

#include "tsat_internal.h"

namespace tsat {

// ------------------------------------------------------------------ helpers
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

// ------------------------------------------------------------------ (a1) init
// theta_vn ~ N(0,1): Philox4x32-10(key = seed, ctr = (n>>2, v, 0, 0)), Box-Muller
// on (x0,x1) -> candidates 4q, 4q+1 and (x2,x3) -> 4q+2, 4q+3.  m = v = 0.
__global__ void k_init(float* __restrict__ theta, float* __restrict__ m, float* __restrict__ vv, int V, int N,
                       long long n0, unsigned long long seed) {
    const int NQ = N >> 2;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)V * NQ) return;
    int v = (int)(i / NQ), q = (int)(i % NQ);
    long long n = n0 + 4LL * q;
    uint32_t c[4] = {(uint32_t)(n >> 2), (uint32_t)v, 0u, 0u};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const double two_pi = 6.283185307179586;
    const double s32 = 2.3283064365386963e-10;
    double u1a = ((double)c[0] + 1.0) * s32, u2a = (double)c[1] * s32;
    double u1b = ((double)c[2] + 1.0) * s32, u2b = (double)c[3] * s32;
    double ra = sqrt(-2.0 * log(u1a)), aa = two_pi * u2a;
    double rb = sqrt(-2.0 * log(u1b)), ab = two_pi * u2b;
    float4 z;
    z.x = (float)(ra * cos(aa));
    z.y = (float)(ra * sin(aa));
    z.z = (float)(rb * cos(ab));
    z.w = (float)(rb * sin(ab));
    size_t o = (size_t)v * N + 4 * (size_t)q;
    *reinterpret_cast<float4*>(theta + o) = z;
    *reinterpret_cast<float4*>(m + o) = make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4*>(vv + o) = make_float4(0.f, 0.f, 0.f, 0.f);
}

// ------------------------------------------------------------------ (a2,a3) row statistics + bits
// One CTA per variable: exact Q_v, Eq. 5 d/rho/guard, Eq. 2 bits, max |theta|.
__global__ void __launch_bounds__(256) k_rowstats(const float* __restrict__ theta, int N, MethodConsts mc,
                                                  long long* __restrict__ rowQ, double* __restrict__ rowD,
                                                  double* __restrict__ rowRho, unsigned char* __restrict__ rowGuard,
                                                  uint32_t* __restrict__ A, unsigned int* __restrict__ thmax_bits) {
    __shared__ long long sh_s[32];
    __shared__ float sh_m[32];
    __shared__ double sh_d;
    const int v = blockIdx.x;
    const float* row = theta + (size_t)v * N;
    long long s = 0;
    float mx = 0.0f;
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
        float x = row[n];
        s += __double2ll_rn((double)x * 4294967296.0);
        mx = fmaxf(mx, fabsf(x));
    }
    block_sum_max(s, mx, sh_s, sh_m);
    if (threadIdx.x == 0) {
        double d, rho;
        unsigned char g;
        row_finish(s, mc, &d, &rho, &g);
        rowQ[v] = s; rowD[v] = d; rowRho[v] = rho; rowGuard[v] = g;
        sh_d = d;
        atomicMax(thmax_bits, __float_as_uint(mx));
    }
    __syncthreads();
    const bool dpos = sh_d > 0.0;
    const int NW = N >> 5;
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
        float x = row[n];
        bool b = dpos ? (x > 0.0f) : (x < 0.0f);
        unsigned w = __ballot_sync(0xffffffffu, b);
        if ((threadIdx.x & 31) == 0) A[(size_t)v * NW + (n >> 5)] = w;
    }
}

// ------------------------------------------------------------------ (a4,a5) clause evaluation
// Bit-sliced: lane = one 32-candidate word, warp = 32 consecutive words (1024
// candidates, 128-byte coalesced gathers), each warp a chunk of clauses.
// R_cn (count of true literals) is accumulated as NP bit-planes; the one-hot
// masks [R = r] feed CB-bit vertical counters per bin; at the end each lane
// extracts per-candidate counts into a shared histogram.
template <int KB>
__global__ void __launch_bounds__(256) k_clause(const uint32_t* __restrict__ A, int NW, const uint32_t* __restrict__ cptr,
                                                const uint32_t* __restrict__ clit, long long C, int chunk,
                                                int* __restrict__ hist, int N) {
    constexpr int NP = (KB == 4) ? 2 : 3;
    constexpr int CB = 7;                       // chunk <= 127
    __shared__ int sh[(KB - 1) * 1024];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int w = blockIdx.x * 32 + lane;
    const bool valid = w < NW;
    for (int i = threadIdx.x; i < (KB - 1) * 1024; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    long long c0 = ((long long)blockIdx.y * 8 + warp) * chunk;
    long long c1 = c0 + chunk < C ? c0 + chunk : C;
    uint32_t cnt[KB - 1][CB];
#pragma unroll
    for (int r = 0; r < KB - 1; ++r)
#pragma unroll
        for (int b = 0; b < CB; ++b) cnt[r][b] = 0u;
    for (long long c = c0; c < c1; ++c) {
        uint32_t beg = cptr[c], end = cptr[c + 1];
        uint32_t s[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) s[p] = 0u;
        for (uint32_t l = beg; l < end; ++l) {
            uint32_t code = clit[l];
            uint32_t x = valid ? A[(size_t)(code >> 1) * NW + w] : 0u;
            x ^= (code & 1u) ? 0xffffffffu : 0u;
            uint32_t carry = x;
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                uint32_t t = s[p] & carry;
                s[p] ^= carry;
                carry = t;
            }
        }
#pragma unroll
        for (int r = 0; r < KB - 1; ++r) {
            uint32_t msk = 0xffffffffu;
#pragma unroll
            for (int p = 0; p < NP; ++p) msk &= ((r >> p) & 1) ? s[p] : ~s[p];
            uint32_t carry = msk;
#pragma unroll
            for (int b = 0; b < CB; ++b) {
                uint32_t t = cnt[r][b] & carry;
                cnt[r][b] ^= carry;
                carry = t;
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

// ------------------------------------------------------------------ (a6) SmoothMin / g table
// Per candidate: h[0..K] (top bin KB-1 derived as C - sum), rmin, Eq. 4 via
// the E table, g[r] = (E[r-rmin]/den)(1 - tau(r - S)); unsat; best key; gmax.
// Clears the histogram for the next iteration.
template <int KB>
__global__ void __launch_bounds__(256) k_gtable(int* __restrict__ hist, int N, long long C, MethodConsts mc,
                                                double* __restrict__ gtab, double* __restrict__ S,
                                                int* __restrict__ unsat, DevScalars* __restrict__ ds) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    unsigned long long key = ~0ull;
    double gm = 0.0;
    if (n < N) {
        long long h[KB];
        long long acc = 0;
#pragma unroll
        for (int r = 0; r < KB - 1; ++r) {
            h[r] = hist[(size_t)n * KB + r];
            hist[(size_t)n * KB + r] = 0;
            acc += h[r];
        }
        h[KB - 1] = C - acc;
        const int K = mc.K;
        int rmin = 0;
        while (rmin <= K && h[rmin] == 0) ++rmin;
        double g[KB];
#pragma unroll
        for (int r = 0; r < KB; ++r) g[r] = 0.0;
        double s = 0.0;
        if (rmin <= K) {
            double den = 0.0, num = 0.0;
            for (int r = rmin; r <= K; ++r) {
                den = den + (double)h[r] * mc.E[r - rmin];
                num = num + (double)((long long)r * h[r]) * mc.E[r - rmin];
            }
            s = num / den;
#pragma unroll
            for (int r = 0; r < KB; ++r) {
                if (r >= rmin && r <= K) {
                    double wgt = mc.E[r - rmin] / den;
                    double u = (double)r - s;
                    g[r] = wgt * (1.0 - mc.tau * u);
                    gm = fmax(gm, fabs(g[r]));
                }
            }
        }
#pragma unroll
        for (int r = 0; r < KB; ++r) gtab[(size_t)n * KB + r] = g[r];
        S[n] = s;
        unsat[n] = (int)h[0];
        key = ((unsigned long long)h[0] << 32) | (unsigned long long)(mc.n0 + n);
    }
    unsigned long long gb = (unsigned long long)__double_as_longlong(gm);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long k2 = __shfl_xor_sync(0xffffffffu, key, o);
        unsigned long long g2 = __shfl_xor_sync(0xffffffffu, gb, o);
        key = k2 < key ? k2 : key;
        gb = g2 > gb ? g2 : gb;
    }
    if (lane == 0) {
        atomicMin(&ds->best_key, key);
        atomicMax(&ds->gmax_bits, gb);
    }
}

// ------------------------------------------------------------------ (a7-a10) backward + Jacobian + AdamW + re-binarise
// One CTA per variable v, all N candidates of the row (W = 1 fused path).
//  1. G_vn = sum_r (cneg - cpos)[r] g_n[r]: for every occurrence of v the
//     clause's R_cn is recomputed from the bit planes of the evaluated state.
//  2. J_v = sum_n G_vn theta_vn in int64 fixed point (scale s_v from the
//     global gmax, thmax); c_v = ((J/N) rho) rho.
//  3. grad = (float)(G rho - c); AdamW (PyTorch order, R6); optional noise.
//  4. Q_{t+1} exact, d/rho/guard for t+1, bits of theta_{t+1}, max |theta|.
template <int KB>
__global__ void __launch_bounds__(256) k_update(float* __restrict__ theta, float* __restrict__ m, float* __restrict__ vv,
                                                int N, const uint32_t* __restrict__ Acur, uint32_t* __restrict__ Anext,
                                                const uint32_t* __restrict__ occ_ptr, const uint32_t* __restrict__ occ_rec,
                                                const uint32_t* __restrict__ occ_cnt, const double* __restrict__ gtab,
                                                long long* __restrict__ rowQ, double* __restrict__ rowD,
                                                double* __restrict__ rowRho, unsigned char* __restrict__ rowGuard,
                                                DevScalars* __restrict__ ds, const StepScalars* __restrict__ sc,
                                                MethodConsts mc, unsigned char* __restrict__ sol) {
    extern __shared__ double smem[];
    double* Gs = smem;                                       // [N]
    float* Ts = reinterpret_cast<float*>(smem + N);          // [N]
    __shared__ long long sh_s[32];
    __shared__ float sh_m[32];
    __shared__ double sh_c, sh_d;
    const int v = blockIdx.x;
    const int NW = N >> 5;
    const long long t = sc->t;
    const unsigned rb = occ_ptr[v], re = occ_ptr[v + 1];
    const unsigned occ = occ_cnt[v];
    const double d = rowD[v], rho = rowRho[v];
    const unsigned char guard = rowGuard[v];
    const double gmax = __longlong_as_double((long long)ds->gmax_bits);
    const float thmax = __uint_as_float(ds->thmax_bits[t & 1]);
    // fixed-point scale for J_v (R13)
    int s = 0;
    bool jvalid = false;
    {
        double x = (double)mc.Nglobal * (double)occ;
        x = x * gmax;
        x = x * (double)thmax;
        if (occ > 0 && x > 0.0) { jvalid = true; s = 61 - ceil_log2(x); }
    }
    const uint32_t* Arow = Acur + (size_t)v * NW;
    float* trow = theta + (size_t)v * N;
    float* mrow = m + (size_t)v * N;
    float* vrow = vv + (size_t)v * N;
    long long I = 0;
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
        const int w = n >> 5, j = n & 31;
        const uint32_t own = (Arow[w] >> j) & 1u;
        int cnt[KB];
#pragma unroll
        for (int r = 0; r < KB; ++r) cnt[r] = 0;
        for (unsigned p = rb; p < re;) {
            const uint32_t hdr = occ_rec[p];
            const uint32_t len = hdr >> 1;
            uint32_t R = own ^ (hdr & 1u);
            for (uint32_t i = 1; i < len; ++i) {
                const uint32_t code = occ_rec[p + i];
                R += ((Acur[(size_t)(code >> 1) * NW + w] >> j) & 1u) ^ (code & 1u);
            }
            const int delta = (hdr & 1u) ? 1 : -1;         // cneg - cpos
#pragma unroll
            for (int r = 0; r < KB; ++r) cnt[r] += (R == (uint32_t)r) ? delta : 0;
            p += len;
        }
        double G = 0.0;
        const double* gn = gtab + (size_t)n * KB;
#pragma unroll
        for (int r = 0; r < KB; ++r)
            if (r <= mc.K) G = G + (double)cnt[r] * gn[r];
        Gs[n] = G;
        if (jvalid) {
            double pr = G * (double)trow[n];
            I += __double2ll_rn(scalbn(pr, s));
        }
    }
    float dummy = 0.0f;
    block_sum_max(I, dummy, sh_s, sh_m);
    if (threadIdx.x == 0) {
        double J = jvalid ? scalbn((double)I, -s) : 0.0;
        double c = 0.0;
        if (mc.normalize && !guard) {
            c = J / (double)mc.Nglobal;
            c = c * rho;
            c = c * rho;
        }
        sh_c = c;
    }
    __syncthreads();
    const double c = sh_c;
    const float wdf = sc->wdf, a1 = sc->a1, b2f = sc->b2f, a2 = sc->a2, nss = sc->nss, bc2s = sc->bc2s,
                epsf = sc->epsf, nz = sc->nz;
    long long Qn = 0;
    float mx = 0.0f;
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
        const double a = Gs[n] * rho;
        const float g = (float)(a - c);
        float th = trow[n] * wdf;
        const float m0 = mrow[n];
        const float mm = __fmaf_rn(a1, g - m0, m0);
        const float vb = vrow[n] * b2f;
        const float vn = __fmaf_rn(a2 * g, g, vb);
        const float den = __fsqrt_rn(vn) / bc2s + epsf;
        th = th + (nss * mm) / den;
        if (mc.noise) {
            const long long ng = mc.n0 + n;
            uint32_t x[4] = {(uint32_t)(ng >> 2), (uint32_t)v, (uint32_t)(1 + t), 0u};
            philox4x32_10(x, (uint32_t)mc.seed, (uint32_t)(mc.seed >> 32));
            const float xi = (float)(x[ng & 3] >> 8) * 5.9604644775390625e-08f - 0.5f;
            th = th + nz * xi;
        }
        trow[n] = th;
        mrow[n] = mm;
        vrow[n] = vn;
        Ts[n] = th;
        Qn += __double2ll_rn((double)th * 4294967296.0);
        mx = fmaxf(mx, fabsf(th));
    }
    block_sum_max(Qn, mx, sh_s, sh_m);
    if (threadIdx.x == 0) {
        double dn, rhon;
        unsigned char gn;
        row_finish(Qn, mc, &dn, &rhon, &gn);
        rowQ[v] = Qn; rowD[v] = dn; rowRho[v] = rhon; rowGuard[v] = gn;
        sh_d = dn;
        atomicMax(&ds->thmax_bits[(t + 1) & 1], __float_as_uint(mx));
        // first model: keep its bits of the evaluated state (A22)
        const unsigned long long bk = ds->best_key;
        if ((bk >> 32) == 0ull && ds->sol_step < 0) {
            const long long idx = (long long)(bk & 0xffffffffull) - mc.n0;
            if (idx >= 0 && idx < N) sol[v] = (unsigned char)((Arow[idx >> 5] >> (idx & 31)) & 1u);
        }
    }
    __syncthreads();
    const bool dpos = sh_d > 0.0;
    uint32_t* Anrow = Anext + (size_t)v * NW;
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
        const float x = Ts[n];
        const unsigned wv = __ballot_sync(0xffffffffu, dpos ? (x > 0.0f) : (x < 0.0f));
        if ((threadIdx.x & 31) == 0) Anrow[n >> 5] = wv;
    }
}

// ------------------------------------------------------------------ end of iteration
// Loss (deterministic fixed-shape reduction), first-model bookkeeping, step
// info, and reset of the per-iteration accumulators.
__global__ void __launch_bounds__(1024) k_step_end(const double* __restrict__ S, int N, DevScalars* __restrict__ ds,
                                                   const StepScalars* __restrict__ sc) {
    __shared__ double sh[32];
    double a = 0.0;
    for (int n = threadIdx.x; n < N; n += blockDim.x) a = a + S[n];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = a + __shfl_xor_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x < 32) {
        double b = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) b = b + __shfl_xor_sync(0xffffffffu, b, o);
        if (threadIdx.x == 0) {
            const long long t = sc->t;
            const unsigned long long bk = ds->best_key;
            const int bu = (int)(bk >> 32);
            const long long bi = (long long)(bk & 0xffffffffull);
            if (bu == 0 && ds->sol_step < 0) { ds->sol_step = t; ds->sol_idx = bi; }
            ds->loss = -b;
            ds->info_t = t + 1;
            ds->info_best_unsat = bu;
            ds->info_best_idx = bi;
            ds->info_loss = -b;
            ds->best_key = ~0ull;
            ds->gmax_bits = 0ull;
            ds->thmax_bits[t & 1] = 0u;
        }
    }
}

// ------------------------------------------------------------------ export helpers
// Variable gradient G_vn (pre-Jacobian) of the last evaluated state for a list
// of candidates: out[m * V + v] = |G| as fp64.
template <int KB>
__global__ void __launch_bounds__(256) k_grad_cols(int V, int N, const uint32_t* __restrict__ Acur,
                                                   const uint32_t* __restrict__ occ_ptr, const uint32_t* __restrict__ occ_rec,
                                                   const double* __restrict__ gtab, const int* __restrict__ cols, int M,
                                                   int K, double* __restrict__ out) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)M * V) return;
    const int mi = (int)(i / V), v = (int)(i % V);
    const int n = cols[mi];
    const int NW = N >> 5;
    const int w = n >> 5, j = n & 31;
    const uint32_t own = (Acur[(size_t)v * NW + w] >> j) & 1u;
    int cnt[KB];
#pragma unroll
    for (int r = 0; r < KB; ++r) cnt[r] = 0;
    for (unsigned p = occ_ptr[v]; p < occ_ptr[v + 1];) {
        const uint32_t hdr = occ_rec[p];
        const uint32_t len = hdr >> 1;
        uint32_t R = own ^ (hdr & 1u);
        for (uint32_t q = 1; q < len; ++q) {
            const uint32_t code = occ_rec[p + q];
            R += ((Acur[(size_t)(code >> 1) * NW + w] >> j) & 1u) ^ (code & 1u);
        }
        const int delta = (hdr & 1u) ? 1 : -1;
#pragma unroll
        for (int r = 0; r < KB; ++r) cnt[r] += (R == (uint32_t)r) ? delta : 0;
        p += len;
    }
    double G = 0.0;
#pragma unroll
    for (int r = 0; r < KB; ++r)
        if (r <= K) G = G + (double)cnt[r] * gtab[(size_t)n * KB + r];
    out[(size_t)mi * V + v] = fabs(G);
}

// Single-CTA bitonic sort of n64 (power of two) u64 keys in global memory.
__global__ void __launch_bounds__(1024) k_bitonic_sort(unsigned long long* __restrict__ keys, int n64) {
    for (int k = 2; k <= n64; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int i = threadIdx.x; i < n64; i += blockDim.x) {
                int ixj = i ^ jj;
                if (ixj > i) {
                    unsigned long long a = keys[i], b = keys[ixj];
                    bool up = (i & k) == 0;
                    if ((a > b) == up) { keys[i] = b; keys[ixj] = a; }
                }
            }
            __syncthreads();
        }
    }
}

__global__ void k_make_keys(const int* __restrict__ unsat, int N, long long n0, int n64,
                            unsigned long long* __restrict__ keys) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n64) return;
    keys[i] = i < N ? (((unsigned long long)(unsigned)unsat[i] << 32) | (unsigned long long)(n0 + i)) : ~0ull;
}

// k smallest (|G|, v) per column: MSB-first radix select over the 96-bit key
// (fp64 bits of |G| : v), then an in-CTA bitonic sort of the k winners.
// One CTA (1024 threads) per column; k <= kTopkMax.
__global__ void __launch_bounds__(1024) k_topk_cols(const double* __restrict__ absG, int V, int k,
                                                    int* __restrict__ out_v, double* __restrict__ out_g) {
    __shared__ unsigned int hist[256];
    __shared__ unsigned long long pref_hi;
    __shared__ unsigned int pref_lo;
    __shared__ int remaining, nsel;
    __shared__ unsigned long long sel_hi[kTopkMax];
    __shared__ unsigned int sel_lo[kTopkMax];
    const int col = blockIdx.x;
    const double* g = absG + (size_t)col * V;
    if (threadIdx.x == 0) { pref_hi = 0; pref_lo = 0; remaining = k; nsel = 0; }
    __syncthreads();
    // 12 digit passes: digits 0..7 from the 64-bit |G| bits, 8..11 from v
    for (int pass = 0; pass < 12; ++pass) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const unsigned long long ph = pref_hi;
        const unsigned int pl = pref_lo;
        for (int v = threadIdx.x; v < V; v += blockDim.x) {
            unsigned long long hi = (unsigned long long)__double_as_longlong(g[v]);
            unsigned int lo = (unsigned int)v;
            bool match;
            unsigned digit;
            if (pass < 8) {
                int sh = 64 - 8 * pass;                       // bits above the current digit
                match = (pass == 0) || ((hi >> sh) == ph);
                digit = (unsigned)((hi >> (56 - 8 * pass)) & 0xffu);
            } else {
                int p2 = pass - 8;
                int sh = 32 - 8 * p2;
                match = (hi == ph) && (p2 == 0 || (lo >> sh) == pl);
                digit = (lo >> (24 - 8 * p2)) & 0xffu;
            }
            if (match) atomicAdd(&hist[digit], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int rem = remaining;
            unsigned b = 0;
            for (; b < 256; ++b) {
                if ((int)hist[b] >= rem) break;
                rem -= (int)hist[b];
            }
            if (b > 255) b = 255;
            remaining = rem;
            if (pass < 8) pref_hi = (pref_hi << 8) | b;
            else pref_lo = (pref_lo << 8) | b;
        }
        __syncthreads();
    }
    // threshold key T = (pref_hi, pref_lo): the k-th smallest; collect keys <= T
    const unsigned long long th = pref_hi;
    const unsigned int tl = pref_lo;
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
        unsigned long long hi = (unsigned long long)__double_as_longlong(g[v]);
        if (hi < th || (hi == th && (unsigned)v <= tl)) {
            int pos = atomicAdd(&nsel, 1);
            if (pos < kTopkMax) { sel_hi[pos] = hi; sel_lo[pos] = (unsigned)v; }
        }
    }
    __syncthreads();
    int cnt = nsel < kTopkMax ? nsel : kTopkMax;
    int n2 = 1;
    while (n2 < cnt) n2 <<= 1;
    for (int i = cnt + threadIdx.x; i < n2; i += blockDim.x) { sel_hi[i] = ~0ull; sel_lo[i] = ~0u; }
    __syncthreads();
    for (int kk = 2; kk <= n2; kk <<= 1)
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                int ixj = i ^ jj;
                if (ixj > i) {
                    bool up = (i & kk) == 0;
                    bool gt = sel_hi[i] > sel_hi[ixj] || (sel_hi[i] == sel_hi[ixj] && sel_lo[i] > sel_lo[ixj]);
                    if (gt == up) {
                        unsigned long long a = sel_hi[i]; sel_hi[i] = sel_hi[ixj]; sel_hi[ixj] = a;
                        unsigned int b = sel_lo[i]; sel_lo[i] = sel_lo[ixj]; sel_lo[ixj] = b;
                    }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < k && i < cnt; i += blockDim.x) {
        out_v[(size_t)col * k + i] = (int)sel_lo[i];
        out_g[(size_t)col * k + i] = __longlong_as_double((long long)sel_hi[i]);
    }
}

// ------------------------------------------------------------------ launchers
#define TSAT_CK(x)                                   \
    do {                                             \
        cudaError_t e_ = (x);                        \
        if (e_ != cudaSuccess) return e_;            \
    } while (0)

cudaError_t launch_init(float* theta, float* m, float* v, int V, int N, long long n0, unsigned long long seed,
                        cudaStream_t st) {
    long long total = (long long)V * (N / 4);
    int threads = 256;
    long long blocks = (total + threads - 1) / threads;
    if (blocks > 0) k_init<<<(unsigned)blocks, threads, 0, st>>>(theta, m, v, V, N, n0, seed);
    return cudaGetLastError();
}

cudaError_t launch_rowstats(const float* theta, int V, int N, const MethodConsts& mc, long long* rowQ, double* rowD,
                            double* rowRho, unsigned char* rowGuard, uint32_t* A, unsigned int* thmax_bits,
                            cudaStream_t st) {
    if (V > 0) k_rowstats<<<V, 256, 0, st>>>(theta, N, mc, rowQ, rowD, rowRho, rowGuard, A, thmax_bits);
    return cudaGetLastError();
}

// kernel index: 0 clause, 1 gtable, 2 update, 3 step_end
cudaError_t launch_step_kernel(int which, const StepArgs& a, const StepScalars* sc_dev, long long t, cudaStream_t st) {
    const int NW = a.N >> 5;
    const uint32_t* Acur = (t & 1) ? a.A1 : a.A0;
    uint32_t* Anext = (t & 1) ? a.A0 : a.A1;
    switch (which) {
        case 0: {
            const int chunk = 64;
            dim3 grid((NW + 31) / 32, (unsigned)((a.C + 8LL * chunk - 1) / (8LL * chunk)));
            if (a.C == 0) return cudaGetLastError();
            if (a.KB == 4) k_clause<4><<<grid, 256, 0, st>>>(Acur, NW, a.cptr, a.clit, a.C, chunk, a.hist, a.N);
            else k_clause<8><<<grid, 256, 0, st>>>(Acur, NW, a.cptr, a.clit, a.C, chunk, a.hist, a.N);
            break;
        }
        case 1: {
            int blocks = (a.N + 255) / 256;
            if (a.KB == 4) k_gtable<4><<<blocks, 256, 0, st>>>(a.hist, a.N, a.C, a.mc, a.gtab, a.S, a.unsat, a.ds);
            else k_gtable<8><<<blocks, 256, 0, st>>>(a.hist, a.N, a.C, a.mc, a.gtab, a.S, a.unsat, a.ds);
            break;
        }
        case 2: {
            size_t smem = (size_t)a.N * (sizeof(double) + sizeof(float));
            if (a.V == 0) return cudaGetLastError();
            if (a.KB == 4)
                k_update<4><<<a.V, 256, smem, st>>>(a.theta, a.m, a.v, a.N, Acur, Anext, a.occ_ptr, a.occ_rec, a.occ_cnt,
                                                    a.gtab, a.rowQ, a.rowD, a.rowRho, a.rowGuard, a.ds, sc_dev, a.mc, a.sol);
            else
                k_update<8><<<a.V, 256, smem, st>>>(a.theta, a.m, a.v, a.N, Acur, Anext, a.occ_ptr, a.occ_rec, a.occ_cnt,
                                                    a.gtab, a.rowQ, a.rowD, a.rowRho, a.rowGuard, a.ds, sc_dev, a.mc, a.sol);
            break;
        }
        case 3:
            k_step_end<<<1, 1024, 0, st>>>(a.S, a.N, a.ds, sc_dev);
            break;
    }
    return cudaGetLastError();
}

cudaError_t configure_kernels(int N) {
    size_t smem = (size_t)N * (sizeof(double) + sizeof(float));
    TSAT_CK(cudaFuncSetAttribute(k_update<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    TSAT_CK(cudaFuncSetAttribute(k_update<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    return cudaSuccess;
}

cudaError_t launch_export(const StepArgs& a, long long t_eval, const int* cols_dev, int M, int k, double* absG,
                          unsigned long long* keys, int n64, int* out_v, double* out_g, cudaStream_t st, int phase) {
    const uint32_t* Aeval = (t_eval & 1) ? a.A1 : a.A0;
    if (phase == 0) {
        k_make_keys<<<(n64 + 255) / 256, 256, 0, st>>>(a.unsat, a.N, a.mc.n0, n64, keys);
        k_bitonic_sort<<<1, 1024, 0, st>>>(keys, n64);
    } else {
        long long total = (long long)M * a.V;
        unsigned blocks = (unsigned)((total + 255) / 256);
        if (a.KB == 4) k_grad_cols<4><<<blocks, 256, 0, st>>>(a.V, a.N, Aeval, a.occ_ptr, a.occ_rec, a.gtab, cols_dev, M, a.mc.K, absG);
        else k_grad_cols<8><<<blocks, 256, 0, st>>>(a.V, a.N, Aeval, a.occ_ptr, a.occ_rec, a.gtab, cols_dev, M, a.mc.K, absG);
        k_topk_cols<<<M, 1024, 0, st>>>(absG, a.V, k, out_v, out_g);
    }
    return cudaGetLastError();
}

}  // namespace tsat
