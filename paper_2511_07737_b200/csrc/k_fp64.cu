// k_fp64.cu - variant f2 "fp64 state" (reading R30):
// rows (a1)-(a3) and (a7)-(a9) with theta, m, v in fp64 and every rounding the
// fp32 readings R13/R26/R27/R27b/R6 make taken in fp64 instead
// (§3.2 l.189-191, l.226; §4.1 l.250-269).  The clause evaluation,
// histogram and SmoothMin kernels are shared with the fp32 path (k_gtable
// also writes its fp64 table).  Correctness-first, one thread per (variable,
// candidate), 48 B of state per (v, n):
//   k_fold64  : counts of the row's occurrences per candidate (bits read from
//               the evaluated state's planes), G = fp64 FMA chain over the
//               bins r ascending, J_v partial in int64 fixed point (exact,
//               integer atomics are order-free);
//   k_adam64  : grad = fma(G, rho, -c), fp64 AdamW, 128-bit row-sum partial
//               at 2^-64 per 256-candidate block, max |theta|, sign words;
//   k_rows64  : Eq. 5 statistics of the next state from the exact 128-bit
//               row sum, its bit planes, the first model's bits.
#include "device_common.cuh"

namespace tsat {

namespace {
constexpr int kB64 = 256;            // candidates per block (8 warps = 8 words of the bit planes)

// round_half_even(x 2^64) as a 128-bit integer (x 2^64 exact in fp64; R30).
__device__ __forceinline__ __int128 round64_q(double x) {
    const double y = x * 18446744073709551616.0;
    if (fabs(y) < 4503599627370496.0) return (__int128)__double2ll_rn(y);
    const double hi = floor(y * 5.421010862427522e-20);
    const double lo = y - hi * 18446744073709551616.0;
    return (__int128)(long long)hi * ((__int128)1 << 64) + (__int128)(unsigned long long)lo;
}

__device__ __forceinline__ __int128 warp_sum128(__int128 x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long lo = (unsigned long long)x, hi = (unsigned long long)(x >> 64);
        const unsigned long long lo2 = __shfl_xor_sync(0xffffffffu, lo, o);
        const unsigned long long hi2 = __shfl_xor_sync(0xffffffffu, hi, o);
        x += ((__int128)hi2 << 64) | (__int128)lo2;
    }
    return x;
}

// Eq. 5 statistics from the 128-bit row sum (R30): S = (double)hi 2^64 +
// (double)lo, mu = (S 2^-64) / N, then d, rho, guard as row_finish (R3).
__device__ __forceinline__ void row_finish64(long long hi, unsigned long long lo, const MethodConsts& mc, double* d,
                                             double* rho, unsigned char* guard) {
    if (!mc.normalize) { *d = 1.0; *rho = 1.0; *guard = 1; return; }
    const double S = __dadd_rn(__dmul_rn((double)hi, 18446744073709551616.0), __ull2double_rn(lo));
    const double mu = __dmul_rn(S, 5.421010862427522e-20) / (double)mc.Nnorm;
    const double a = fabs(mu);
    const double mag = a > mc.eps_norm ? a : mc.eps_norm;
    *d = mu >= 0.0 ? mag : -mag;
    *rho = 1.0 / *d;
    *guard = (a <= mc.eps_norm) ? 1 : 0;
}

// ceil(log2(x)) for finite x > 0
__device__ __forceinline__ int ceil_log2_64(double x) {
    int e;
    const double f = frexp(x, &e);
    return (f == 0.5) ? e - 1 : e;
}
}  // namespace

int fp64_blocks_per_row(int N) { return (N + kB64 - 1) / kB64; }

// theta0 = the fp64 Box-Muller value of k_init's Philox draw (not rounded).
__global__ void k_init64(double* __restrict__ th, double* __restrict__ m, double* __restrict__ v, int V, int N,
                         long long n0, unsigned long long seed) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int vr = blockIdx.y;
    if (j >= N) return;
    const long long n = n0 + j;
    uint32_t x[4] = {(uint32_t)(n >> 2), (uint32_t)vr, 0u, 0u};
    philox4x32_10(x, (uint32_t)seed, (uint32_t)(seed >> 32));
    const int q = (int)(n & 3), pair = q >> 1;
    const double u1 = ((double)x[2 * pair] + 1.0) * 2.3283064365386963e-10;
    const double u2 = (double)x[2 * pair + 1] * 2.3283064365386963e-10;
    const double r = sqrt(-2.0 * log(u1));
    const double ang = 6.283185307179586 * u2;
    const size_t i = (size_t)vr * N + j;
    th[i] = (q & 1) ? r * sin(ang) : r * cos(ang);
    m[i] = 0.0;
    v[i] = 0.0;
}

// Row-sum partials, max |theta| and sign words of a state (init / set_state).
__global__ void __launch_bounds__(kB64) k_rowpart64(const double* __restrict__ th, int N, int mag,
                                                    unsigned long long* __restrict__ Qp, uint32_t* __restrict__ Pw,
                                                    uint32_t* __restrict__ Nw, unsigned long long* __restrict__ thmax) {
    __shared__ __int128 sq[kB64 / 32];
    __shared__ double sm[kB64 / 32];
    const int vr = blockIdx.y, j = blockIdx.x * kB64 + threadIdx.x, lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int NW = N >> 5, nb = gridDim.x;
    const double x = j < N ? th[(size_t)vr * N + j] : 0.0;
    __int128 q = j < N ? round64_q(mag ? fabs(x) : x) : 0;
    double mx = fabs(x);
    const uint32_t pw = __ballot_sync(0xffffffffu, x > 0.0), nw = __ballot_sync(0xffffffffu, x < 0.0);
    if (lane == 0 && j < N) { Pw[(size_t)vr * NW + (j >> 5)] = pw; Nw[(size_t)vr * NW + (j >> 5)] = nw; }
    q = warp_sum128(q);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) { sq[wp] = q; sm[wp] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        __int128 t = 0;
        double m2 = 0.0;
        for (int i = 0; i < kB64 / 32; ++i) { t += sq[i]; m2 = fmax(m2, sm[i]); }
        Qp[((size_t)vr * nb + blockIdx.x) * 2] = (unsigned long long)t;
        Qp[((size_t)vr * nb + blockIdx.x) * 2 + 1] = (unsigned long long)(t >> 64);
        atomicMax(thmax, (unsigned long long)__double_as_longlong(m2));
    }
}

// Row statistics + bit planes of the state whose partials k_rowpart64 / k_adam64 wrote.
__global__ void k_rows64(StepArgs a, const uint32_t* __restrict__ Acur, uint32_t* __restrict__ Aout,
                         const StepScalars* __restrict__ sc, int nb) {
    const int vr = blockIdx.x * blockDim.x + threadIdx.x;
    if (vr >= a.V) return;
    const int NW = a.N >> 5;
    __int128 Q = 0;
    for (int b = 0; b < nb; ++b)
        Q += ((__int128)(long long)a.Qp64[((size_t)vr * nb + b) * 2 + 1] << 64) |
             (__int128)a.Qp64[((size_t)vr * nb + b) * 2];
    const long long hi = (long long)(Q >> 64);
    const unsigned long long lo = (unsigned long long)Q;
    double d, rho;
    unsigned char g;
    row_finish64(hi, lo, a.mc, &d, &rho, &g);
    a.rowQ[vr] = hi;
    a.rowD[vr] = d;
    a.rowRho[vr] = rho;
    a.rowGuard[vr] = g;
    const bool dpos = !a.mc.normalize || Q >= 0;
    const uint32_t* src = dpos ? a.Pw64 : a.Nw64;
    for (int w = 0; w < NW; ++w) Aout[(size_t)vr * NW + w] = src[(size_t)vr * NW + w];
    a.J64[vr] = 0;
    if (sc) {                                              // step: the first model's bits (A22), W = 1
        const long long t = sc->t;
        const unsigned long long bk = a.ds->best_key;
        if ((bk >> 32) == 0ull && (a.ds->sol_step < 0 || a.ds->sol_step == t)) {
            const long long idx = (long long)(bk & 0xffffffffull);
            if (idx >= 0 && idx < a.N)
                a.sol[vr] = (unsigned char)((Acur[(size_t)vr * NW + (idx >> 5)] >> (idx & 31)) & 1u);
        }
    }
}

// (a7) + (a8) partial: G_vn over the row's occurrence records and the J_v partial.
__global__ void __launch_bounds__(kB64) k_fold64(StepArgs a, const uint32_t* __restrict__ Acur,
                                                 const StepScalars* __restrict__ sc) {
    __shared__ long long sj[kB64 / 32];
    const int vr = blockIdx.y, j = blockIdx.x * kB64 + threadIdx.x, lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int N = a.N, NW = N >> 5, K = a.mc.K;
    const long long t = sc->t;
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) a.ds->thmax64_bits[(t + 1) & 1] = 0ull;
    long long I = 0;
    if (j < N) {
        const uint32_t own = (Acur[(size_t)vr * NW + (j >> 5)] >> (j & 31)) & 1u;
        int cnt[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) cnt[r] = 0;
        for (unsigned p = a.occ_ptr[vr]; p < a.occ_ptr[vr + 1];) {
            const uint32_t hdr = a.occ_rec[p], len = hdr >> 1;
            uint32_t R = own ^ (hdr & 1u);
            for (uint32_t q = 1; q < len; ++q) {
                const uint32_t code = a.occ_rec[p + q];
                R += ((Acur[(size_t)(code >> 1) * NW + (j >> 5)] >> (j & 31)) & 1u) ^ (code & 1u);
            }
            const int delta = (hdr & 1u) ? 1 : -1;                // cneg - cpos
#pragma unroll
            for (int r = 0; r < 16; ++r) cnt[r] += (R == (uint32_t)r) ? delta : 0;
            p += len;
        }
        double G = 0.0;                                             // R30: fp64 FMA chain, r ascending
#pragma unroll
        for (int r = 0; r < 16; ++r)
            if (r <= K) G = __fma_rn((double)cnt[r], a.gt64[(size_t)r * N + j], G);
        a.G64[(size_t)vr * N + j] = G;
        // J_v fixed point (R13 at fp64): s = 61 - ceil(log2(N occ gmax thmax)) in [-1022, 1023]
        const int2 pn = a.occ_pn[vr];
        const int occ = pn.x + pn.y;
        const double gmax = __longlong_as_double((long long)a.ds->gmax_bits);
        const double thmax = __longlong_as_double((long long)a.ds->thmax64_bits[t & 1]);
        double x = __dmul_rn((double)a.mc.Nnorm, (double)occ);
        x = __dmul_rn(x, gmax);
        x = __dmul_rn(x, thmax);
        if (occ > 0 && x > 0.0) {
            int s = 61 - ceil_log2_64(x);
            s = s > 1023 ? 1023 : (s < -1022 ? -1022 : s);
            const double p2 = __longlong_as_double((long long)(1023 + s) << 52);
            I = __double2ll_rn(__dmul_rn(G, __dmul_rn(a.th64[(size_t)vr * N + j], p2)));
        }
    }
    I = warp_sum(I);
    if (lane == 0) sj[wp] = I;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long tot = 0;
        for (int i = 0; i < kB64 / 32; ++i) tot += sj[i];
        atomicAdd(reinterpret_cast<unsigned long long*>(&a.J64[vr]), (unsigned long long)tot);
    }
}

// (a8) + (a9): gradient, fp64 AdamW, next state's row-sum partials and sign words.
__global__ void __launch_bounds__(kB64) k_adam64(StepArgs a, const StepScalars* __restrict__ sc) {
    __shared__ __int128 sq[kB64 / 32];
    __shared__ double sm[kB64 / 32];
    const int vr = blockIdx.y, j = blockIdx.x * kB64 + threadIdx.x, lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const int N = a.N, NW = N >> 5, nb = gridDim.x;
    const long long t = sc->t;
    const MethodConsts& mc = a.mc;
    const bool mag = mc.normalize == 3;
    // c_v = ((J/N) rho) rho from the exact J (0 when the guard is active or normalisation is off)
    const double rho = a.rowRho[vr];
    double c = 0.0;
    if (mc.normalize && !a.rowGuard[vr]) {
        const int2 pn = a.occ_pn[vr];
        const int occ = pn.x + pn.y;
        const double gmax = __longlong_as_double((long long)a.ds->gmax_bits);
        const double thmax = __longlong_as_double((long long)a.ds->thmax64_bits[t & 1]);
        double x = __dmul_rn((double)mc.Nnorm, (double)occ);
        x = __dmul_rn(x, gmax);
        x = __dmul_rn(x, thmax);
        double J = 0.0;
        if (occ > 0 && x > 0.0) {
            int s = 61 - ceil_log2_64(x);
            s = s > 1023 ? 1023 : (s < -1022 ? -1022 : s);
            J = scalbn((double)a.J64[vr], -s);
        }
        c = J / (double)mc.Nnorm;
        c = c * rho;
        c = c * rho;
    }
    double xn = 0.0;
    if (j < N) {
        const size_t i = (size_t)vr * N + j;
        const double th = a.th64[i];
        const double cc = mag ? (th > 0.0 ? c : (th < 0.0 ? -c : 0.0)) : c;
        const double g = __fma_rn(a.G64[i], rho, -cc);
        double x = __dmul_rn(th, sc->wdf64);
        const double mm0 = __dmul_rn(a.m64[i], (double)sc->mkeep);
        const double mm = __fma_rn(sc->a1_64, __dsub_rn(g, mm0), mm0);
        const double vb = __dmul_rn(a.v64[i], sc->b2_64);
        const double vn = __fma_rn(__dmul_rn(sc->a2_64, g), g, vb);
        const double den = __dadd_rn(__dmul_rn(__dsqrt_rn(vn), sc->rbc2_64), sc->eps64);
        x = __dadd_rn(x, __ddiv_rn(__dmul_rn(sc->nss64, mm), den));
        if (mc.noise) {
            const long long n = mc.n0 + j;
            uint32_t xr[4] = {(uint32_t)(n >> 2), (uint32_t)vr, (uint32_t)(1 + t), 0u};
            philox4x32_10(xr, (uint32_t)mc.seed, (uint32_t)(mc.seed >> 32));
            const double xi = (double)(xr[n & 3] >> 8) * 5.9604644775390625e-08 - 0.5;
            x = __dadd_rn(x, __dmul_rn(sc->nz64, xi));
        }
        a.th64[i] = x;
        a.m64[i] = mm;
        a.v64[i] = vn;
        xn = x;
    }
    __int128 q = j < N ? round64_q(mag ? fabs(xn) : xn) : 0;
    double mx = fabs(xn);
    const uint32_t pw = __ballot_sync(0xffffffffu, xn > 0.0), nw = __ballot_sync(0xffffffffu, xn < 0.0);
    if (lane == 0 && j < N) { a.Pw64[(size_t)vr * NW + (j >> 5)] = pw; a.Nw64[(size_t)vr * NW + (j >> 5)] = nw; }
    q = warp_sum128(q);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) { sq[wp] = q; sm[wp] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        __int128 tq = 0;
        double m2 = 0.0;
        for (int k = 0; k < kB64 / 32; ++k) { tq += sq[k]; m2 = fmax(m2, sm[k]); }
        a.Qp64[((size_t)vr * nb + blockIdx.x) * 2] = (unsigned long long)tq;
        a.Qp64[((size_t)vr * nb + blockIdx.x) * 2 + 1] = (unsigned long long)(tq >> 64);
        atomicMax(&a.ds->thmax64_bits[(t + 1) & 1], (unsigned long long)__double_as_longlong(m2));
    }
}

__global__ void k_absG64(const double* __restrict__ G, int V, int N, const int* __restrict__ cols, int M,
                         double* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)M * V) return;
    const int mi = (int)(i / V), v = (int)(i % V);
    out[i] = fabs(G[(size_t)v * N + cols[mi]]);
}

cudaError_t launch_init64(const StepArgs& a, unsigned long long seed, cudaStream_t st) {
    if (a.V == 0) return cudaGetLastError();
    k_init64<<<dim3((unsigned)((a.N + 255) / 256), (unsigned)a.V), 256, 0, st>>>(a.th64, a.m64, a.v64, a.V, a.N,
                                                                                  a.mc.n0, seed);
    return cudaGetLastError();
}

cudaError_t launch_rowstats64(const StepArgs& a, long long t, cudaStream_t st) {
    if (a.V == 0) return cudaGetLastError();
    const int nb = fp64_blocks_per_row(a.N);
    uint32_t* A = (t & 1) ? a.A1 : a.A0;
    k_rowpart64<<<dim3((unsigned)nb, (unsigned)a.V), kB64, 0, st>>>(a.th64, a.N, a.mc.normalize == 3 ? 1 : 0, a.Qp64,
                                                                     a.Pw64, a.Nw64, &a.ds->thmax64_bits[t & 1]);
    k_rows64<<<(a.V + 127) / 128, 128, 0, st>>>(a, A, A, nullptr, nb);
    return cudaGetLastError();
}

cudaError_t launch_update64(const StepArgs& a, const uint32_t* Acur, uint32_t* Anext, const StepScalars* sc,
                            cudaStream_t st) {
    if (a.V == 0) return cudaGetLastError();
    const int nb = fp64_blocks_per_row(a.N);
    const dim3 g((unsigned)nb, (unsigned)a.V);
    k_fold64<<<g, kB64, 0, st>>>(a, Acur, sc);
    k_adam64<<<g, kB64, 0, st>>>(a, sc);
    k_rows64<<<(a.V + 127) / 128, 128, 0, st>>>(a, Acur, Anext, sc, nb);
    return cudaGetLastError();
}

cudaError_t launch_absG64(const StepArgs& a, const int* cols_dev, int M, double* absG, cudaStream_t st) {
    const long long total = (long long)M * a.V;
    if (total > 0) k_absG64<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(a.G64, a.V, a.N, cols_dev, M, absG);
    return cudaGetLastError();
}

}  // namespace tsat
