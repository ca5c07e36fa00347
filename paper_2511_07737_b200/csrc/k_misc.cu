// k_misc.cu - init (a1), row statistics (a2/a3), SmoothMin table (a6),
// end-of-iteration bookkeeping and the export kernels (a10/a11).
//
// Compiled with -fmad=false: every floating operation is a separate IEEE
// round-to-nearest op unless written as an explicit fma.
#include "device_common.cuh"
#include "peer.cuh"

namespace tsat {

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
        s += __float2ll_rn((mc.normalize == 3 ? fabsf(x) : x) * 4294967296.0f);   // x 2^32 is exact in fp32
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

// ------------------------------------------------------------------ (a6) SmoothMin / g table
// Per candidate: h[0..K] (top bin KB-1 derived as C - sum), rmin, Eq. 4 via
// the E table, g[r] = (E[r-rmin]/den)(1 - tau(r - S)) rounded to fp32 (R26)
// into the bin-major table gtab[r][n]; unsat; best key; gmax over |g32|.
// Clears the histogram for the next iteration.
// W = 1: the last block to finish also closes the iteration's bookkeeping
// (what a separate end-of-step kernel did): the loss -sum_n S_n from the
// per-block sums in block order (deterministic), the step info, and the first
// model's iteration / index (its bits are kept by k_update, A22).
template <int KB>
__global__ void __launch_bounds__(256) k_gtable(int* __restrict__ hist, int N, long long C, MethodConsts mc,
                                                float* __restrict__ gtab, double* __restrict__ S,
                                                int* __restrict__ unsat, DevScalars* __restrict__ ds, int sharded,
                                                double* __restrict__ lossp, const StepScalars* __restrict__ sc,
                                                int peer, const PeerArgs px, double* __restrict__ gt64) {
    __shared__ double shS[8];
    __shared__ bool last;
    pdl_wait();
    pdl_trigger();
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    unsigned long long key = ~0ull;
    double gm = 0.0;
    long long lfx = 0;               // sharded loss: S_n 2^e, exact int64 sum across ranks (mc.loss_scale)
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
        int rmin = KB;
#pragma unroll
        for (int r = KB - 1; r >= 0; --r)
            if (r <= K && h[r] != 0) rmin = r;
        float g[KB];
        double gd[KB];                       // fp64 state (R30): the table before rounding
#pragma unroll
        for (int r = 0; r < KB; ++r) { g[r] = 0.0f; gd[r] = 0.0; }
        double s = 0.0;
        if (rmin <= K) {
            double den = 0.0, num = 0.0;
#pragma unroll
            for (int r = 0; r < KB; ++r) {
                if (r >= rmin && r <= K) {
                    double e = sc->E[r - rmin];
                    den = den + (double)h[r] * e;
                    num = num + (double)((long long)r * h[r]) * e;
                }
            }
            s = num / den;
#pragma unroll
            for (int r = 0; r < KB; ++r) {
                if (r >= rmin && r <= K) {
                    double wgt = sc->E[r - rmin] / den;
                    double u = (double)r - s;
                    gd[r] = wgt * (1.0 - sc->tau * u);
                    g[r] = (float)gd[r];
                    gm = fmax(gm, gt64 ? fabs(gd[r]) : fabs((double)g[r]));
                }
            }
        }
#pragma unroll
        for (int r = 0; r < KB; ++r) gtab[(size_t)r * N + n] = g[r];
        if (gt64) {
#pragma unroll
            for (int r = 0; r < KB; ++r) gt64[(size_t)r * N + n] = gd[r];
        }
        S[n] = s;
        lfx = __double2ll_rn(s * mc.loss_scale);
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
    const bool fx = sharded || peer;            // exact fixed-point loss, summed across ranks
    if (fx) lfx = warp_sum(lfx);
    if (lane == 0) {
        atomicMin(&ds->best_key, key);
        atomicMax(&ds->gmax_bits, gb);
        if (fx) atomicAdd(reinterpret_cast<unsigned long long*>(&ds->loss_fx), (unsigned long long)lfx);
    }
    if (sharded) return;                       // the sharded step ends in k_step_end_sharded
    if (peer) {
        // peer path: the last block publishes this rank's (best key, gmax,
        // max|theta_t|, loss) to every rank; k_update combines them
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            last = atomicAdd(&ds->gt_done, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (last && threadIdx.x == 0) {
            __threadfence();
            const long long t = sc->t;
            const unsigned long long x[4] = {~*((volatile unsigned long long*)&ds->best_key),
                                             *((volatile unsigned long long*)&ds->gmax_bits),
                                             (unsigned long long)*((volatile unsigned int*)&ds->thmax_bits[t & 1]),
                                             (unsigned long long)*((volatile long long*)&ds->loss_fx)};
            ds->gt_done = 0u;
            peer_send_scalars(px, x, sc->xgen);
        }
        return;
    }
    // block sum of S in a fixed order (warp trees, then warps ascending)
    double sv = n < N ? S[n] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sv = sv + __shfl_xor_sync(0xffffffffu, sv, o);
    if (lane == 0) shS[threadIdx.x >> 5] = sv;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) b = b + shS[i];
        lossp[blockIdx.x] = b;
        __threadfence();
        last = atomicAdd(&ds->gt_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        double tot = 0.0;
        for (unsigned i = 0; i < gridDim.x; ++i) tot = tot + *((volatile double*)lossp + i);
        const long long t = sc->t;
        const unsigned long long bk = *((volatile unsigned long long*)&ds->best_key);
        const int bu = (int)(bk >> 32);
        const long long bi = (long long)(bk & 0xffffffffull);
        if (bu == 0 && ds->sol_step < 0) { ds->sol_step = t; ds->sol_idx = bi; }
        ds->loss = -tot;
        ds->info_t = t + 1;
        ds->info_best_unsat = bu;
        ds->info_best_idx = bi;
        ds->info_loss = -tot;
        ds->gt_done = 0u;
    }
}

// ------------------------------------------------------------------ export helpers
// Variable gradient |G_vn| (pre-Jacobian, R14) of the last evaluated state for
// a list of candidates: out[m * V + v] as fp64.  One thread per (column, v).
template <int KB>
__global__ void __launch_bounds__(256) k_grad_cols(int V, int N, const uint32_t* __restrict__ Acur,
                                                   const uint32_t* __restrict__ occ_ptr, const uint32_t* __restrict__ occ_rec,
                                                   const float* __restrict__ gtab, const int* __restrict__ cols, int M,
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
    float G = 0.0f;                                               // R27: fp32 FMA chain
#pragma unroll
    for (int r = 0; r < KB; ++r)
        if (r <= K) G = __fmaf_rn((float)cnt[r], gtab[(size_t)r * N + n], G);
    out[(size_t)mi * V + v] = fabs((double)G);
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
                int sh = 64 - 8 * pass;
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

// Export entries of the owned selected columns: entry (pos[i], j) of the
// M x k table = (|G| fp32 bits << 32) | (v << 1) | b_vn, with b_vn read from
// the evaluated state's bit plane (only the M columns' bits leave the GPU).
__global__ void k_export_pack(const uint32_t* __restrict__ Aeval, int NW, const int* __restrict__ cols,
                              const int* __restrict__ pos, int Mo, int k, const int* __restrict__ out_v,
                              const double* __restrict__ out_g, unsigned long long* __restrict__ entries) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)Mo * k) return;
    const int mi = (int)(i / k), j = (int)(i % k);
    const int n = cols[mi], v = out_v[i];
    const uint32_t b = (Aeval[(size_t)v * NW + (n >> 5)] >> (n & 31)) & 1u;
    const float g = (float)out_g[i];                     // |G| is an fp32 value (R27): exact
    entries[(size_t)pos[mi] * k + j] = ((unsigned long long)__float_as_uint(g) << 32) | ((unsigned long long)v << 1) | b;
}

// ------------------------------------------------------------------ launchers
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

cudaError_t launch_gtable(const StepArgs& a, const StepScalars* sc, cudaStream_t st) {
    int blocks = (a.N + 255) / 256;
    if (a.KB == 4)
        return launch_maybe_pdl(a.pdl, k_gtable<4>, dim3(blocks), dim3(256), 0, st, a.hist, a.N, a.C, a.mc, a.gtab, a.S,
                                a.unsat, a.ds, a.sharded, a.lossp, sc, a.peer, a.px, a.fp64 ? a.gt64 : nullptr);
    if (a.KB == 8)
        return launch_maybe_pdl(a.pdl, k_gtable<8>, dim3(blocks), dim3(256), 0, st, a.hist, a.N, a.C, a.mc, a.gtab, a.S,
                                a.unsat, a.ds, a.sharded, a.lossp, sc, a.peer, a.px, a.fp64 ? a.gt64 : nullptr);
    return launch_maybe_pdl(a.pdl, k_gtable<16>, dim3(blocks), dim3(256), 0, st, a.hist, a.N, a.C, a.mc, a.gtab, a.S,
                            a.unsat, a.ds, a.sharded, a.lossp, sc, a.peer, a.px, a.fp64 ? a.gt64 : nullptr);
}

cudaError_t launch_export_pack(const StepArgs& a, long long t_eval, const int* cols_dev, const int* pos_dev, int Mo,
                               int k, const int* out_v, const double* out_g, unsigned long long* entries,
                               cudaStream_t st) {
    const uint32_t* Aeval = (t_eval & 1) ? a.A1 : a.A0;
    const long long total = (long long)Mo * k;
    if (total > 0)
        k_export_pack<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(Aeval, a.N >> 5, cols_dev, pos_dev, Mo, k, out_v,
                                                                       out_g, entries);
    return cudaGetLastError();
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
        if (a.fp64) launch_absG64(a, cols_dev, M, absG, st);                  // |G| of the evaluated state (R30)
        else if (a.KB == 4) k_grad_cols<4><<<blocks, 256, 0, st>>>(a.V, a.N, Aeval, a.occ_ptr, a.occ_rec, a.gtab, cols_dev, M, a.mc.K, absG);
        else if (a.KB == 8) k_grad_cols<8><<<blocks, 256, 0, st>>>(a.V, a.N, Aeval, a.occ_ptr, a.occ_rec, a.gtab, cols_dev, M, a.mc.K, absG);
        else k_grad_cols<16><<<blocks, 256, 0, st>>>(a.V, a.N, Aeval, a.occ_ptr, a.occ_rec, a.gtab, cols_dev, M, a.mc.K, absG);
        k_topk_cols<<<M, 1024, 0, st>>>(absG, a.V, k, out_v, out_g);
    }
    return cudaGetLastError();
}

}  // namespace tsat
