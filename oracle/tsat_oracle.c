/*
 * tsat_oracle.c - TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU oracle of TurboSAT's batched
 * differentiable SAT step (arXiv 2511.07737, /root/reference/PAPER.md), used
 * to prove the CUDA path (paper_2511_07737_b200/) correct.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  It shares NO code with the CUDA path (no headers, helpers or
 * tables); the only common inputs come from tsat_synth/ (seeded instances).
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared -o liboracle.so tsat_oracle.c -lm
 * (-ffp-contract=off: every floating operation below is a separate IEEE
 *  round-to-nearest op; fused multiply-adds appear only as explicit fmaf()).
 * OpenMP mode (SURVEY §8(c) "Form"): the same source built with -fopenmp
 * (liboracle_omp.so).  The `#pragma omp` lines split only loops whose
 * iterations write disjoint outputs (rows v, clauses c, candidates j); the
 * histograms are integer counts summed from per-thread copies.  No value
 * depends on the thread count (tests/test_oracle_pins2.py checks the two
 * builds bit for bit); without -fopenmp the pragmas are ignored.
 *
 * Notation follows the paper: V variables, C clauses, N candidate
 * assignments; theta = A_real (one parameter per variable and candidate,
 * DESIGN.md reading R2); R = P A (Eq. 1); B = clip(sign, 0, 1) (Eq. 2);
 * L = -sum S_i (Eq. 3); S_i = SmoothMin (Eq. 4); Eq. 5 per-variable
 * normalisation; AdamW + step-decay LR with restarts (§4.1).
 * Array layouts: theta/m/v/G/b are [V][N] row-major (candidate fastest);
 * R is [C][N]; h and g are [N][K+1].
 *
 * Where the paper is silent the readings are DESIGN.md §"Readings" R1..R28.
 * Parity pins (tests/, all -m "not gpu"), one per function:
 *   or_philox4x32_10   Random123 KAT vectors              test_oracle_pins
 *   or_init            N(0,1) statistics, KS, shard slices test_oracle_pins
 *   or_row_sums(_abs), or_row_finish, or_binarize, or_clause_eval, or_histogram
 *                      Fig. 2 values, brute-force enumeration (V <= 20),
 *                      double-counting invariants          test_oracle_pins
 *   or_smoothmin(_direct) 40-digit mpmath of Eq. 4 and its derivative
 *   or_backward, or_jacobian_*, or_grad(_mag), or_gmax, or_abs_max
 *                      fp64 torch autograd of the dense graph, element by
 *                      element at 1e-5 rel (+ operand floor); Euler
 *                      invariant; fsum                     test_oracle_pins(2)
 *   or_lr_at           schedule values (R9)
 *   or_adamw           torch.optim.AdamW fp32 (m, v bit-exact) and fp64
 *                      (element-wise 1e-5 rel); noise xi distribution (R17)
 *   or_hist_stream, or_backward_rows (and oracle.step_sampled)
 *                      bit-exact against or_histogram / or_backward /
 *                      Oracle.step                         test_oracle_pins2
 * "parity unpinned": none of the functions; only trajectory QUALITY
 * (steps-to-SAT) is unpinned (the paper prints no value).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11).  Counter-based RNG  */
/* used for (a1) init (§4.1 l.250: "random values from the      */
/* standard normal distribution") and the optional noise hook (R17).     */
/* ------------------------------------------------------------------ */
void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* (a1) Init, §4.1 l.250-252.  theta_vn ~ N(0,1): Philox keyed by
 * seed, counter (n>>2, v, 0, 0) over the GLOBAL candidate index n, then
 * Box-Muller on the pairs (x0,x1), (x2,x3): u1 = (x+1) 2^-32 in (0,1],
 * u2 = x 2^-32, z = sqrt(-2 ln u1) {cos,sin}(2 pi u2) in fp64 -> fp32.
 * m = v = 0.  Candidates [n0, n0+Nl) are produced (a shard). */
void or_init(int V, int64_t n0, int Nl, uint64_t seed, float* theta, float* m, float* vv)
{
    const double two_pi = 6.283185307179586;
    const double two_m32 = 2.3283064365386963e-10; /* 2^-32 */
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    #pragma omp parallel for schedule(static)
    for (int v = 0; v < V; ++v) {
        for (int j = 0; j < Nl; ++j) {
            int64_t n = n0 + j;
            uint32_t ctr[4] = {(uint32_t)(n >> 2), (uint32_t)v, 0u, 0u};
            uint32_t x[4];
            or_philox4x32_10(ctr, key, x);
            int q = (int)(n & 3);
            int pair = q >> 1;
            double u1 = ((double)x[2 * pair] + 1.0) * two_m32;
            double u2 = (double)x[2 * pair + 1] * two_m32;
            double r = sqrt(-2.0 * log(u1));
            double a = two_pi * u2;
            double z = (q & 1) ? r * sin(a) : r * cos(a);
            theta[(size_t)v * Nl + j] = (float)z;
            m[(size_t)v * Nl + j] = 0.0f;
            vv[(size_t)v * Nl + j] = 0.0f;
        }
    }
}

/* ------------------------------------------------------------------ */
/* (a2) Eq. 5 row statistics (§4.1 l.262-269).                   */
/* The row mean is taken over ALL N candidates (R20).  The sum is exact: */
/* Q_v = sum_n round_half_even(theta_vn 2^32) in int64 (R10), so any     */
/* partition of the candidates gives the same Q_v.                       */
/* ------------------------------------------------------------------ */
int or_row_sums(int V, int Nl, const float* theta, int64_t* Q)
{
    #pragma omp parallel for schedule(static)
    for (int v = 0; v < V; ++v) {
        int64_t s = 0;
        for (int j = 0; j < Nl; ++j) {
            double x = (double)theta[(size_t)v * Nl + j] * 4294967296.0; /* exact */
            s += (int64_t)llrint(x);
        }
        Q[v] = s;
    }
    return 0;
}

/* normalize == 3 (variant f2, reading R28): Eq. 5's denominator is the mean
 * MAGNITUDE of the row, mean_n |theta_vn|, so Q_v = sum_n round(|theta| 2^32)
 * (same exact fixed point, Q_v >= 0). */
int or_row_sums_abs(int V, int Nl, const float* theta, int64_t* Q)
{
    #pragma omp parallel for schedule(static)
    for (int v = 0; v < V; ++v) {
        int64_t s = 0;
        for (int j = 0; j < Nl; ++j) {
            double x = fabs((double)theta[(size_t)v * Nl + j]) * 4294967296.0; /* exact */
            s += (int64_t)llrint(x);
        }
        Q[v] = s;
    }
    return 0;
}

/* mu_v = (Q_v 2^-32)/N; d_v = sign(mu_v) max(|mu_v|, eps), sign(0)=+1;
 * rho_v = 1/d_v (R3: x/mu computed as x * (1/mu)); guard_v = |mu_v| <= eps.
 * normalize == 0 (variant, R20): d = rho = 1, guard = 1. */
void or_row_finish(int V, int64_t N, const int64_t* Q, int normalize, double eps_norm,
                   double* mu, double* d, double* rho, uint8_t* guard)
{
    for (int v = 0; v < V; ++v) {
        if (!normalize) {
            mu[v] = 0.0; d[v] = 1.0; rho[v] = 1.0; guard[v] = 1;
            continue;
        }
        double m_ = ((double)Q[v] * 2.3283064365386963e-10) / (double)N;
        double a = fabs(m_);
        double mag = a > eps_norm ? a : eps_norm;
        mu[v] = m_;
        d[v] = (m_ >= 0.0) ? mag : -mag;
        rho[v] = 1.0 / d[v];
        guard[v] = (a <= eps_norm) ? 1 : 0;
    }
}

/* (a3) Eq. 2, A = B(A_real^norm) = clip(sign(theta/d), 0, 1), evaluated by
 * sign logic (no division): b = (theta>0 && d>0) || (theta<0 && d<0).
 * theta = 0 gives 0 (R5). */
void or_binarize(int V, int Nl, const float* theta, const double* d, uint8_t* b)
{
    #pragma omp parallel for schedule(static)
    for (int v = 0; v < V; ++v)
        for (int j = 0; j < Nl; ++j) {
            float x = theta[(size_t)v * Nl + j];
            b[(size_t)v * Nl + j] = (uint8_t)((x > 0.0f && d[v] > 0.0) || (x < 0.0f && d[v] < 0.0));
        }
}

/* (a4) Eq. 1, R = P A: R_cn = number of literals of clause c that candidate n
 * sets true (§3.1.3 l.161-167).  Positive literal +v takes b_vn, negative -v
 * takes 1 - b_vn (§3.1.2 l.155-158).  Literals are signed 1-based DIMACS. */
void or_clause_eval(int C, const int64_t* cptr, const int32_t* lits, int Nl,
                    const uint8_t* b, uint8_t* R)
{
#pragma omp parallel for schedule(static)
    for (int c = 0; c < C; ++c) {
        uint8_t* row = R + (size_t)c * Nl;
        for (int j = 0; j < Nl; ++j) row[j] = 0;
        for (int64_t l = cptr[c]; l < cptr[c + 1]; ++l) {
            int32_t lit = lits[l];
            int v = (lit > 0 ? lit : -lit) - 1;
            const uint8_t* brow = b + (size_t)v * Nl;
            for (int j = 0; j < Nl; ++j) {
                uint8_t val = lit > 0 ? brow[j] : (uint8_t)(1 - brow[j]);
                row[j] = (uint8_t)(row[j] + val);
            }
        }
    }
}

/* (a5) §3.1.4: per candidate the number of clauses with R_cn = r, r=0..K.
 * unsat_n = h_n[0]; the hard S_n (column minimum) is the least r with h>0. */
void or_histogram(int C, int Nl, int K, const uint8_t* R, int32_t* h)
{
    for (int j = 0; j < Nl * (K + 1); ++j) h[j] = 0;
#pragma omp parallel
    {
        int32_t* hl = h;
#ifdef _OPENMP
        hl = (int32_t*)calloc((size_t)Nl * (K + 1), sizeof(int32_t));   /* this thread's counts */
#endif
#pragma omp for schedule(static)
        for (int c = 0; c < C; ++c)
            for (int j = 0; j < Nl; ++j) hl[(size_t)j * (K + 1) + R[(size_t)c * Nl + j]] += 1;
#ifdef _OPENMP
#pragma omp critical
        for (int j = 0; j < Nl * (K + 1); ++j) h[j] += hl[j];
        free(hl);
#endif
    }
}

/* (a6) Eq. 4 SmoothMin and its derivative, per candidate.
 * R takes only the integer values 0..K, so the C-term sums of Eq. 4 group
 * exactly into K+1 terms (R11): with E[d] = exp(-tau d) (host libm) and the
 * max-shift by rmin,
 *   den = sum_{r>=rmin} h_r E[r-rmin],  num = sum_{r>=rmin} (r h_r) E[r-rmin],
 *   S = num/den,
 *   dS/dR at value r: g[r] = (E[r-rmin]/den) (1 - tau (r - S))  (r >= rmin).
 * (The derivative of sum R w / sum w with w = e^{-tau R}.)  Sums ascending r.
 * Returns via S[n], g[n*(K+1)+r], rmin[n]. */
void or_smoothmin(int Nl, int K, const int32_t* h, const double* E, double tau,
                  double* S, double* g, int32_t* rmin_out)
{
#pragma omp parallel for schedule(static)
    for (int j = 0; j < Nl; ++j) {
        const int32_t* hn = h + (size_t)j * (K + 1);
        double* gn = g + (size_t)j * (K + 1);
        int rmin = 0;
        while (rmin <= K && hn[rmin] == 0) ++rmin;
        for (int r = 0; r <= K; ++r) gn[r] = 0.0;
        if (rmin > K) { /* C == 0: no clauses, nothing to minimise */
            S[j] = 0.0; rmin_out[j] = 0;
            continue;
        }
        double den = 0.0, num = 0.0;
        for (int r = rmin; r <= K; ++r) {
            den = den + (double)hn[r] * E[r - rmin];
            num = num + (double)((int64_t)r * (int64_t)hn[r]) * E[r - rmin];
        }
        double s = num / den;
        for (int r = rmin; r <= K; ++r) {
            double w = E[r - rmin] / den;
            double u = (double)r - s;
            gn[r] = w * (1.0 - tau * u);
        }
        S[j] = s;
        rmin_out[j] = rmin;
    }
}

/* Eq. 4 written out over the C entries of one column (pin helper): shift by
 * the column minimum, sum in clause order. */
double or_smoothmin_direct(int C, const int32_t* Rcol, double tau)
{
    int mn = Rcol[0];
    for (int c = 1; c < C; ++c) if (Rcol[c] < mn) mn = Rcol[c];
    double den = 0.0, num = 0.0;
    for (int c = 0; c < C; ++c) {
        double w = exp(-tau * (double)(Rcol[c] - mn));
        den += w;
        num += (double)Rcol[c] * w;
    }
    return num / den;
}

/* (a7) Backward through R = P A and the STE (§3.2 l.189-191, l.226):
 * dL/dR_cn = -g_n[R_cn]; dL/dA = P^T dL/dR; the binariser is the identity in
 * the backward pass (STE), and since A_neg = 1 - A_pos (R2) the variable
 * gradient folds as dL/dA_pos - dL/dA_neg:
 *   G_vn = sum_{c contains -v} g_n[R_cn] - sum_{c contains +v} g_n[R_cn].
 * Equal terms are grouped by value (exact integer counts, R12):
 *   G_vn = sum_r (cneg_vn[r] - cpos_vn[r]) g_n[r], ascending r,
 * with g the fp32 table (R26: g rounded once to fp32, the paper's tensor
 * precision) accumulated in fp32 by fused multiply-adds, r ascending (R27).
 * G is returned in a double array (exact fp32 values).
 * occ lists (variable -> (clause, sign)) are built here from the CNF. */
void or_backward(int V, int C, const int64_t* cptr, const int32_t* lits, int Nl, int K,
                 const uint8_t* R, const float* g, double* G)
{
    /* transpose: count occurrences per variable */
    int64_t* vptr = (int64_t*)calloc((size_t)V + 1, sizeof(int64_t));
    int64_t nnz = cptr[C];
    int32_t* occ_c = (int32_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
    int8_t* occ_s = (int8_t*)malloc((size_t)(nnz > 0 ? nnz : 1));
    for (int64_t l = 0; l < nnz; ++l) vptr[(lits[l] > 0 ? lits[l] : -lits[l])]++;
    for (int v = 0; v < V; ++v) vptr[v + 1] += vptr[v];
    int64_t* fill = (int64_t*)malloc(((size_t)V + 1) * sizeof(int64_t));
    memcpy(fill, vptr, ((size_t)V + 1) * sizeof(int64_t));
    for (int c = 0; c < C; ++c)
        for (int64_t l = cptr[c]; l < cptr[c + 1]; ++l) {
            int v = (lits[l] > 0 ? lits[l] : -lits[l]) - 1;
            occ_c[fill[v]] = c;
            occ_s[fill[v]] = lits[l] > 0 ? 1 : -1;
            fill[v]++;
        }
#pragma omp parallel
    {
    int32_t* cnt = (int32_t*)malloc((size_t)Nl * (K + 1) * sizeof(int32_t));
#pragma omp for schedule(dynamic, 16)
    for (int v = 0; v < V; ++v) {
        memset(cnt, 0, (size_t)Nl * (K + 1) * sizeof(int32_t));
        for (int64_t o = vptr[v]; o < vptr[v + 1]; ++o) {
            const uint8_t* Rrow = R + (size_t)occ_c[o] * Nl;
            int delta = occ_s[o] < 0 ? +1 : -1;  /* cneg - cpos */
            for (int j = 0; j < Nl; ++j) cnt[(size_t)j * (K + 1) + Rrow[j]] += delta;
        }
        for (int j = 0; j < Nl; ++j) {
            float acc = 0.0f;
            for (int r = 0; r <= K; ++r)
                acc = fmaf((float)cnt[(size_t)j * (K + 1) + r], g[(size_t)j * (K + 1) + r], acc);
            G[(size_t)v * Nl + j] = (double)acc;
        }
    }
    free(cnt);
    }
    free(fill); free(occ_s); free(occ_c); free(vptr);
}

/* ceil(log2(x)) for finite x > 0, exactly (frexp: x = f 2^e, f in [0.5,1)). */
static int ceil_log2(double x)
{
    int e;
    double f = frexp(x, &e);
    return (f == 0.5) ? e - 1 : e;
}

/* (a8) Eq. 5 Jacobian (l.269 "fully differentiable").  With x = theta/mu
 * (mu the row mean over all N), dL/dtheta_vn = G_vn/d_v - J_v/(N d_v^2),
 * J_v = sum_m G_vm theta_vm.  J_v is summed in int64 fixed point (R13):
 * s_v = 61 - ceil(log2(N occ_v gmax thmax)) (a global bound on |sum|),
 * clamped to [-126, 127] so 2^s_v is an fp32; each term is the fp32 product
 * p = G * (theta * 2^s_v) (the paper's arithmetic is fp32; theta * 2^s_v is
 * exact) rounded to the nearest integer, I_v = sum llrintf(p).  The integer
 * sum makes J_v independent of summation order and of the candidate sharding.
 * This function returns the partial sums I_v over the local candidates and
 * s_v.  occ_v = number of literal occurrences of v; gmax = max |g_n[r]| over
 * all candidates and r in [rmin_n, K]; thmax = max |theta| over the batch.
 * G holds the fp32 variable gradient (R27). */
void or_jacobian_partial(int V, int Nl, const double* G, const float* theta,
                         const int32_t* occ, int64_t N, double gmax, float thmax,
                         int64_t* I, int32_t* s_out, uint8_t* valid)
{
    #pragma omp parallel for schedule(static)
    for (int v = 0; v < V; ++v) {
        double x = (double)N * (double)occ[v];
        x = x * gmax;
        x = x * (double)thmax;
        I[v] = 0; s_out[v] = 0; valid[v] = 0;
        if (occ[v] == 0 || !(x > 0.0)) continue;
        int s = 61 - ceil_log2(x);
        if (s > 127) s = 127;
        if (s < -126) s = -126;
        const float p2 = ldexpf(1.0f, s);
        int64_t acc = 0;
        for (int j = 0; j < Nl; ++j) {
            float ts = theta[(size_t)v * Nl + j] * p2;
            float p = (float)G[(size_t)v * Nl + j] * ts;
            acc += (int64_t)llrintf(p);
        }
        I[v] = acc; s_out[v] = s; valid[v] = 1;
    }
}

/* c_v = ((J_v/N) rho_v) rho_v = J_v / (N d_v^2); zero when the guard is
 * active or normalisation is off (the guard's derivative is 0). */
void or_jacobian_finish(int V, int64_t N, const int64_t* I, const int32_t* s, const uint8_t* valid,
                        const double* rho, const uint8_t* guard, int normalize, double* J, double* cv)
{
    for (int v = 0; v < V; ++v) {
        double j = valid[v] ? ldexp((double)I[v], -s[v]) : 0.0;
        J[v] = j;
        if (!normalize || guard[v]) { cv[v] = 0.0; continue; }
        double t = j / (double)N;
        t = t * rho[v];
        cv[v] = t * rho[v];
    }
}

/* grad_vn = G_vn rho_v - c_v in fp32 (the paper's precision): one fused
 * multiply-add of the fp32 G with the row scalars rounded to fp32 (R27b). */
void or_grad(int V, int Nl, const double* G, const double* rho, const double* cv, float* grad)
{
    #pragma omp parallel for schedule(static)
    for (int v = 0; v < V; ++v) {
        const float rf = (float)rho[v], cf = (float)cv[v];
        for (int j = 0; j < Nl; ++j)
            grad[(size_t)v * Nl + j] = fmaf((float)G[(size_t)v * Nl + j], rf, -cf);
    }
}

/* normalize == 3 (R28): d_v = mean_n |theta_vn|, so d(theta_vm/d_v)/d theta_vn
 * = delta_mn/d_v - theta_vm sign(theta_vn)/(N d_v^2) and
 * grad_vn = G_vn rho_v - sign(theta_vn) c_v, c_v = J_v/(N d_v^2) as above:
 * fmaf(G, (float)rho, -t) with t = (float)c, -(float)c or 0 by the sign of
 * theta_vn (the subgradient of |x| at 0 is taken as 0). */
void or_grad_mag(int V, int Nl, const double* G, const double* rho, const double* cv, const float* theta, float* grad)
{
    #pragma omp parallel for schedule(static)
    for (int v = 0; v < V; ++v) {
        const float rf = (float)rho[v], cf = (float)cv[v];
        for (int j = 0; j < Nl; ++j) {
            const float x = theta[(size_t)v * Nl + j];
            const float t = x > 0.0f ? cf : (x < 0.0f ? -cf : 0.0f);
            grad[(size_t)v * Nl + j] = fmaf((float)G[(size_t)v * Nl + j], rf, -t);
        }
    }
}

/* (a9) LR schedule, §4.1 l.255-259: lr0 = 1e-1, /10 every 30
 * iterations, floor 1e-15, restart to lr0 every 360 iterations (0-based t,
 * R9).  lr = max(lr0 / factor^i, lr_min), i = (t mod restart) div decay;
 * factor^i by repeated multiplication. */
double or_lr_at(int64_t t, double lr0, double factor, int decay_every, int restart_every, double lr_min)
{
    int64_t i = (t % restart_every) / decay_every;
    double p = 1.0;
    for (int64_t k = 0; k < i; ++k) p = p * factor;
    double lr = lr0 / p;
    return lr < lr_min ? lr_min : lr;
}

/* AdamW (§4.1 l.255, "AdamW"; hyper-parameters = PyTorch defaults,
 * R6), in PyTorch's single-tensor order (torch/optim/adam.py:419,457,476,
 * 531-547) with its CPU kernels' rounding (lerp and addcmul use one fused
 * multiply-add; R6b), except that v's bias correction multiplies by
 * the host-rounded 1/sqrt(1 - beta2^s) (R6c: the same AdamW, one division
 * fewer).  s = bstep is the bias-correction step: t + 1, or (t mod restart) + 1
 * when the moments are reset at each LR restart (variant, the caller zeroes
 * m and v at those iterations).
 *   theta *= (float)(1 - lr wd)
 *   m      = fmaf(a1, g - m, m),           a1 = (float)(1 - beta1)
 *   v      = fmaf(a2 g, g, v beta2),       a2 = (float)(1 - beta2)
 *   den    = sqrtf(v) (float)(1/sqrt(1 - beta2^s)) + eps
 *   theta  = theta + ((float)(-lr/(1 - beta1^s)) m)/den
 * Optional noise (R17, default sigma = 0): theta += (float)(lr sigma) xi,
 * xi = (x>>8) 2^-24 - 1/2, x = Philox(key=seed, ctr=(n>>2, v, 1+t, 0))[n&3]. */
void or_adamw(int V, int64_t n0, int Nl, float* theta, float* m, float* vv, const float* grad,
              int64_t t, int64_t bstep, double lr, double beta1, double beta2, double eps, double wd,
              double noise_sigma, uint64_t seed)
{
    double s = (double)bstep;
    float wdf = (float)(1.0 - lr * wd);
    float a1 = (float)(1.0 - beta1);
    float b2f = (float)beta2;
    float a2 = (float)(1.0 - beta2);
    double bc1 = 1.0 - pow(beta1, s);
    double bc2 = 1.0 - pow(beta2, s);
    float nss = (float)(-(lr / bc1));
    float rbc2 = (float)(1.0 / sqrt(bc2));
    float epsf = (float)eps;
    float nz = (float)(lr * noise_sigma);
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
#pragma omp parallel for schedule(static)
    for (int v = 0; v < V; ++v)
        for (int j = 0; j < Nl; ++j) {
            size_t i = (size_t)v * Nl + j;
            float g = grad[i];
            float th = theta[i] * wdf;
            float mm = fmaf(a1, g - m[i], m[i]);
            float vb = vv[i] * b2f;
            float vn = fmaf(a2 * g, g, vb);
            float den = sqrtf(vn) * rbc2 + epsf;
            th = th + (nss * mm) / den;
            if (noise_sigma != 0.0) {
                int64_t n = n0 + j;
                uint32_t ctr[4] = {(uint32_t)(n >> 2), (uint32_t)v, (uint32_t)(1 + t), 0u};
                uint32_t x[4];
                or_philox4x32_10(ctr, key, x);
                float xi = (float)(x[n & 3] >> 8) * 5.9604644775390625e-08f - 0.5f;
                th = th + nz * xi;
            }
            theta[i] = th; m[i] = mm; vv[i] = vn;
        }
}

/* max |theta| (exact). */
float or_abs_max(size_t n, const float* x)
{
    float mx = 0.0f;
    for (size_t i = 0; i < n; ++i) { float a = fabsf(x[i]); if (a > mx) mx = a; }
    return mx;
}

/* gmax = max over candidates and r in [rmin_n, K] of |g_n[r]| (fp32 table). */
double or_gmax(int Nl, int K, const float* g, const int32_t* rmin)
{
    double mx = 0.0;
    for (int j = 0; j < Nl; ++j)
        for (int r = rmin[j]; r <= K; ++r) {
            double a = fabs((double)g[(size_t)j * (K + 1) + r]);
            if (a > mx) mx = a;
        }
    return mx;
}

/* ------------------------------------------------------------------ */
/* Full-size sampled checks (tests/test_gpu_fullsize.py): the same steps as   */
/* above, but the histogram is accumulated clause by clause without storing  */
/* R (C x N bytes), and the backward is evaluated only for listed rows.      */
/* ------------------------------------------------------------------ */

/* §3.1.4 histogram h[n][r] of R = P A (Eq. 1), streaming over clauses. */
void or_hist_stream(int C, const int64_t* cptr, const int32_t* lits, int Nl, int K,
                    const uint8_t* b, int32_t* h, uint8_t* rowbuf)
{
    for (int j = 0; j < Nl * (K + 1); ++j) h[j] = 0;
#pragma omp parallel
    {
    int32_t* hl = h;
    uint8_t* rb = rowbuf;
#ifdef _OPENMP
    hl = (int32_t*)calloc((size_t)Nl * (K + 1), sizeof(int32_t));
    rb = (uint8_t*)malloc((size_t)Nl);
#endif
#pragma omp for schedule(static)
    for (int c = 0; c < C; ++c) {
        for (int j = 0; j < Nl; ++j) rb[j] = 0;
        for (int64_t l = cptr[c]; l < cptr[c + 1]; ++l) {
            int32_t lit = lits[l];
            int v = (lit > 0 ? lit : -lit) - 1;
            const uint8_t* brow = b + (size_t)v * Nl;
            for (int j = 0; j < Nl; ++j) rb[j] = (uint8_t)(rb[j] + (lit > 0 ? brow[j] : (uint8_t)(1 - brow[j])));
        }
        for (int j = 0; j < Nl; ++j) hl[(size_t)j * (K + 1) + rb[j]] += 1;
    }
#ifdef _OPENMP
#pragma omp critical
    for (int j = 0; j < Nl * (K + 1); ++j) h[j] += hl[j];
    free(hl); free(rb);
#endif
    }
}

/* Backward (as or_backward) for the variables rows[0..nrows): G[i][n] for
 * variable rows[i], evaluating R_cn of each of its clauses directly. */
void or_backward_rows(int C, const int64_t* cptr, const int32_t* lits, int Nl, int K, const uint8_t* b,
                      const float* g, const int32_t* rows, int nrows, double* G, int32_t* cnt, uint8_t* rowbuf)
{
    for (int i = 0; i < nrows; ++i) {
        int v = rows[i];
        memset(cnt, 0, (size_t)Nl * (K + 1) * sizeof(int32_t));
        for (int c = 0; c < C; ++c) {
            int sign = 0;
            for (int64_t l = cptr[c]; l < cptr[c + 1]; ++l) {
                int32_t lit = lits[l];
                if ((lit > 0 ? lit : -lit) - 1 == v) sign += lit > 0 ? -1 : +1;   /* cneg - cpos */
            }
            if (sign == 0) {
                /* v absent, or a tautology x v ~x whose two terms cancel */
                int present = 0;
                for (int64_t l = cptr[c]; l < cptr[c + 1]; ++l)
                    if (((lits[l] > 0 ? lits[l] : -lits[l]) - 1) == v) present = 1;
                if (!present) continue;
            }
            for (int j = 0; j < Nl; ++j) rowbuf[j] = 0;
            for (int64_t l = cptr[c]; l < cptr[c + 1]; ++l) {
                int32_t lit = lits[l];
                int u = (lit > 0 ? lit : -lit) - 1;
                const uint8_t* brow = b + (size_t)u * Nl;
                for (int j = 0; j < Nl; ++j) rowbuf[j] = (uint8_t)(rowbuf[j] + (lit > 0 ? brow[j] : (uint8_t)(1 - brow[j])));
            }
            for (int64_t l = cptr[c]; l < cptr[c + 1]; ++l) {
                int32_t lit = lits[l];
                if (((lit > 0 ? lit : -lit) - 1) != v) continue;
                int delta = lit > 0 ? -1 : +1;
                for (int j = 0; j < Nl; ++j) cnt[(size_t)j * (K + 1) + rowbuf[j]] += delta;
            }
        }
        for (int j = 0; j < Nl; ++j) {
            float acc = 0.0f;
            for (int r = 0; r <= K; ++r)
                acc = fmaf((float)cnt[(size_t)j * (K + 1) + r], g[(size_t)j * (K + 1) + r], acc);
            G[(size_t)i * Nl + j] = (double)acc;
        }
    }
}

/* ------------------------------------------------------------------ fp64 state
 * Variant f2 "fp64 state" (SPEC S:278 chose double throughout; reading R30):
 * theta, m, v in fp64 and every rounding R13/R26/R27/R27b/R6 makes to fp32
 * is made to fp64 instead.  Same definitions, same operation order:
 *   init: the fp64 Box-Muller value (not rounded to fp32);
 *   Q_v = sum round_half_even(theta 2^32) (theta 2^32 is exact in fp64);
 *   g table: Eq. 4's derivative in fp64 (not rounded);
 *   G_vn = fma chain over r ascending of (cneg - cpos)[r] g_n[r] in fp64;
 *   J_v: s_v = 61 - ceil(log2(N occ gmax thmax)) clamped to [-1022, 1023],
 *        terms llrint(G (theta 2^s)) with fp64 products;
 *   grad = fma(G, rho, -c) in fp64 (normalize 3: -sign(theta) c);
 *   AdamW in fp64 with the host scalars unrounded (R6b/R6c order).  */
void or_init64(int V, int64_t n0, int Nl, uint64_t seed, double* theta, double* m, double* vv)
{
    const double two_pi = 6.283185307179586;
    const double two_m32 = 2.3283064365386963e-10; /* 2^-32 */
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    #pragma omp parallel for schedule(static)
    for (int v = 0; v < V; ++v) {
        for (int j = 0; j < Nl; ++j) {
            int64_t n = n0 + j;
            uint32_t ctr[4] = {(uint32_t)(n >> 2), (uint32_t)v, 0u, 0u};
            uint32_t x[4];
            or_philox4x32_10(ctr, key, x);
            int q = (int)(n & 3);
            int pair = q >> 1;
            double u1 = ((double)x[2 * pair] + 1.0) * two_m32;
            double u2 = (double)x[2 * pair + 1] * two_m32;
            double r = sqrt(-2.0 * log(u1));
            double a = two_pi * u2;
            theta[(size_t)v * Nl + j] = (q & 1) ? r * sin(a) : r * cos(a);
            m[(size_t)v * Nl + j] = 0.0;
            vv[(size_t)v * Nl + j] = 0.0;
        }
    }
}

/* R30 row sums: Q_v = sum_n round_half_even(theta_vn 2^64) in a 128-bit
 * integer (theta 2^64 is exact in fp64; |theta| < 2^14 and N <= 2^30 keep
 * |Q| < 2^108), returned as hi (signed) and lo (unsigned) 64-bit halves,
 * Q = hi 2^64 + lo.  The sum is exact and order-free, like R10's, but at
 * the 2^-64 resolution an fp64 state needs.  magnitude: sum |theta| (R28). */
static __int128 round64_q(double x)
{
    double y = x * 18446744073709551616.0;          /* 2^64, exact */
    if (fabs(y) < 4503599627370496.0)               /* < 2^52: may have a fraction */
        return (__int128)llrint(y);                 /* round half even */
    double hi = floor(y * 5.421010862427522e-20);  /* y 2^-64, exact; an integer-valued double */
    double lo = y - hi * 18446744073709551616.0;    /* exact, in [0, 2^64) */
    return (__int128)(int64_t)hi * ((__int128)1 << 64) + (__int128)(uint64_t)lo;
}

int or_row_sums64(int V, int Nl, const double* theta, int64_t* Qhi, uint64_t* Qlo, int magnitude)
{
    int bad = 0;
    #pragma omp parallel for schedule(static) reduction(|:bad)
    for (int v = 0; v < V; ++v) {
        __int128 acc = 0;
        for (int j = 0; j < Nl; ++j) {
            double x = theta[(size_t)v * Nl + j];
            if (magnitude) x = fabs(x);
            if (!(fabs(x) < 16384.0)) bad = 1;
            acc += round64_q(x);
        }
        Qhi[v] = (int64_t)(acc >> 64);
        Qlo[v] = (uint64_t)acc;
    }
    return bad;
}

/* R30 row statistics: S = (double)hi 2^64 + (double)lo (two roundings, in
 * this order), mu = (S 2^-64) / N, then d, rho, guard as or_row_finish. */
void or_row_finish64(int V, int64_t N, const int64_t* Qhi, const uint64_t* Qlo, int normalize, double eps_norm,
                     double* mu, double* d, double* rho, uint8_t* guard)
{
    for (int v = 0; v < V; ++v) {
        if (!normalize) { mu[v] = 0.0; d[v] = 1.0; rho[v] = 1.0; guard[v] = 1; continue; }
        double S = (double)Qhi[v] * 18446744073709551616.0 + (double)Qlo[v];
        double m = (S * 5.421010862427522e-20) / (double)N;
        double a = fabs(m);
        double mag = a > eps_norm ? a : eps_norm;
        mu[v] = m;
        d[v] = m >= 0.0 ? mag : -mag;
        rho[v] = 1.0 / d[v];
        guard[v] = (uint8_t)(a <= eps_norm);
    }
}

void or_binarize64(int V, int Nl, const double* theta, const double* d, uint8_t* b)
{
    #pragma omp parallel for schedule(static)
    for (int v = 0; v < V; ++v)
        for (int j = 0; j < Nl; ++j) {
            double x = theta[(size_t)v * Nl + j];
            b[(size_t)v * Nl + j] = (uint8_t)((x > 0.0 && d[v] > 0.0) || (x < 0.0 && d[v] < 0.0));
        }
}

void or_backward64(int V, int C, const int64_t* cptr, const int32_t* lits, int Nl, int K,
                   const uint8_t* R, const double* g, double* G)
{
    int64_t* vptr = (int64_t*)calloc((size_t)V + 1, sizeof(int64_t));
    int64_t nnz = cptr[C];
    int32_t* occ_c = (int32_t*)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
    int8_t* occ_s = (int8_t*)malloc((size_t)(nnz > 0 ? nnz : 1));
    for (int64_t l = 0; l < nnz; ++l) vptr[(lits[l] > 0 ? lits[l] : -lits[l])]++;
    for (int v = 0; v < V; ++v) vptr[v + 1] += vptr[v];
    int64_t* fill = (int64_t*)malloc(((size_t)V + 1) * sizeof(int64_t));
    memcpy(fill, vptr, ((size_t)V + 1) * sizeof(int64_t));
    for (int c = 0; c < C; ++c)
        for (int64_t l = cptr[c]; l < cptr[c + 1]; ++l) {
            int v = (lits[l] > 0 ? lits[l] : -lits[l]) - 1;
            occ_c[fill[v]] = c;
            occ_s[fill[v]] = lits[l] > 0 ? 1 : -1;
            fill[v]++;
        }
#pragma omp parallel
    {
    int32_t* cnt = (int32_t*)malloc((size_t)Nl * (K + 1) * sizeof(int32_t));
#pragma omp for schedule(dynamic, 16)
    for (int v = 0; v < V; ++v) {
        memset(cnt, 0, (size_t)Nl * (K + 1) * sizeof(int32_t));
        for (int64_t o = vptr[v]; o < vptr[v + 1]; ++o) {
            const uint8_t* Rrow = R + (size_t)occ_c[o] * Nl;
            int delta = occ_s[o] < 0 ? +1 : -1;  /* cneg - cpos */
            for (int j = 0; j < Nl; ++j) cnt[(size_t)j * (K + 1) + Rrow[j]] += delta;
        }
        for (int j = 0; j < Nl; ++j) {
            double acc = 0.0;
            for (int r = 0; r <= K; ++r)
                acc = fma((double)cnt[(size_t)j * (K + 1) + r], g[(size_t)j * (K + 1) + r], acc);
            G[(size_t)v * Nl + j] = acc;
        }
    }
    free(cnt);
    }
    free(fill); free(occ_s); free(occ_c); free(vptr);
}

void or_jacobian_partial64(int V, int Nl, const double* G, const double* theta,
                           const int32_t* occ, int64_t N, double gmax, double thmax,
                           int64_t* I, int32_t* s_out, uint8_t* valid)
{
    #pragma omp parallel for schedule(static)
    for (int v = 0; v < V; ++v) {
        double x = (double)N * (double)occ[v];
        x = x * gmax;
        x = x * thmax;
        I[v] = 0; s_out[v] = 0; valid[v] = 0;
        if (occ[v] == 0 || !(x > 0.0)) continue;
        int s = 61 - ceil_log2(x);
        if (s > 1023) s = 1023;
        if (s < -1022) s = -1022;
        const double p2 = ldexp(1.0, s);
        int64_t acc = 0;
        for (int j = 0; j < Nl; ++j) {
            double ts = theta[(size_t)v * Nl + j] * p2;
            double p = G[(size_t)v * Nl + j] * ts;
            acc += (int64_t)llrint(p);
        }
        I[v] = acc; s_out[v] = s; valid[v] = 1;
    }
}

void or_grad64(int V, int Nl, const double* G, const double* rho, const double* cv, const double* theta,
               int magnitude, double* grad)
{
    #pragma omp parallel for schedule(static)
    for (int v = 0; v < V; ++v)
        for (int j = 0; j < Nl; ++j) {
            double c = cv[v];
            if (magnitude) {
                const double x = theta[(size_t)v * Nl + j];
                c = x > 0.0 ? c : (x < 0.0 ? -c : 0.0);
            }
            grad[(size_t)v * Nl + j] = fma(G[(size_t)v * Nl + j], rho[v], -c);
        }
}

void or_adamw64(int V, int64_t n0, int Nl, double* theta, double* m, double* vv, const double* grad,
                int64_t t, int64_t bstep, double lr, double beta1, double beta2, double eps, double wd,
                double noise_sigma, uint64_t seed)
{
    double s = (double)bstep;
    double wdf = 1.0 - lr * wd;
    double a1 = 1.0 - beta1;
    double a2 = 1.0 - beta2;
    double bc1 = 1.0 - pow(beta1, s);
    double bc2 = 1.0 - pow(beta2, s);
    double nss = -(lr / bc1);
    double rbc2 = 1.0 / sqrt(bc2);
    double nz = lr * noise_sigma;
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
#pragma omp parallel for schedule(static)
    for (int v = 0; v < V; ++v)
        for (int j = 0; j < Nl; ++j) {
            size_t i = (size_t)v * Nl + j;
            double g = grad[i];
            double th = theta[i] * wdf;
            double mm = fma(a1, g - m[i], m[i]);
            double vb = vv[i] * beta2;
            double vn = fma(a2 * g, g, vb);
            double den = sqrt(vn) * rbc2 + eps;
            th = th + (nss * mm) / den;
            if (noise_sigma != 0.0) {
                int64_t n = n0 + j;
                uint32_t ctr[4] = {(uint32_t)(n >> 2), (uint32_t)v, (uint32_t)(1 + t), 0u};
                uint32_t x[4];
                or_philox4x32_10(ctr, key, x);
                double xi = (double)(x[n & 3] >> 8) * 5.9604644775390625e-08 - 0.5;
                th = th + nz * xi;
            }
            theta[i] = th; m[i] = mm; vv[i] = vn;
        }
}

double or_abs_max64(size_t n, const double* x)
{
    double mx = 0.0;
    for (size_t i = 0; i < n; ++i) { double a = fabs(x[i]); if (a > mx) mx = a; }
    return mx;
}

double or_gmax64(int Nl, int K, const double* g, const int32_t* rmin)
{
    double mx = 0.0;
    for (int j = 0; j < Nl; ++j)
        for (int r = rmin[j]; r <= K; ++r) {
            double a = fabs(g[(size_t)j * (K + 1) + r]);
            if (a > mx) mx = a;
        }
    return mx;
}
