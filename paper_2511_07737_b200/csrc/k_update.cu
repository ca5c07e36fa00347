// k_update.cu - rows (a7) STE backward, (a8) Eq. 5 Jacobian, (a9) AdamW +
// re-binarisation, fused (§3.2 l.189-191, l.226; §4.1 l.255-269).
//
// k_update (fused, persistent): one CTA per SM holds the fp32 derivative
// table g[r][n] of the whole batch in shared memory (loaded once per launch);
// its warp groups pull rows v from a global counter.  For a row:
//  1. gather (word-major, lane = 32-candidate word): for every occurrence of
//     v the clause's R_cn is recomputed from the bit planes of the evaluated
//     state (coalesced 128-byte gathers, no R matrix in HBM) and the one-hot
//     masks [R = r] are added (+ for a negated occurrence, - for a positive
//     one) to 8-bit two's-complement vertical counters d_r = cneg - cpos;
//  2. a 32x32 bit transpose turns the counter planes into one packed word of
//     signed bytes per candidate, staged in shared memory;
//  3. candidate-major (float4 streams of theta, m, v): G = sum_r d_r g[r]
//     (fp32 FMA chain over the exact counts, r ascending: R27), J_v = sum G
//     theta in int64 fixed point (R13, group reduction), c_v, grad =
//     fmaf(G, rho, -c) (R27b), AdamW, Q_{t+1}, max|theta|, and the sign planes
//     of theta_{t+1} -> bits of the next state.
// Records: uniform 3-SAT rows are staged as plain occurrence records, every
// other instance as batched records (host_cnf.cpp build_batched).
// Rows whose counts can leave int8 ("hubs", SURVEY §7 hard parts) get their
// counts from k_hub, which splits a hub's occurrences over many CTAs and adds
// exact int32 counts (integer atomics: order-free, deterministic).
#include "cluster.cuh"
#include "peer.cuh"

#include "upd_common.cuh"

// L2 bulk prefetch of each row's theta / m / v at the row's start: 0 never,
// 1 always, 2 while the rows in flight (CTAs x groups x 12 B x candidates)
// stay below TSAT_PREFETCH_BYTES - beyond that the prefetched lines are
// evicted before pass 3b reads them (c5 N = 8192: 87 MB in flight, k_update
// 5.82 -> 5.26 ms without; c2 49.7 MB: 0.264 -> 0.249 ms with)
#ifndef TSAT_UPD_NT
#define TSAT_UPD_NT 1                // compile-time batch size for c4's shape (MODE 0, KB = 8, N = 2048)
#endif
#ifndef TSAT_ROW_PREFETCH
#define TSAT_ROW_PREFETCH 2
#endif
#ifndef TSAT_PREFETCH_BYTES
#define TSAT_PREFETCH_BYTES 64.0e6
#endif
#ifndef TSAT_PREFETCH_THETA
#define TSAT_PREFETCH_THETA 1        // beyond the bound, prefetch theta alone if that fits (c5 N = 8192 step 5.85 -> 5.67 ms)
#endif

namespace tsat {

// MODE 0: fused W = 1 iteration.  MODE 1: phase A of the sharded iteration
// (G -> Gbuf, int64 J partial -> Jbuf; the AdamW phase runs after the J exchange).
// MODE 2: the fused iteration on W GPUs with the exchanges inside the kernel
// over peer memory (peer.cuh): the per-step scalars at the start, and per row
// the J partial (before the gradient) and the Q partial (before the next
// state's statistics); other warp groups keep streaming while one waits.
// Rows come from a global counter (dynamic: hub rows, ragged occurrence counts
// and the tail stay balanced); tg 0 fetches the next row at the start of the
// current one into a parity-double-buffered slot, read after the J barrier.
// MAG: normalize 3 (R28, d = mean |theta|): the Jacobian addend carries
// sign(theta) and the next row sums are of |theta| (a template flag: a
// run-time one costs the default path ~3 % at c2 / c3).
// CW: counter planes of the K <= 3 gather (8, or 6 when no row has more than
// 31 same-sign occurrences: 6 fewer registers, compiled for 896 threads).
// MODE 3: cluster-split rows (W = 1, large N): the CL CTAs of a cluster each
// own N / CL candidates of every row (their slice of the g table in shared
// memory) and process the same rows in a static order; the row's J and Q
// partials are summed over DSMEM (cluster.cuh), so no G round trip through
// HBM and no g table reads from L2.
// NT > 0 (MODE 0): the batch size as a compile-time constant, used for c4's
// shape (KB = 8, N = 2048: k_update -0.9 %); for KB = 4 at c2's 4096, c3's
// 1024 and c5's 8192 it measured equal or slower (c2 +3 %: more spills), so
// those keep the run-time geometry.
template <int KB, int MODE, bool MAG = false, bool GSG = false, int CW = 8, int NT = 0>
__global__ void __launch_bounds__(KB == 4 ? (MODE == 2 ? TSAT_UPD_THREADS4P : (CW == 6 ? TSAT_UPD_THREADS4C6 : TSAT_UPD_THREADS4))
                                          : TSAT_UPD_THREADS8, 1) k_update(StepArgs a, const uint32_t* __restrict__ Acur,
                                                                    uint32_t* __restrict__ Anext,
                                                                    const StepScalars* __restrict__ sc) {
    constexpr int NP = (KB == 4) ? 2 : (KB == 8 ? 3 : 4);
    constexpr int NCTR = KB - 1;
    extern __shared__ __align__(16) unsigned char smem[];
    const int N = NT ? NT : a.N, NW = N >> 5;
    const int GT = NT ? ((NT >> 5) >= 128 ? 128 : ((NT >> 5) > 32 ? 64 : 32)) : a.upd_GT;   // as configure_update
    // work item = (row, chunk of NCH candidates); NCH == N except for batches
    // too large for shared memory (MODE 1 only), whose g table stays in L2
    constexpr bool CLU = MODE == 3;
    const int NCH = (MODE == 1 || CLU) ? a.upd_chunk : N;
    const int nch = MODE == 1 ? (N + NCH - 1) / NCH : 1;  // compile-time 1: fused modes keep smem addressing
    const unsigned crank = CLU ? cluster_rank() : 0u;      // MODE 3: this CTA's candidate slice
    const int n0cl = CLU ? (int)crank * NCH : 0;
    const int NWg = NCH >> 5;                              // words of the group's sign-plane slots
    // g table read through L1/L2: chunked items (MODE 1, run-time flag), or the
    // fused kernel for large N (GSG: a separate instantiation, so the default
    // path keeps its shared-memory loads)
    const bool gs_global = GSG || (MODE == 1 && a.upd_gs_global != 0);
    const size_t dpkw = upd_dpk_words(NCH);
    float* gs = gs_global ? a.gtab : reinterpret_cast<float*>(smem);
    const int grp = threadIdx.x / GT, tg = threadIdx.x - grp * GT;
    const int rec_cap = a.upd_rec_cap;
    constexpr int nbufs = upd_recbufs(KB);
    constexpr bool DEFER = MODE == 2 || CLU;                 // the row's Q arrives late: finish it one row later
    const size_t grb = upd_group_bytes(KB, NCH, rec_cap, nbufs, DEFER ? 2 : 1, CLU);
    unsigned char* gb = smem + (gs_global ? 0 : upd_gs_bytes(KB, CLU ? NCH : N)) + (size_t)grp * grb;
    const int nitems = a.V * nch;
    uint32_t* dpk = reinterpret_cast<uint32_t*>(gb);
    uint32_t* rec = reinterpret_cast<uint32_t*>(gb + align16((size_t)(KB == 4 ? 1 : 2) * dpkw * 4));
    const size_t recw = align16((size_t)rec_cap * 4) / 4;            // words per record buffer
    uint32_t* posw0 = rec + nbufs * recw;            // [parity][pos | neg][NW] (MODE 2 finishes a row late)
    long long* red = reinterpret_cast<long long*>(gb + grb - 128);                      // 4 + 4 slots
    float* redf = reinterpret_cast<float*>(red + 8);                                    // 4 slots
    int* rowslot = reinterpret_cast<int*>(redf + 4);                                    // 2 slots
    long long* pxs = red + 11;                                                          // 2 slots (MODE 2)
    unsigned long long* xsl = reinterpret_cast<unsigned long long*>(gb + grb - 128 - kClusterSlotBytes);   // MODE 3
    unsigned long long* xsJ = xsl;                           // [kMaxCluster][2] J partials
    unsigned long long* xsQ = xsl + 2 * kMaxCluster;         // [kMaxCluster][2] Q partials
    const int bar = 1 + grp;
    const int lane = threadIdx.x & 31, gw = tg >> 5, ngw = GT >> 5;
    const bool uni3 = a.uniform_len && a.mc.K == 3 && KB == 4;
    const unsigned long long pol = plane_policy(planes_fit_l2(a.V, NW));

    pdl_wait();                                          // k_gtable's table and scalars
    pdl_trigger();
    // fp32 derivative table of the whole batch (MODE 3: of this CTA's slice) -> shared memory
    if (CLU) {
        for (int i = threadIdx.x * 4; i < KB * NCH; i += blockDim.x * 4) {
            const int r = i / NCH, c = i - r * NCH;
            *reinterpret_cast<float4*>(gs + i) = *reinterpret_cast<const float4*>(a.gtab + (size_t)r * N + n0cl + c);
        }
        for (int i = tg; i < 4 * kMaxCluster; i += GT) xsl[i] = 0ull;   // no message seq is 0
    } else if (!gs_global) {
        for (int i = threadIdx.x * 4; i < KB * N; i += blockDim.x * 4)
            *reinterpret_cast<float4*>(gs + i) = *reinterpret_cast<const float4*>(a.gtab + i);
    }
    if (!CLU && tg == 0) rowslot[1] = atomicAdd(&a.ds->row_counter, 1);
    const long long t = sc->t;
    __shared__ unsigned long long pscal[3];         // MODE 2: global best key, gmax bits, thmax bits
    if (MODE == 2 && threadIdx.x == 0) {
        const unsigned long long own[4] = {~a.ds->best_key, a.ds->gmax_bits,
                                           (unsigned long long)a.ds->thmax_bits[t & 1],
                                           (unsigned long long)a.ds->loss_fx};
        unsigned long long x[4];
        peer_recv_scalars(a.px, sc->xgen, a.ds, own, x);
        pscal[0] = ~x[0];
        pscal[1] = a.px.exchange_rows ? x[1] : a.ds->gmax_bits;           // per shard: J scale stays local
        pscal[2] = a.px.exchange_rows ? x[2] : (unsigned long long)a.ds->thmax_bits[t & 1];
        if (blockIdx.x == 0) {                      // step bookkeeping with the global values
            const int bu = (int)(pscal[0] >> 32);
            const long long bi = (long long)(pscal[0] & 0xffffffffull);
            if (bu == 0 && a.ds->sol_step < 0) { a.ds->sol_step = t; a.ds->sol_idx = bi; }
            const double loss = -((double)(long long)x[3] * a.mc.loss_unscale);     // * 2^-e
            a.ds->loss = loss;
            a.ds->info_t = t + 1;
            a.ds->info_best_unsat = bu;
            a.ds->info_best_idx = bi;
            a.ds->info_loss = loss;
        }
    }
    __syncthreads();
    // MODE 3: static row schedule (the cluster's CTAs must pair their groups
    // on the same rows); every CTA's slots are zeroed before any DSMEM write
    const int cl_slot = CLU ? (int)cluster_id_x() * a.upd_NG + grp : 0;
    const int cl_stride = CLU ? (int)cluster_count_x() * a.upd_NG : 0;
    const unsigned CLn = CLU ? (unsigned)a.upd_cl : 1u;
    if (CLU) cluster_sync_all();

    const double gmax = __longlong_as_double((long long)(MODE == 2 ? pscal[1] : a.ds->gmax_bits));
    const float thmax = __uint_as_float(MODE == 2 ? (unsigned)pscal[2] : a.ds->thmax_bits[t & 1]);
    const float wdf = sc->wdf, a1 = sc->a1, b2f = sc->b2f, a2 = sc->a2, nss = sc->nss, rbc2 = sc->rbc2,
                epsf = sc->epsf, nz = sc->nz, mkeep = sc->mkeep;
    const MethodConsts& mc = a.mc;

    // Row v of theta_{t+1} is complete once its global Q is known: bit planes
    // (sign(d) = sign(Q), R3) and, by tg 0, Eq. 5's statistics, max |theta|
    // and the first model's bits.
    auto finish_row = [&](int vr, long long Qg, const uint32_t* pw, float m2) {
        const bool dpos = !mc.normalize || Qg >= 0;
        const uint32_t* src = dpos ? pw : pw + NWg;
        uint32_t* dst = Anext + (size_t)vr * NW + (n0cl >> 5);   // MODE 3: this CTA's words of the row
        for (int w = tg; w < NWg; w += GT) {
#if TSAT_ANEXT_CS
            __stcs(dst + w, src[w]);                            // streaming: keep L2 for the current planes
#else
            dst[w] = src[w];
#endif
        }
        if (tg == 0) {
            if (crank == 0) {
                double dn, rhon;
                unsigned char gn;
                row_finish(Qg, mc, &dn, &rhon, &gn);
                a.rowQ[vr] = Qg; a.rowD[vr] = dn; a.rowRho[vr] = rhon; a.rowGuard[vr] = gn;
            }
            atomicMax(&a.ds->thmax_bits[(t + 1) & 1], __float_as_uint(m2));
            const unsigned long long bk = MODE == 2 ? pscal[0] : a.ds->best_key;
            if ((bk >> 32) == 0ull && (a.ds->sol_step < 0 || a.ds->sol_step == t)) {          // first model: keep its bits (A22)
                const long long idx = (long long)(bk & 0xffffffffull) - mc.n0;
                if (idx >= n0cl && idx < n0cl + NCH)
                    a.sol[vr] = (unsigned char)((Acur[(size_t)vr * NW + (idx >> 5)] >> (idx & 31)) & 1u);
            }
        }
    };
    // MODE 2: the row awaiting its global Q (finished one row late); its
    // local Q partial and max |theta| live in the group's scratch (tg 0 alone
    // writes and reads them), its sign planes in the other parity slot
    int pend_v = -1;
    long long* pend_q = red + 13;
    float* pend_m2 = reinterpret_cast<float*>(red + 14);

    int item = CLU ? cl_slot : rowslot[1];
    if (item < nitems && a.hub_of[item / nch] < 0) {      // first row: stage its records now
        const int v0 = item / nch;
        const unsigned rb0 = a.upd_ptr[v0], re0 = a.upd_ptr[v0 + 1];
        for (unsigned i = tg; i < re0 - rb0; i += GT) rec[i] = a.upd_rec[rb0 + i];
    }
    gsync(bar, GT);
    int it = 0;
    for (; item < nitems; ++it) {
        const int v = item / nch;
        const int n0c = CLU ? n0cl : (item - v * nch) * NCH;    // first candidate of this chunk
        const int ncand = min(NCH, N - n0c), w0 = n0c >> 5, NWc = ncand >> 5;
        uint32_t* rb_cur = rec + (size_t)(nbufs == 2 ? (it & 1) : 0) * recw;     // this row's records
        uint32_t* rb_nxt = rec + (size_t)(nbufs == 2 ? ((it + 1) & 1) : 0) * recw;
        // ---- fetch the next row; prefetch this row's streams into L2
        if (tg == 0) {
            if (!CLU) rowslot[it & 1] = atomicAdd(&a.ds->row_counter, 1);
            const uint32_t rowbytes = (uint32_t)ncand * 4u;
            if (a.upd_prefetch) {                            // configure_update: rows in flight fit L2
                prefetch_l2(a.theta + (size_t)v * N + n0c, rowbytes);
                if (MODE != 1 && a.upd_prefetch == 1) {
                    prefetch_l2(a.m + (size_t)v * N + n0c, rowbytes);
                    prefetch_l2(a.v + (size_t)v * N + n0c, rowbytes);
                }
            }
        }
        uint32_t* posw = posw0 + (DEFER ? (size_t)(it & 1) * 2 * NWg : 0);
        uint32_t* negw = posw + NWg;
        const int hub = a.hub_of[v];
        const int2 pn = a.occ_pn[v];
        const int dsum = pn.y - pn.x;                       // sum_r (cneg - cpos)[r]
        const unsigned rb = a.upd_ptr[v], re = a.upd_ptr[v + 1];
        const double rho = a.rowRho[v];
        const unsigned char guard = a.rowGuard[v];
        const int occ = pn.x + pn.y;
        int s;
        float p2;
        const bool jvalid = jscale(mc.Nnorm, occ, gmax, thmax, &s, &p2);
        int* hubrow = hub >= 0 ? a.hubD + (size_t)hub * NCTR * N : nullptr;
        float* trow = a.theta + (size_t)v * N;
        float* mrow = a.m + (size_t)v * N;
        float* vrow = a.v + (size_t)v * N;

        // ---- 1+2: bit-sliced gather of the row's occurrences, transpose to bytes
        // (KB = 16: every row is a hub row, counted by k_hub)
        if constexpr (KB <= 8) if (hub < 0) {
            const unsigned nrec = re - rb;
            for (int wl = tg; wl < NWc; wl += GT) {
                const int w = w0 + wl;
                const uint32_t own = __ldg(Acur + (size_t)v * NW + w);
                constexpr int kB = KB == 4 ? CW : kCtr;        // counter planes (two's complement)
                uint32_t cnt[NCTR][kB];
                auto recf = [&](unsigned i) { return rb_cur[i]; };
                if (uni3) {
#if TSAT_UNI3 == 0
                    count_occurrences<NP, NCTR, kB, true, true>(cnt, recf, nrec, own, Acur, (unsigned)NW, (unsigned)w, pol);
#else
                    count_uni3<NCTR, kB, TSAT_UNI3 == 1>(cnt, recf, (unsigned)pn.y, (unsigned)pn.x, own, Acur,
                                                          (unsigned)NW, (unsigned)w, pol);
#endif
                }
                else count_batched<NP, NCTR, kB>(cnt, recf, nrec, own, Acur, (unsigned)NW, (unsigned)w, pol);
                // counter planes of bins 4 blk .. 4 blk + 3 -> one packed word per
                // candidate; KB = 8 loops over two blocks (one transpose in the
                // code: the kernel is instruction-cache bound there)
#pragma unroll 1
                for (int blk = 0; blk < (KB == 8 ? 2 : 1); ++blk) {
                    uint32_t T[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int r = i / kCtr, b = (i % kCtr) < kB ? (i % kCtr) : kB - 1;   // sign-extend to 8 bits
                        const uint32_t lo = (r < NCTR && r < 4) ? cnt[r][b] : 0u;
                        const uint32_t hi = (4 + r < NCTR) ? cnt[4 + r][b] : 0u;
                        T[i] = blk ? hi : lo;
                    }
                    transpose32(T);
#pragma unroll
                    for (int j = 0; j < 32; ++j) dpk[blk * dpkw + 33 * wl + j] = T[j];
                }
            }
        }
        if (MODE == 2 && pend_v >= 0 && tg == 0)             // previous row's Q, sent a row ago
            pxs[1] = peer_row_recv(a.px, 1, pend_v, sc->xgen, a.ds, *pend_q);
        if (CLU && pend_v >= 0 && tg == 0)                   // previous row's Q over the cluster (seq = it)
            pxs[1] = cl_recv_sum(xsQ, CLn, crank, (unsigned)it, *pend_q, a.ds);
        gsync(bar, GT);
        const int item_next = CLU ? item + cl_stride : rowslot[it & 1];   // fetched by tg 0 before the gather
        const int vnext = item_next < nitems ? item_next / nch : a.V;
        // stage the next row's records asynchronously (cp.async global -> smem);
        // they land while this row streams and are waited for before the Q
        // barrier.  One buffer: this row's records are dead after the gather.
        auto stage_next = [&]() {
            if (vnext < a.V && a.hub_of[vnext] < 0) {
                const unsigned nb = a.upd_ptr[vnext], ne = a.upd_ptr[vnext + 1];
                for (unsigned i = tg; i < ne - nb; i += GT) cp_async4(rb_nxt + i, a.upd_rec + nb + i);
            }
            cp_async_commit();
        };
        if (nbufs == 1) stage_next();
        if (DEFER && pend_v >= 0) {
            finish_row(pend_v, pxs[1], posw0 + (size_t)((it + 1) & 1) * 2 * NWg, *pend_m2);
            pend_v = -1;
        }

        // ---- 3a: G (fp32 FMA chain over exact counts, R27) -> smem; J_v partial
        float* gout = MODE == 1 ? a.Gbuf + (size_t)v * N + n0c : nullptr;
        int* hubc = hubrow ? hubrow + n0c : nullptr;
        long long I;
        const float* gsc = CLU ? gs : gs + n0c;             // MODE 3: the slice table, row stride NCH
        const int Ngs = CLU ? NCH : N;
        if (KB > 8 || hub >= 0)
            I = pass_fold<KB, true>(trow + n0c, dpk, dpkw, gsc, hubc, ncand, N, GT, tg, dsum, jvalid, p2, gout, Ngs);
        else
            I = pass_fold<KB <= 8 ? KB : 8, false>(trow + n0c, dpk, dpkw, gsc, hubc, ncand, N, GT, tg, dsum, jvalid,
                                                   p2, gout, Ngs);
        I = warp_sum(I);
        if (lane == 0) red[gw] = I;
        gsync(bar, GT);
        long long Itot = 0;                                  // every thread folds the warp partials
        for (int i = 0; i < ngw; ++i) Itot += red[i];
        if (MODE == 2 && a.px.exchange_rows) {               // J_v over all ranks
            // every thread adds the W - 1 remote partials itself: no broadcast barrier
            if (tg == 0) peer_row_send(a.px, 0, v, Itot, sc->xgen);
            Itot = peer_row_recv(a.px, 0, v, sc->xgen, a.ds, Itot);
        }
        if (CLU) {                                           // J_v over the cluster's slices (DSMEM)
            if (tg == 0) cl_send(xsJ, CLn, crank, (unsigned)it + 1u, Itot);
            long long Jr = 0;                                // lane 0 of each warp polls, then broadcasts
            if (lane == 0) Jr = cl_recv_sum(xsJ, CLn, crank, (unsigned)it + 1u, Itot, a.ds);
            Itot = __shfl_sync(0xffffffffu, Jr, 0);
        }
        if (nbufs == 2) stage_next();
        if (MODE == 1) {                                     // sharded / chunked: J partial out, next item
            if (tg == 0) {
                if (nch > 1) atomicAdd(reinterpret_cast<unsigned long long*>(a.Jbuf + v), (unsigned long long)Itot);
                else a.Jbuf[v] = Itot;
            }
            cp_async_wait_all();
            gsync(bar, GT);
            item = item_next;
            continue;
        }
        double c = 0.0;
        if (mc.normalize && !guard) {
            const double J = jvalid ? times_pow2((double)Itot, -s) : 0.0;
            c = J / (double)mc.Nnorm;
            c = c * rho;
            c = c * rho;
        }
        const float rhof = __double2float_rn(rho), ncf = -__double2float_rn(c);     // R27b: fp32 operands
        constexpr bool mag = MAG;

        // ---- 3b: grad, AdamW, next-state statistics and sign planes
        long long Qn = 0;
        float mx = 0.0f;
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        float4 thn = z4, mn4 = z4, vn4 = z4;
        // this CTA's candidates of the row (MODE 3: its slice; otherwise the row)
        const int NL = CLU ? NCH : N;
        float* const tr = trow + (CLU ? n0cl : 0);
        float* const mr = mrow + (CLU ? n0cl : 0);
        float* const vr3 = vrow + (CLU ? n0cl : 0);
        if (4 * tg < NL) {
            thn = ld_last(tr + 4 * tg);
            mn4 = ld_last(mr + 4 * tg);
            vn4 = ld_last(vr3 + 4 * tg);
        }
#pragma unroll kUnroll3b
        for (int base = 0; base < NL; base += 4 * GT) {
            const int n = base + 4 * tg;
            unsigned pnib = 0, nnib = 0;
            const float4 th4 = thn, m4 = mn4, v4 = vn4;       // software pipeline: next loads in flight
            if (n + 4 * GT < NL) {
                thn = ld_last(tr + n + 4 * GT);
                mn4 = ld_last(mr + n + 4 * GT);
                vn4 = ld_last(vr3 + n + 4 * GT);
            }
            if (n < NL) {
                float th[4] = {th4.x, th4.y, th4.z, th4.w};
                float mm[4] = {m4.x, m4.y, m4.z, m4.w};
                float vv[4] = {v4.x, v4.y, v4.z, v4.w};
                const uint32_t* dp = dpk + n + (n >> 5);
                float gg[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) gg[q] = __fmaf_rn(__uint_as_float(dp[q]), rhof, jac_addend(ncf, th[q], mag));
                // AdamW on candidate pairs: packed fp32x2 ops are per-lane
                // correctly rounded, i.e. the same canonical ops (R6-R6c)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float2 g2 = make_float2(gg[2 * h], gg[2 * h + 1]);
                    const float2 m2 = mul2_unfused(make_float2(mm[2 * h], mm[2 * h + 1]), make_float2(mkeep, mkeep));
                    const float2 v2 = make_float2(vv[2 * h], vv[2 * h + 1]);
                    float2 x2 = mul2_unfused(make_float2(th[2 * h], th[2 * h + 1]), make_float2(wdf, wdf));
                    const float2 mn2 = __ffma2_rn(make_float2(a1, a1), __fadd2_rn(g2, make_float2(-m2.x, -m2.y)), m2);
                    const float2 vb2 = __fmul2_rn(v2, make_float2(b2f, b2f));
                    const float2 vn2 = __ffma2_rn(__fmul2_rn(make_float2(a2, a2), g2), g2, vb2);
                    const float2 sq2 = make_float2(__fsqrt_rn(vn2.x), __fsqrt_rn(vn2.y));
                    const float2 den2 = __fadd2_rn(mul2_unfused(sq2, make_float2(rbc2, rbc2)), make_float2(epsf, epsf));
                    const float2 num2 = __fmul2_rn(make_float2(nss, nss), mn2);
                    x2 = __fadd2_rn(x2, make_float2(num2.x / den2.x, num2.y / den2.y));
                    float xs0 = x2.x, xs1 = x2.y;
                    if (mc.noise) {
                        xs0 = xs0 + nz * noise_xi(mc.seed, mc.n0 + n0cl + n + 2 * h, v, t);
                        xs1 = xs1 + nz * noise_xi(mc.seed, mc.n0 + n0cl + n + 2 * h + 1, v, t);
                    }
                    const float xs[2] = {xs0, xs1};
                    const float2 q2 = __fmul2_rn(mag ? make_float2(fabsf(xs0), fabsf(xs1)) : make_float2(xs0, xs1),
                                                 make_float2(4294967296.0f, 4294967296.0f));   // R28: |theta|
                    Qn += __float2ll_rn(q2.x) + __float2ll_rn(q2.y);      // x 2^32 is exact in fp32
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int q = 2 * h + e;
                        const float x = xs[e];
                        th[q] = x;
                        mm[q] = e ? mn2.y : mn2.x;
                        vv[q] = e ? vn2.y : vn2.x;
                        mx = fmaxf(mx, fabsf(x));
                        pnib |= (x > 0.0f ? 1u : 0u) << q;
                        nnib |= (x < 0.0f ? 1u : 0u) << q;
                    }
                }
                st_stream(tr + n, make_float4(th[0], th[1], th[2], th[3]));
                st_stream(mr + n, make_float4(mm[0], mm[1], mm[2], mm[3]));
                st_stream(vr3 + n, make_float4(vv[0], vv[1], vv[2], vv[3]));
            }
            // 8 lanes x 4 candidates = one 32-candidate word
            unsigned pw = pnib << (4 * (lane & 7)), nw = nnib << (4 * (lane & 7));
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                pw |= __shfl_xor_sync(0xffffffffu, pw, o);
                nw |= __shfl_xor_sync(0xffffffffu, nw, o);
            }
            if ((lane & 7) == 0 && n < NL) { posw[n >> 5] = pw; negw[n >> 5] = nw; }
        }
        Qn = warp_sum(Qn);
        mx = warp_maxf(mx);
        if (lane == 0) { red[4 + gw] = Qn; redf[gw] = mx; }
        cp_async_wait_all();                                 // next row's records visible after this barrier
        gsync(bar, GT);
        long long Qtot = 0;
        for (int i = 0; i < ngw; ++i) Qtot += red[4 + i];
        float m2 = 0.0f;
        if (tg == 0)
            for (int i = 0; i < ngw; ++i) m2 = fmaxf(m2, redf[i]);
        if (CLU) {                                           // Q_{t+1,v} over the cluster: finished after the next gather
            if (tg == 0) {
                cl_send(xsQ, CLn, crank, (unsigned)it + 1u, Qtot);
                *pend_m2 = m2;
                *pend_q = Qtot;
            }
            pend_v = v;
        } else if (MODE == 2 && a.px.exchange_rows) {
            // Q_{t+1,v} over all ranks: send now, finish the row after the
            // next row's gather (the peers' partials have arrived by then)
            if (tg == 0) peer_row_send(a.px, 1, v, Qtot, sc->xgen);
            pend_v = v;
            if (tg == 0) { *pend_m2 = m2; *pend_q = Qtot; }
        } else {
            finish_row(v, Qtot, posw, m2);
        }
        item = item_next;
        // (the next row's barriers order these smem reads before any reuse)
    }
    if (DEFER && pend_v >= 0) {
        if (tg == 0)
            pxs[1] = CLU ? cl_recv_sum(xsQ, CLn, crank, (unsigned)it, *pend_q, a.ds)
                         : peer_row_recv(a.px, 1, pend_v, sc->xgen, a.ds, *pend_q);
        gsync(bar, GT);
        finish_row(pend_v, pxs[1], posw0 + (size_t)((it + 1) & 1) * 2 * NWg, *pend_m2);
    }
    if (CLU) cluster_sync_all();                             // no DSMEM write may target an exited CTA
}

// ------------------------------------------------------------------ hub pre-pass
// One warp per (hub super-chunk: <= kHubSlab occurrences, or kHubSlabBatches batches, 32-word block):
// 11-bit signed vertical counters, two counters per 32x32 transpose (16-bit
// fields), then exact int32 atomic adds into hubD[hub][r][n].
#ifndef TSAT_HUB_MINB
#define TSAT_HUB_MINB 16          // k_hub blocks (warps) per SM the kernel is compiled for (<= 128 registers)
#endif
// Bins R0 .. R0 + NB - 1 of one super-chunk (KB = 16 runs two passes of <= 8
// bins over the same records so the counters stay within the register budget).
template <int KB, bool BATCHED, int R0, int NB>
__device__ __forceinline__ void hub_bins(const StepArgs& a, const uint32_t* __restrict__ Acur, int (&sh)[2][1024 + 32]) {
    constexpr int NP = (KB == 4) ? 2 : (KB == 8 ? 3 : 4);
    constexpr int NCTR = KB - 1;
    constexpr int kHubCtr = BATCHED ? kHubCtrBatched : kHubCtrPlain;
    const int lane = threadIdx.x;
    const int NW = a.N >> 5;
    const int w = blockIdx.y * 32 + lane;
    const bool valid = w < NW;
    const int4 sc = a.hub_sc[blockIdx.x];          // hub, var, rec_begin, rec_end
    const int v = sc.y;
    const uint32_t own = valid ? __ldg(Acur + (size_t)v * NW + w) : 0u;
    const unsigned long long pol = plane_policy(planes_fit_l2(a.V, NW));
    uint32_t cnt[NB][kHubCtr];
    const uint32_t* recg = a.upd_rec + sc.z;             // the records k_update stages (plain or batched)
    auto recf = [&](unsigned i) { return __ldg(recg + i); };
    if constexpr (BATCHED)
        count_batched<NP, NB, kHubCtr, R0>(cnt, recf, (unsigned)(sc.w - sc.z), own, Acur, (unsigned)NW,
                                           valid ? (unsigned)w : 0u, pol);
    else
        count_occurrences<NP, NB, kHubCtr, false, true>(cnt, recf, (unsigned)(sc.w - sc.z), own, Acur, (unsigned)NW,
                                                        valid ? (unsigned)w : 0u, pol);
    // two counters per transpose (16-bit fields, bits 11..15 = sign extension),
    // staged through shared memory two bins at a time so the atomics coalesce
    int* dst = a.hubD + (size_t)sc.x * NCTR * a.N;
#pragma unroll
    for (int r0 = 0; r0 < NB; r0 += 2) {
        uint32_t T[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const int r = r0 + i / 16, b = i % 16;
            T[i] = (r < NB) ? cnt[r][b < kHubCtr ? b : kHubCtr - 1] : 0u;
        }
        transpose32(T);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            sh[0][33 * lane + j] = (int)(short)(T[j] & 0xffffu);
            sh[1][33 * lane + j] = (int)(short)(T[j] >> 16);
        }
        __syncwarp();
        for (int rr = 0; rr < 2 && r0 + rr < NB; ++rr)
#pragma unroll 4
            for (int k = 0; k < 32; ++k) {
                const int nl = 32 * k + lane;                  // candidate within the block (coalesced)
                const int n = blockIdx.y * 1024 + nl;
                const int val = sh[rr][33 * k + lane];
                if (n < a.N && val) atomicAdd(dst + (size_t)(R0 + r0 + rr) * a.N + n, val);
            }
        __syncwarp();
    }
}

template <int KB, bool BATCHED>
__global__ void __launch_bounds__(32, TSAT_HUB_MINB) k_hub(StepArgs a, const uint32_t* __restrict__ Acur) {
    __shared__ int sh[2][1024 + 32];
    if constexpr (KB <= 8) {
        hub_bins<KB, BATCHED, 0, KB - 1>(a, Acur, sh);
    } else {                          // KB = 16 (batched records only): bins 0-7, then 8-14
        hub_bins<KB, true, 0, 8>(a, Acur, sh);
        hub_bins<KB, true, 8, 7>(a, Acur, sh);
    }
}

// Fused geometry (g table of the batch in smem, one work item per row) when
// at least two warp groups fit; otherwise work items of NCH candidates with
// the g table read from L2 (MODE 1, the split sequence; capi.cu).
bool update_fits_fused(int KB, int N, int rec_cap, int optin) {
    const int NW = N >> 5;
    const int GT = NW >= 128 ? 128 : (NW > 32 ? 64 : 32);
    const size_t gsb = upd_gs_bytes(KB, N), grb = upd_group_bytes(KB, N, rec_cap, upd_recbufs(KB));
    const long long ng = optin > (long long)gsb ? ((long long)optin - (long long)gsb) / (long long)grb : 0;
    return ng >= 2 || (ng == 1 && GT == 128);
}

#ifndef TSAT_GS_GLOBAL_BELOW
#define TSAT_GS_GLOBAL_BELOW 4       // fused kernel: g table from L2 when smem would hold fewer groups
#endif
// Cluster-split rows (MODE 3, W = 1): the smallest cluster size CL = 2, 4, 8,
// 16 whose slice N / CL (a multiple of 128 candidates) keeps the slice's g
// table in shared memory beside >= TSAT_GS_GLOBAL_BELOW warp groups; 0 when
// the fused kernel already holds the whole table with that many groups, or
// no cluster size fits.
#ifndef TSAT_CLUSTER_DEFAULT
#define TSAT_CLUSTER_DEFAULT 0       // measured slower than the L2 g table / split sequence: opt-in
#endif
int update_cluster_size(int KB, int N, int rec_cap, int optin) {
    if (std::getenv("TSAT_NO_CLUSTER")) return 0;
    if (!TSAT_CLUSTER_DEFAULT && !std::getenv("TSAT_CLUSTER")) return 0;
    auto groups = [&](int n, bool xs) -> long long {
        const size_t gsb = upd_gs_bytes(KB, n), grb = upd_group_bytes(KB, n, rec_cap, upd_recbufs(KB), xs ? 2 : 1, xs);
        return optin > (long long)gsb ? ((long long)optin - (long long)gsb) / (long long)grb : 0;
    };
    if (groups(N, false) >= TSAT_GS_GLOBAL_BELOW) return 0;
    for (int cl = 2; cl <= kMaxCluster; cl *= 2) {
        if (N % (cl * 128)) return 0;
        if (groups(N / cl, true) >= TSAT_GS_GLOBAL_BELOW) return cl;
    }
    return 0;
}

int update_chunk(int KB, int N) {
    const int c = KB == 4 ? 4096 : (KB == 8 ? 2048 : 1024);
    return N < c ? N : c;
}

template <int KB>
static cudaError_t set_update_attrs(int need, int optin) {
    const cudaFuncAttribute attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
    cudaError_t e;
    if ((e = set_max_dyn_smem(k_update<KB, 0>, need, optin)) != cudaSuccess) return e;
    if ((e = set_max_dyn_smem(k_update<KB, 1>, need, optin)) != cudaSuccess) return e;
    if ((e = set_max_dyn_smem(k_update<KB, 2>, need, optin)) != cudaSuccess) return e;
    if ((e = set_max_dyn_smem(k_update<KB, 0, true>, need, optin)) != cudaSuccess) return e;
    if ((e = set_max_dyn_smem(k_update<KB, 0, false, true>, need, optin)) != cudaSuccess) return e;
    if ((e = set_max_dyn_smem(k_update<KB, 2, false, true>, need, optin)) != cudaSuccess) return e;
    if ((e = set_max_dyn_smem(k_update<KB, 0, true, true>, need, optin)) != cudaSuccess) return e;
    if ((e = set_max_dyn_smem(k_update<KB, 2, true, true>, need, optin)) != cudaSuccess) return e;
    if ((e = set_max_dyn_smem(k_update<KB, 0, false, false, 6>, need, optin)) != cudaSuccess) return e;
    if ((e = set_max_dyn_smem(k_update<KB, 0, true, false, 6>, need, optin)) != cudaSuccess) return e;
    if ((e = set_max_dyn_smem(k_update<KB, 2, false, false, 6>, need, optin)) != cudaSuccess) return e;
    if constexpr (TSAT_UPD_NT && KB == 8)
        if ((e = set_max_dyn_smem(k_update<8, 0, false, false, 8, 2048>, need, optin)) != cudaSuccess) return e;
    if ((e = set_max_dyn_smem(k_update<KB, 2, true, false, 6>, need, optin)) != cudaSuccess) return e;
    return set_max_dyn_smem(k_update<KB, 2, true>, need, optin);
}

template <int KB>
static cudaError_t cluster_attrs(int need, int optin, int CL, int threads, int* max_clusters) {
    cudaError_t e;
    auto k0 = k_update<KB, 3, false>;
    auto k1 = k_update<KB, 3, true>;
    if ((e = set_max_dyn_smem(k0, need, optin)) != cudaSuccess) return e;
    if ((e = set_max_dyn_smem(k1, need, optin)) != cudaSuccess) return e;
    if (CL > 8) {
        if ((e = cudaFuncSetAttribute(k0, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess) return e;
        if ((e = cudaFuncSetAttribute(k1, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = need;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaOccupancyMaxActiveClusters(max_clusters, k0, &cfg);
}

// MODE 3 geometry: slice NCH = N / CL per CTA, its g table in shared memory,
// warp groups of the slice, and exactly as many clusters as can be resident
// at once (the static row schedule needs every CTA running).
static cudaError_t configure_update_cluster(StepArgs* a, int optin, int sms) {
    const int KB = a->KB, CL = a->upd_cl, NCH = a->N / CL, NWc = NCH >> 5;
    const int GT = NWc >= 128 ? 128 : (NWc > 32 ? 64 : 32);
    const int nbufs = upd_recbufs(KB);
    const size_t gsb = upd_gs_bytes(KB, NCH), grb = upd_group_bytes(KB, NCH, a->upd_rec_cap, nbufs, 2, true);
    const int max_threads = KB == 4 ? TSAT_UPD_THREADS4 : TSAT_UPD_THREADS8;
    long long ng = optin > (long long)gsb ? ((long long)optin - (long long)gsb) / (long long)grb : 0;
    ng = ng < max_threads / GT ? ng : max_threads / GT;
    if (GT > 32) ng = ng < 15 ? ng : 15;
    if (const char* mg = std::getenv("TSAT_UPD_MAXGROUPS")) {
        const long long x = std::atoll(mg);
        if (x > 0 && x < ng) ng = x;
    }
    if (ng < 1) return cudaErrorInvalidConfiguration;
    a->upd_mode = 0;                  // (0: k_hub still counts the hub rows)
    a->upd_chunk = NCH;
    a->upd_gs_global = 0;
    a->upd_recbufs = nbufs;
    a->upd_GT = GT;
    a->upd_NG = (int)ng;
    a->upd_smem = gsb + (size_t)ng * grb;
    int mc = 0;
    cudaError_t e;
    const int need = (int)a->upd_smem, threads = GT * (int)ng;
    if (KB == 4) e = cluster_attrs<4>(need, optin, CL, threads, &mc);
    else if (KB == 8) e = cluster_attrs<8>(need, optin, CL, threads, &mc);
    else e = cluster_attrs<16>(need, optin, CL, threads, &mc);
    if (e != cudaSuccess) return e;
    if (mc < 1) return cudaErrorInvalidConfiguration;
    a->upd_grid = mc * CL;
    a->upd_prefetch = TSAT_ROW_PREFETCH == 1 ||
                      (TSAT_ROW_PREFETCH == 2 && (double)a->upd_grid * (double)ng * 12.0 * (double)NCH < TSAT_PREFETCH_BYTES);
    if (std::getenv("TSAT_GEOM_VERBOSE"))
        std::fprintf(stderr, "k_update cluster geometry: KB %d N %d CL %d slice %d GT %d groups %lld clusters %d smem %zu\n",
                     KB, a->N, CL, NCH, GT, ng, mc, a->upd_smem);
    return cudaSuccess;
}

cudaError_t configure_update(StepArgs* a) {
    const int N = a->N, KB = a->KB;
    int dev = 0, optin = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    a->num_sms = sms;
    if (a->upd_cl > 1) return configure_update_cluster(a, optin, sms);
    const bool fused = update_fits_fused(KB, N, a->upd_rec_cap, optin);
    a->upd_chunk = fused ? N : update_chunk(KB, N);
    a->upd_gs_global = fused ? 0 : 1;
    const int NWc = a->upd_chunk >> 5;
    const int GT = NWc >= 128 ? 128 : (NWc > 32 ? 64 : 32);
    if (fused) {
        // the batch's g table in shared memory leaves few warp groups for
        // large batches (N = 8192: 128 KB of table, 2 groups); read it through
        // L1 / L2 instead when that buys at least twice the groups
        const size_t gsb0 = upd_gs_bytes(KB, N), grb0 = upd_group_bytes(KB, N, a->upd_rec_cap, upd_recbufs(KB), a->peer ? 2 : 1);
        const long long ng_s = optin > (long long)gsb0 ? ((long long)optin - (long long)gsb0) / (long long)grb0 : 0;
        const long long ng_g = (long long)optin / (long long)grb0;
        if (ng_s < TSAT_GS_GLOBAL_BELOW && ng_g >= 2 * ng_s && !std::getenv("TSAT_NO_GS_GLOBAL")) a->upd_gs_global = 1;
    }
    const size_t gsb = (fused && !a->upd_gs_global) ? upd_gs_bytes(KB, N) : 0;
    const int max_threads = KB == 4 ? (a->peer ? TSAT_UPD_THREADS4P : ((a->upd_cw6 && !a->upd_gs_global) ? TSAT_UPD_THREADS4C6 : TSAT_UPD_THREADS4))
                                    : TSAT_UPD_THREADS8;   // register budget (launch bounds)
    auto groups = [&](int nbufs) {
        const size_t grb = upd_group_bytes(KB, a->upd_chunk, a->upd_rec_cap, nbufs, a->peer ? 2 : 1);
        long long ng = optin > (long long)gsb ? ((long long)optin - (long long)gsb) / (long long)grb : 0;
        ng = ng < max_threads / GT ? ng : max_threads / GT;
        if (GT > 32) ng = ng < 15 ? ng : 15;      // named barriers 1..15 (warp groups use __syncwarp)
        return ng;
    };
    // (upd_recbufs: measured c4 7 -> 8 groups with one buffer, k_update -11 %;
    // c2 / c3 are register-bound, and two buffers are faster there, c2 +4 %)
    const int nbufs = upd_recbufs(KB);
    long long ng = groups(nbufs);
    if (const char* mg = std::getenv("TSAT_UPD_MAXGROUPS")) {   // A/B hook: cap the warp groups per CTA
        const long long x = std::atoll(mg);
        if (x > 0 && x < ng) ng = x;
    }
    const size_t grb = upd_group_bytes(KB, a->upd_chunk, a->upd_rec_cap, nbufs, a->peer ? 2 : 1);
    if (ng < 1) return cudaErrorInvalidConfiguration;
    a->upd_recbufs = nbufs;
    if (std::getenv("TSAT_GEOM_VERBOSE"))
        std::fprintf(stderr, "k_update geometry: KB %d N %d GT %d groups %lld recbufs %d rec_cap %d smem %zu\n", KB, N, GT, ng,
                     nbufs, a->upd_rec_cap, gsb + (size_t)ng * grb);
    a->upd_mode = 0;
    a->upd_GT = GT;
    a->upd_NG = (int)ng;
    a->upd_smem = gsb + (size_t)ng * grb;
    a->upd_grid = sms;
    {
        const double fl = (double)sms * (double)ng * 12.0 * (double)a->upd_chunk;   // rows in flight (bytes)
        a->upd_prefetch = (TSAT_ROW_PREFETCH == 1 || (TSAT_ROW_PREFETCH == 2 && fl < TSAT_PREFETCH_BYTES)) ? 1
                        : (TSAT_PREFETCH_THETA && fl / 3.0 < TSAT_PREFETCH_BYTES) ? 2 : 0;    // 2: theta only
    }
    // test hook: several ranks' persistent kernels sharing one GPU must be
    // co-resident, so each may be limited to a part of the SMs
    if (const char* g = std::getenv("TSAT_UPD_GRID")) {
        const int x = std::atoi(g);
        if (x > 0 && x < sms) a->upd_grid = x;
    }
    // the attribute is a process-wide per-function limit, raised to this
    // launch's need and never lowered (set_max_dyn_smem)
    const int smem = (int)a->upd_smem;
    if (KB == 4) return set_update_attrs<4>(smem, optin);
    if (KB == 8) return set_update_attrs<8>(smem, optin);
    return set_update_attrs<16>(smem, optin);
}

cudaError_t launch_hub(const StepArgs& a, const uint32_t* Acur, cudaStream_t st) {
    if (a.n_hub_sc == 0) return cudaGetLastError();
    const int NW = a.N >> 5;
    dim3 grid(a.n_hub_sc, (NW + 31) / 32);            // super-chunks on x (no 65535 limit)
    const bool bat = a.upd_rec != a.occ_rec;
    if (a.KB == 4) {
        if (bat) k_hub<4, true><<<grid, 32, 0, st>>>(a, Acur);
        else k_hub<4, false><<<grid, 32, 0, st>>>(a, Acur);
    } else if (a.KB == 8) {
        if (bat) k_hub<8, true><<<grid, 32, 0, st>>>(a, Acur);
        else k_hub<8, false><<<grid, 32, 0, st>>>(a, Acur);
    } else {
        k_hub<16, true><<<grid, 32, 0, st>>>(a, Acur);
    }
    return cudaGetLastError();
}

template <int KB, bool GSG>
static cudaError_t launch_update_kbg(const StepArgs& a, const uint32_t* Acur, uint32_t* Anext, const StepScalars* sc,
                                    cudaStream_t st) {
    const bool mag = a.mc.normalize == 3;
    const dim3 g(a.upd_grid), b(a.upd_GT * a.upd_NG);
    const size_t sm = a.upd_smem;
    if (a.upd_cl > 1) {                          // MODE 3: cluster-split rows
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = g;
        cfg.blockDim = b;
        cfg.dynamicSmemBytes = sm;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = a.upd_cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return a.mc.normalize == 3 ? cudaLaunchKernelEx(&cfg, k_update<KB, 3, true>, a, Acur, Anext, sc)
                                   : cudaLaunchKernelEx(&cfg, k_update<KB, 3, false>, a, Acur, Anext, sc);
    }
    if (a.peer) {
        if (!GSG && a.upd_cw6) {                  // 6-plane counters (fewer registers under the exchange state)
            if (mag) k_update<KB, 2, true, false, 6><<<g, b, sm, st>>>(a, Acur, Anext, sc);
            else k_update<KB, 2, false, false, 6><<<g, b, sm, st>>>(a, Acur, Anext, sc);
            return cudaGetLastError();
        }
        if (mag) k_update<KB, 2, true, GSG><<<g, b, sm, st>>>(a, Acur, Anext, sc);
        else k_update<KB, 2, false, GSG><<<g, b, sm, st>>>(a, Acur, Anext, sc);
        return cudaGetLastError();
    }
    if constexpr (TSAT_UPD_NT && KB == 8) {      // compile-time batch size of c4's shape
        if (!mag && !GSG && a.N == 2048)
            return launch_maybe_pdl(a.pdl, k_update<8, 0, false, false, 8, 2048>, g, b, sm, st, a, Acur, Anext, sc);
    }
    if (!GSG && a.upd_cw6)                       // K <= 3, every row within 6-bit counters
        return mag ? launch_maybe_pdl(a.pdl, k_update<KB, 0, true, false, 6>, g, b, sm, st, a, Acur, Anext, sc)
                   : launch_maybe_pdl(a.pdl, k_update<KB, 0, false, false, 6>, g, b, sm, st, a, Acur, Anext, sc);
    return mag ? launch_maybe_pdl(a.pdl, k_update<KB, 0, true, GSG>, g, b, sm, st, a, Acur, Anext, sc)
               : launch_maybe_pdl(a.pdl, k_update<KB, 0, false, GSG>, g, b, sm, st, a, Acur, Anext, sc);
}
template <int KB>
static cudaError_t launch_update_kb(const StepArgs& a, const uint32_t* Acur, uint32_t* Anext, const StepScalars* sc,
                                   cudaStream_t st) {
    return a.upd_gs_global ? launch_update_kbg<KB, true>(a, Acur, Anext, sc, st)
                           : launch_update_kbg<KB, false>(a, Acur, Anext, sc, st);
}

cudaError_t launch_update(const StepArgs& a, const uint32_t* Acur, uint32_t* Anext, const StepScalars* sc,
                          cudaStream_t st) {
    if (a.V == 0) return cudaGetLastError();
    if (a.KB == 4) return launch_update_kb<4>(a, Acur, Anext, sc, st);
    if (a.KB == 8) return launch_update_kb<8>(a, Acur, Anext, sc, st);
    return launch_update_kb<16>(a, Acur, Anext, sc, st);
}

// Phase A of the sharded iteration (always the persistent kernel: the
// sharded path requires the fused geometry, see configure_update).
cudaError_t launch_update_a(const StepArgs& a, const uint32_t* Acur, const StepScalars* sc, cudaStream_t st) {
    if (a.V == 0) return cudaGetLastError();
    const int threads = a.upd_GT * a.upd_NG;
    if (a.KB == 4) k_update<4, 1><<<a.upd_grid, threads, a.upd_smem, st>>>(a, Acur, nullptr, sc);
    else if (a.KB == 8) k_update<8, 1><<<a.upd_grid, threads, a.upd_smem, st>>>(a, Acur, nullptr, sc);
    else k_update<16, 1><<<a.upd_grid, threads, a.upd_smem, st>>>(a, Acur, nullptr, sc);
    return cudaGetLastError();
}

}  // namespace tsat
