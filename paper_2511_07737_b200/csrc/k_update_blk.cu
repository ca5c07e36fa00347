// k_update_blk.cu - rows (a7) STE backward, (a8) Eq. 5 Jacobian, (a9) AdamW +
// re-binarisation for small candidate shards (§3.2 l.189-191, l.226;
// §4.1 l.255-269; the shard sizes of §8(e)'s strong scaling: N = 128 .. 512
// candidates per GPU, e.g. BASELINE c3's 1024 candidates over 2-8 B200).
//
// The per-row kernel (k_update.cu) maps a warp's lanes to the 32-candidate
// words of ONE row: with N = 128 only 4 of 32 lanes gather, every row pays
// its own L2/HBM round trips, barriers and scheduler atomic, and 1M rows
// cost 13 us each per warp group.  Here a work item is a BLOCK of RB =
// 32 / (N/32) consecutive rows, one warp per group:
//   1. gather: lane = (row r = lane / NW, word w = lane % NW), so all lanes
//      count occurrences at once (same bit-sliced counters and transposes);
//   2. the block's theta / m / v rows are contiguous ([V][N] layout), so
//      passes 3a / 3b stream RB * N floats as ONE float4 stream (one-ahead
//      loads cross row boundaries; one L2 bulk prefetch per array);
//      per-row values (J_v, Q_v, max |theta|) are warp reductions at the
//      row's last 128-candidate iteration;
//   3. peer path (MODE 2): the block's RB J partials are sent together and
//      awaited together; its Q partials are sent after pass 3b and the block
//      is finished one block later (as the per-row kernel does per row).
// Arithmetic is the per-row kernel's, operation for operation, so results
// are bit-identical to it (and to the oracle).
#include "peer.cuh"
#include "upd_common.cuh"

namespace tsat {

namespace {
// Per-row values of the current block (lane r writes row r); pq / pm2 belong
// to the pending block of the peer path (finished one block late).
struct BlkRow {
    double rho;
    long long jt, qt, pq;
    float rhof, ncf, p2, m2, pm2;
    int hub, dsum, jvalid, s;
    int guard;
    int roff, nrec, npos, nneg;      // staged records: offset in the block buffer, words, occurrences by sign
    int v, pv;                       // the row (variable) of this block slot; of the pending block's slot
};
// A row's values for the next block, prefetched into the registers of lane r
// while the current block streams (their L2 latency leaves the critical path).
struct RowPre {
    int2 pn;
    int v, hub, guard, roff, nrec, rbeg;
    double rho;
};

__host__ __device__ inline size_t blk_group_bytes(int KB, int N, int RB, int cap, int nbufs) {
    const int NDW = KB == 4 ? 1 : 2;
    return align16((size_t)NDW * RB * upd_dpk_words(N) * 4) + nbufs * align16((size_t)cap * 4) +
           align16((size_t)4 * RB * (N >> 5) * 4) + align16(sizeof(BlkRow) * RB) + 16;
}
}  // namespace

// Warp sum of an int64 whose magnitude is below 2^57 (J and Q partials of a
// lane: 4 terms, each below 2^61 / N with N >= 128, resp. 2^46): three 21-bit
// limbs through the warp-reduce unit (REDUX), exact.
__device__ __forceinline__ long long warp_sum_redux(long long x) {
    const unsigned lo = (unsigned)(x & 0x1FFFFF), mid = (unsigned)((x >> 21) & 0x1FFFFF);
    const int hi = (int)(x >> 42);
    const unsigned slo = __reduce_add_sync(0xffffffffu, lo), smid = __reduce_add_sync(0xffffffffu, mid);
    const int shi = __reduce_add_sync(0xffffffffu, hi);
    return ((long long)shi << 42) + ((long long)smid << 21) + (long long)slo;
}
// Warp max of non-negative floats (their bit patterns order like the values).
__device__ __forceinline__ float warp_max_redux(float x) {
    return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(x)));
}

int update_block_rows(int N) {
    if (N <= 0 || N % 128 != 0) return 1;      // 128-candidate iterations never straddle a row
    const int NW = N >> 5;
    if (NW >= 32) return 1;
    const int rb = 32 / NW;
    return rb >= 2 ? rb : 1;
}

// NT > 0: the shard size as a compile-time constant (N = 128 / 256 / 512, the
// W = 8 / 4 / 2 shares of c3's fixed batch): the block geometry (words per row,
// rows per block, iterations per row, lane -> (row, word)) folds into
// constants instead of living in registers.
template <int KB, int MODE, bool MAG, int NT = 0>
__global__ void __launch_bounds__(KB == 4 ? (MODE == 2 ? TSAT_UPD_THREADS4P : TSAT_UPD_THREADS4) : TSAT_UPD_THREADS8, 1)
    k_update_blk(StepArgs a, const uint32_t* __restrict__ Acur, uint32_t* __restrict__ Anext,
                 const StepScalars* __restrict__ sc) {
    constexpr int NP = (KB == 4) ? 2 : (KB == 8 ? 3 : 4);
    constexpr int NCTR = KB - 1;
    constexpr int NDW = KB == 4 ? 1 : 2;
    constexpr int nbufs = upd_recbufs(KB);
    extern __shared__ __align__(16) unsigned char smem[];
    const int N = NT ? NT : a.N, NW = N >> 5, RB = NT ? 32 / (NT >> 5) : a.upd_RB;
    const int ipr = N >> 7;                              // 128-candidate iterations per row
    const size_t dpkw = upd_dpk_words(N), dplane = (size_t)RB * dpkw;
    float* gs = reinterpret_cast<float*>(smem);
    const int grp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cap = a.upd_blk_cap;
    unsigned char* gb = smem + upd_gs_bytes(KB, N) + (size_t)grp * blk_group_bytes(KB, N, RB, cap, nbufs);
    uint32_t* dpk = reinterpret_cast<uint32_t*>(gb);
    uint32_t* rec = reinterpret_cast<uint32_t*>(gb + align16((size_t)NDW * dplane * 4));
    const size_t recw = align16((size_t)cap * 4) / 4;
    uint32_t* pl0 = rec + nbufs * recw;                  // [parity][pos | neg][RB * NW]
    BlkRow* rp = reinterpret_cast<BlkRow*>(reinterpret_cast<unsigned char*>(pl0) + align16((size_t)16 * RB * NW));
    int* slot = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(rp) + align16(sizeof(BlkRow) * RB));
    const int nitems = (a.V + RB - 1) / RB;
    const bool uni3 = a.uniform_len && a.mc.K == 3 && KB == 4;
    const unsigned long long pol = plane_policy(planes_fit_l2(a.V, NW));
    const int gr = lane / NW, gw = lane - gr * NW;       // gather lane -> (row of the block, word)

    pdl_wait();
    pdl_trigger();
    for (int i = threadIdx.x * 4; i < KB * N; i += blockDim.x * 4)
        *reinterpret_cast<float4*>(gs + i) = *reinterpret_cast<const float4*>(a.gtab + i);
    if (lane == 0) slot[1] = atomicAdd(&a.ds->row_counter, 1);
    const long long t = sc->t;
    __shared__ unsigned long long pscal[3];
    if (MODE == 2 && threadIdx.x == 0) {
        const unsigned long long own[4] = {~a.ds->best_key, a.ds->gmax_bits,
                                           (unsigned long long)a.ds->thmax_bits[t & 1],
                                           (unsigned long long)a.ds->loss_fx};
        unsigned long long x[4];
        peer_recv_scalars(a.px, sc->xgen, a.ds, own, x);
        pscal[0] = ~x[0];
        pscal[1] = a.px.exchange_rows ? x[1] : a.ds->gmax_bits;
        pscal[2] = a.px.exchange_rows ? x[2] : (unsigned long long)a.ds->thmax_bits[t & 1];
        if (blockIdx.x == 0) {
            const int bu = (int)(pscal[0] >> 32);
            const long long bi = (long long)(pscal[0] & 0xffffffffull);
            if (bu == 0 && a.ds->sol_step < 0) { a.ds->sol_step = t; a.ds->sol_idx = bi; }
            const double loss = -((double)(long long)x[3] * a.mc.loss_unscale);
            a.ds->loss = loss;
            a.ds->info_t = t + 1;
            a.ds->info_best_unsat = bu;
            a.ds->info_best_idx = bi;
            a.ds->info_loss = loss;
        }
    }
    __syncthreads();

    const double gmax = __longlong_as_double((long long)(MODE == 2 ? pscal[1] : a.ds->gmax_bits));
    const float thmax = __uint_as_float(MODE == 2 ? (unsigned)pscal[2] : a.ds->thmax_bits[t & 1]);
    const float wdf = sc->wdf, a1 = sc->a1, b2f = sc->b2f, a2 = sc->a2, nss = sc->nss, rbc2 = sc->rbc2,
                epsf = sc->epsf, nz = sc->nz, mkeep = sc->mkeep;
    const MethodConsts& mc = a.mc;

    // records of the block's non-hub rows, back to back -> buf
    // (the rows' record ranges come from the RowPre values lane r holds)
    auto stage = [&](int nr, uint32_t* buf, bool async, const RowPre& P) {
        for (int r = 0; r < nr; ++r) {
            if (__shfl_sync(0xffffffffu, P.hub, r) >= 0) continue;
            const unsigned b = (unsigned)__shfl_sync(0xffffffffu, P.rbeg, r);
            const unsigned len = (unsigned)__shfl_sync(0xffffffffu, P.nrec, r);
            const unsigned off = (unsigned)__shfl_sync(0xffffffffu, P.roff, r);
            for (unsigned i = lane; i < len; i += 32) {
                if (async) cp_async4(buf + off + i, a.upd_rec + b + i);
                else buf[off + i] = a.upd_rec[b + i];
            }
        }
    };
    // Rows of a block are complete once their global Q are known: bit planes
    // (sign(d) = sign(Q), R3), Eq. 5 statistics, max |theta|, first-model bits.
    auto finish_block = [&](int nr, const uint32_t* pl, bool pending) {
        for (int idx = lane; idx < nr * NW; idx += 32) {
            const int r = idx / NW, w = idx - r * NW;
            const long long Qg = pending ? rp[r].pq : rp[r].qt;
            const int vr = pending ? rp[r].pv : rp[r].v;
            const bool dpos = !mc.normalize || Qg >= 0;
#if TSAT_ANEXT_CS
            __stcs(Anext + (size_t)vr * NW + w, dpos ? pl[idx] : pl[RB * NW + idx]);
#else
            Anext[(size_t)vr * NW + w] = dpos ? pl[idx] : pl[RB * NW + idx];
#endif
        }
        float m2 = 0.0f;
        if (lane < nr) {
            const int vr = pending ? rp[lane].pv : rp[lane].v;
            const long long Qg = pending ? rp[lane].pq : rp[lane].qt;
            m2 = pending ? rp[lane].pm2 : rp[lane].m2;
            double dn, rhon;
            unsigned char gn;
            row_finish(Qg, mc, &dn, &rhon, &gn);
            a.rowQ[vr] = Qg; a.rowD[vr] = dn; a.rowRho[vr] = rhon; a.rowGuard[vr] = gn;
            const unsigned long long bk = MODE == 2 ? pscal[0] : a.ds->best_key;
            if ((bk >> 32) == 0ull && (a.ds->sol_step < 0 || a.ds->sol_step == t)) {          // first model (A22)
                const long long idx = (long long)(bk & 0xffffffffull) - mc.n0;
                if (idx >= 0 && idx < N)
                    a.sol[vr] = (unsigned char)((Acur[(size_t)vr * NW + (idx >> 5)] >> (idx & 31)) & 1u);
            }
        }
        m2 = warp_maxf(m2);
        if (lane == 0) atomicMax(&a.ds->thmax_bits[(t + 1) & 1], __float_as_uint(m2));
    };

    // row values of the block's row r for lane r (< nr): occurrence counts,
    // hub index, Eq. 5 statistics of the evaluated state, and the row's
    // record offset within the block's staging buffer (non-hub rows back to back)
    // (the block's rows are item RB ... item RB + nr - 1, or a.blk_rows[item RB ...]: rows grouped by their
    // gather length on the host, so the lanes of a warp finish together)
    // (called by the whole warp: the offsets are an exclusive warp prefix sum
    // of the rows' staged lengths, one load chain per lane)
    auto fetch_row = [&](int item, int nr, RowPre& P) {
        unsigned mine = 0;
        if (lane < nr) {
            const int v = a.blk_rows ? a.blk_rows[(size_t)item * RB + lane] : item * RB + lane;
            P.v = v;
            P.pn = a.occ_pn[v];
            P.hub = a.hub_of[v];
            P.rho = a.rowRho[v];
            P.guard = a.rowGuard[v];
            P.rbeg = (int)a.upd_ptr[v];
            P.nrec = (int)(a.upd_ptr[v + 1] - a.upd_ptr[v]);
            mine = P.hub < 0 ? (unsigned)P.nrec : 0u;
        }
        unsigned incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned x = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += x;
        }
        if (lane < nr) P.roff = (int)(incl - mine);
    };
    RowPre pre{};
    bool pending = false;
    int pend_nr = 0;
    int item = slot[1];
    if (item < nitems) {
        fetch_row(item, min(RB, a.V - item * RB), pre);
        stage(min(RB, a.V - item * RB), rec, false, pre);
    }
    __syncwarp();
    int it = 0;
    for (; item < nitems; ++it) {
        const int nr = min(RB, a.V - item * RB);
        uint32_t* rb_cur = rec + (size_t)(nbufs == 2 ? (it & 1) : 0) * recw;
        uint32_t* rb_nxt = rec + (size_t)(nbufs == 2 ? ((it + 1) & 1) : 0) * recw;
        uint32_t* pl = pl0 + (MODE == 2 ? (size_t)(it & 1) * 2 * RB * NW : 0);
        if (lane == 0) slot[it & 1] = atomicAdd(&a.ds->row_counter, 1);
        if (lane < nr) {                                   // this block's row values (prefetched)
            const uint32_t bytes = (uint32_t)N * 4u;
            prefetch_l2(a.theta + (size_t)pre.v * N, bytes);
            prefetch_l2(a.m + (size_t)pre.v * N, bytes);
            prefetch_l2(a.v + (size_t)pre.v * N, bytes);
            BlkRow& R = rp[lane];
            R.v = pre.v;
            R.hub = pre.hub;
            R.dsum = pre.pn.y - pre.pn.x;
            R.rho = pre.rho;
            R.guard = pre.guard;
            R.roff = pre.roff;
            R.nrec = pre.nrec;
            R.npos = pre.pn.x;
            R.nneg = pre.pn.y;
            int s;
            float p2;
            R.jvalid = jscale(mc.Nnorm, pre.pn.x + pre.pn.y, gmax, thmax, &s, &p2) ? 1 : 0;
            R.s = s;
            R.p2 = p2;
        }
        __syncwarp();

        // ---- 1+2: gather (lane = row x word), transpose to bytes (KB = 16: all rows are hubs)
        if constexpr (KB <= 8) if (gr < nr) {
            const int v = rp[gr].v;
            if (rp[gr].hub < 0) {
                const uint32_t* rbase = rb_cur + rp[gr].roff;
                auto recf = [&](unsigned i) { return rbase[i]; };
                const uint32_t own = __ldg(Acur + (size_t)v * NW + gw);
                uint32_t cnt[NCTR][kCtr];
                if (uni3) {
                    count_uni3<NCTR, kCtr, TSAT_BLK_PIPE != 0>(cnt, recf, (unsigned)rp[gr].nneg, (unsigned)rp[gr].npos, own,
                                                               Acur, (unsigned)NW, (unsigned)gw, pol);
                } else {
                    count_batched<NP, NCTR, kCtr>(cnt, recf, (unsigned)rp[gr].nrec, own, Acur, (unsigned)NW,
                                                  (unsigned)gw, pol);
                }
#pragma unroll 1
                for (int blk = 0; blk < (KB == 8 ? 2 : 1); ++blk) {
                    uint32_t T[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int r = i / kCtr;
                        const uint32_t lo = (r < NCTR && r < 4) ? cnt[r][i % kCtr] : 0u;
                        const uint32_t hi = (4 + r < NCTR) ? cnt[4 + r][i % kCtr] : 0u;
                        T[i] = blk ? hi : lo;
                    }
                    transpose32(T);
                    uint32_t* dst = dpk + blk * dplane + (size_t)gr * dpkw + 33 * gw;
#pragma unroll
                    for (int j = 0; j < 32; ++j) dst[j] = T[j];
                }
            }
        }
        if (MODE == 2 && pending && lane < pend_nr)          // previous block's Q, sent a block ago
            rp[lane].pq = peer_row_recv(a.px, 1, rp[lane].pv, sc->xgen, a.ds, rp[lane].pq);
        __syncwarp();
        const int item_next = slot[it & 1];
        const int nrn = item_next < nitems ? min(RB, a.V - item_next * RB) : 0;
        if (nrn > 0) fetch_row(item_next, nrn, pre);                 // the next block's row values
        auto stage_next = [&]() {
            if (nrn > 0) stage(nrn, rb_nxt, true, pre);
            cp_async_commit();
        };
        if (nbufs == 1) stage_next();
        if (MODE == 2 && pending) {
            finish_block(pend_nr, pl0 + (size_t)((it + 1) & 1) * 2 * RB * NW, true);
            pending = false;
        }

        // ---- 3a: G -> dpk, J partial per row (flat float4 stream over the block)
        {
            // one float4 stream over the block's rows: the one-ahead load
            // crosses to the next row of the block
            auto rowp = [&](const float* base, int r) { return base + (size_t)rp[r].v * N + 4 * lane; };
            float4 th_nx = *reinterpret_cast<const float4*>(rowp(a.theta, 0));
            long long I = 0;
            int k = 0;                                           // flat 128-candidate iteration of the block
            for (int r = 0; r < nr; ++r) {
              const int hub = rp[r].hub, dsum = rp[r].dsum;
              const float p2 = rp[r].p2;
              const bool jv = rp[r].jvalid != 0;
              const float* trn = r + 1 < nr ? rowp(a.theta, r + 1) : nullptr;
              const float* trc = rowp(a.theta, r);
              for (int kk = 0; kk < ipr; ++kk, ++k) {
                const int n = kk * 128 + 4 * lane;
                const float4 th4 = th_nx;
                if (kk + 1 < ipr) th_nx = *reinterpret_cast<const float4*>(trc + (kk + 1) * 128);
                else if (trn) th_nx = *reinterpret_cast<const float4*>(trn);
                const float th[4] = {th4.x, th4.y, th4.z, th4.w};
                float4 g4[KB];
#pragma unroll
                for (int q = 0; q < KB; ++q) g4[q] = *reinterpret_cast<const float4*>(gs + (size_t)q * N + n);
                uint32_t* dp = dpk + (size_t)r * dpkw + n + (n >> 5);
                float Gq[4];
                if (KB > 8 || hub >= 0) {
                    int* hubrow = a.hubD + (size_t)hub * NCTR * N;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        float gq[KB];
#pragma unroll
                        for (int b = 0; b < KB; ++b) gq[b] = q == 0 ? g4[b].x : q == 1 ? g4[b].y : q == 2 ? g4[b].z : g4[b].w;
                        Gq[q] = fold_ints<KB>(hubrow, N, n + q, dsum, gq);
                    }
#pragma unroll
                    for (int b = 0; b < KB - 1; ++b)
                        *reinterpret_cast<int4*>(hubrow + (size_t)b * N + n) = make_int4(0, 0, 0, 0);
                } else if constexpr (KB <= 8) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        float dA[KB], dB[KB];
                        fold_counts<KB>(dA, dp[2 * h], KB == 8 ? dp[dplane + 2 * h] : 0u, dsum);
                        fold_counts<KB>(dB, dp[2 * h + 1], KB == 8 ? dp[dplane + 2 * h + 1] : 0u, dsum);
                        float2 G2 = make_float2(0.0f, 0.0f);
#pragma unroll
                        for (int b = 0; b < KB; ++b)
                            G2 = __ffma2_rn(make_float2(dA[b], dB[b]),
                                            h == 0 ? make_float2(g4[b].x, g4[b].y) : make_float2(g4[b].z, g4[b].w), G2);
                        Gq[2 * h] = G2.x;
                        Gq[2 * h + 1] = G2.y;
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    dp[q] = __float_as_uint(Gq[q]);
                    if (jv) I += jterm(Gq[q], th[q], p2);
                }
              }
              I = warp_sum_redux(I);                             // the row's J partial
              if (lane == 0) rp[r].jt = I;
              I = 0;
            }
        }
        __syncwarp();
        if (MODE == 2 && a.px.exchange_rows) {                   // the block's J_v over all ranks
            if (lane < nr) peer_row_send(a.px, 0, rp[lane].v, rp[lane].jt, sc->xgen);
            if (lane < nr) rp[lane].jt = peer_row_recv(a.px, 0, rp[lane].v, sc->xgen, a.ds, rp[lane].jt);
        }
        if (nbufs == 2) stage_next();
        if (lane < nr) {
            BlkRow& R = rp[lane];
            double c = 0.0;
            if (mc.normalize && !R.guard) {
                const double J = R.jvalid ? times_pow2((double)R.jt, -R.s) : 0.0;
                c = J / (double)mc.Nnorm;
                c = c * R.rho;
                c = c * R.rho;
            }
            R.rhof = __double2float_rn(R.rho);
            R.ncf = -__double2float_rn(c);
        }
        __syncwarp();

        // ---- 3b: grad, AdamW, next-state statistics and sign planes (flat stream)
        {
            constexpr bool mag = MAG;
            size_t o0 = (size_t)rp[0].v * N + 4 * lane;          // element offset of this lane in row 0
            float4 thn = ld_last(a.theta + o0), mn4 = ld_last(a.m + o0), vn4 = ld_last(a.v + o0);
            long long Qn = 0;
            float mx = 0.0f;
            int k = 0;
            for (int r = 0; r < nr; ++r) {
              const float rhof = rp[r].rhof, ncf = rp[r].ncf;
              const int v = rp[r].v;
              const size_t orow = (size_t)v * N + 4 * lane;
              const size_t onext = r + 1 < nr ? (size_t)rp[r + 1].v * N + 4 * lane : 0;
              for (int kk = 0; kk < ipr; ++kk, ++k) {
                const int n = kk * 128 + 4 * lane;
                const size_t e = orow + (size_t)kk * 128;        // this lane's 4 candidates of row v
                const float4 th4 = thn, m4 = mn4, v4 = vn4;
                if (kk + 1 < ipr || r + 1 < nr) {               // one ahead, across the block's rows
                    const size_t en = kk + 1 < ipr ? e + 128 : onext;
                    thn = ld_last(a.theta + en);
                    mn4 = ld_last(a.m + en);
                    vn4 = ld_last(a.v + en);
                }
                float th[4] = {th4.x, th4.y, th4.z, th4.w};
                float mm[4] = {m4.x, m4.y, m4.z, m4.w};
                float vv[4] = {v4.x, v4.y, v4.z, v4.w};
                const uint32_t* dp = dpk + (size_t)r * dpkw + n + (n >> 5);
                float gg[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) gg[q] = __fmaf_rn(__uint_as_float(dp[q]), rhof, jac_addend(ncf, th[q], mag));
                unsigned pnib = 0, nnib = 0;
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
                        xs0 = xs0 + nz * noise_xi(mc.seed, mc.n0 + n + 2 * h, v, t);
                        xs1 = xs1 + nz * noise_xi(mc.seed, mc.n0 + n + 2 * h + 1, v, t);
                    }
                    const float xs[2] = {xs0, xs1};
                    const float2 q2 = __fmul2_rn(mag ? make_float2(fabsf(xs0), fabsf(xs1)) : make_float2(xs0, xs1),
                                                 make_float2(4294967296.0f, 4294967296.0f));
                    Qn += __float2ll_rn(q2.x) + __float2ll_rn(q2.y);
#pragma unroll
                    for (int f = 0; f < 2; ++f) {
                        const int q = 2 * h + f;
                        const float x = xs[f];
                        th[q] = x;
                        mm[q] = f ? mn2.y : mn2.x;
                        vv[q] = f ? vn2.y : vn2.x;
                        mx = fmaxf(mx, fabsf(x));
                        pnib |= (x > 0.0f ? 1u : 0u) << q;
                        nnib |= (x < 0.0f ? 1u : 0u) << q;
                    }
                }
                st_stream(a.theta + e, make_float4(th[0], th[1], th[2], th[3]));
                st_stream(a.m + e, make_float4(mm[0], mm[1], mm[2], mm[3]));
                st_stream(a.v + e, make_float4(vv[0], vv[1], vv[2], vv[3]));
                unsigned pw = pnib << (4 * (lane & 7)), nw = nnib << (4 * (lane & 7));
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) {
                    pw |= __shfl_xor_sync(0xffffffffu, pw, o);
                    nw |= __shfl_xor_sync(0xffffffffu, nw, o);
                }
                if ((lane & 7) == 0) {
                    pl[r * NW + (n >> 5)] = pw;
                    pl[RB * NW + r * NW + (n >> 5)] = nw;
                }
              }
              Qn = warp_sum_redux(Qn);                           // the row's Q partial and max |theta|
              mx = warp_max_redux(mx);
              if (lane == 0) { rp[r].qt = Qn; rp[r].m2 = mx; }
              Qn = 0;
              mx = 0.0f;
            }
        }
        cp_async_wait_all();                                     // next block's records visible after this
        __syncwarp();
        if (MODE == 2 && a.px.exchange_rows) {
            // the block's Q_{t+1,v} over all ranks: send now, finish after the next block's gather
            if (lane < nr) {
                peer_row_send(a.px, 1, rp[lane].v, rp[lane].qt, sc->xgen);
                rp[lane].pq = rp[lane].qt;
                rp[lane].pm2 = rp[lane].m2;
                rp[lane].pv = rp[lane].v;
            }
            pending = true;
            pend_nr = nr;
        } else {
            finish_block(nr, pl, false);
        }
        __syncwarp();
        item = item_next;
    }
    if (MODE == 2 && pending) {
        if (lane < pend_nr) rp[lane].pq = peer_row_recv(a.px, 1, rp[lane].pv, sc->xgen, a.ds, rp[lane].pq);
        __syncwarp();
        finish_block(pend_nr, pl0 + (size_t)((it + 1) & 1) * 2 * RB * NW, true);
    }
}

#ifndef TSAT_BLK_NT
#define TSAT_BLK_NT 1                // compile-time shard sizes 128 / 256 / 512 for KB <= 8 (c3 N = 128: k_update -9 %)
#endif
template <int KB, int NT>
static cudaError_t set_blk_attrs_nt(int need, int optin) {
    cudaError_t e;
    if ((e = set_max_dyn_smem(k_update_blk<KB, 0, false, NT>, need, optin)) != cudaSuccess) return e;
    if ((e = set_max_dyn_smem(k_update_blk<KB, 2, false, NT>, need, optin)) != cudaSuccess) return e;
    if ((e = set_max_dyn_smem(k_update_blk<KB, 0, true, NT>, need, optin)) != cudaSuccess) return e;
    return set_max_dyn_smem(k_update_blk<KB, 2, true, NT>, need, optin);
}
template <int KB>
static cudaError_t set_blk_attrs(int need, int optin) {
    cudaError_t e;
    if (TSAT_BLK_NT && KB <= 8) {
        if ((e = set_blk_attrs_nt<KB, 128>(need, optin)) != cudaSuccess) return e;
        if ((e = set_blk_attrs_nt<KB, 256>(need, optin)) != cudaSuccess) return e;
        if ((e = set_blk_attrs_nt<KB, 512>(need, optin)) != cudaSuccess) return e;
    }
    return set_blk_attrs_nt<KB, 0>(need, optin);
}

cudaError_t configure_update_blk(StepArgs* a) {
    const int N = a->N, KB = a->KB, RB = a->upd_RB;
    int dev = 0, optin = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    a->num_sms = sms;
    const int nbufs = upd_recbufs(KB);
    const size_t gsb = upd_gs_bytes(KB, N), grb = blk_group_bytes(KB, N, RB, a->upd_blk_cap, nbufs);
    const int max_threads = KB == 4 ? (a->peer ? TSAT_UPD_THREADS4P : TSAT_UPD_THREADS4) : TSAT_UPD_THREADS8;
    long long ng = optin > (long long)gsb ? ((long long)optin - (long long)gsb) / (long long)grb : 0;
    if (ng > max_threads / 32) ng = max_threads / 32;
    if (ng < 1) return cudaErrorInvalidConfiguration;
    if (std::getenv("TSAT_GEOM_VERBOSE"))
        std::fprintf(stderr, "k_update_blk geometry: KB %d N %d RB %d groups %lld cap %d smem %zu\n", KB, N, RB, ng,
                     a->upd_blk_cap, gsb + (size_t)ng * grb);
    a->upd_mode = 0;
    a->upd_chunk = N;
    a->upd_gs_global = 0;
    a->upd_recbufs = nbufs;
    a->upd_GT = 32;
    a->upd_NG = (int)ng;
    a->upd_smem = gsb + (size_t)ng * grb;
    a->upd_grid = sms;
    if (const char* g = std::getenv("TSAT_UPD_GRID")) {
        const int x = std::atoi(g);
        if (x > 0 && x < sms) a->upd_grid = x;
    }
    // the attribute is a process-wide per-function limit, raised to this
    // launch's need and never lowered (set_max_dyn_smem)
    const int smem = (int)a->upd_smem;
    if (KB == 4) return set_blk_attrs<4>(smem, optin);
    if (KB == 8) return set_blk_attrs<8>(smem, optin);
    return set_blk_attrs<16>(smem, optin);
}

template <int KB, int NT>
static cudaError_t launch_blk_nt(const StepArgs& a, const uint32_t* Acur, uint32_t* Anext, const StepScalars* sc,
                                 cudaStream_t st) {
    const bool mag = a.mc.normalize == 3;
    const dim3 g(a.upd_grid), b(32 * a.upd_NG);
    const size_t sm = a.upd_smem;
    if (a.peer) {
        if (mag) k_update_blk<KB, 2, true, NT><<<g, b, sm, st>>>(a, Acur, Anext, sc);
        else k_update_blk<KB, 2, false, NT><<<g, b, sm, st>>>(a, Acur, Anext, sc);
        return cudaGetLastError();
    }
    return mag ? launch_maybe_pdl(a.pdl, k_update_blk<KB, 0, true, NT>, g, b, sm, st, a, Acur, Anext, sc)
               : launch_maybe_pdl(a.pdl, k_update_blk<KB, 0, false, NT>, g, b, sm, st, a, Acur, Anext, sc);
}
template <int KB>
static cudaError_t launch_blk_kb(const StepArgs& a, const uint32_t* Acur, uint32_t* Anext, const StepScalars* sc,
                                 cudaStream_t st) {
    if constexpr (TSAT_BLK_NT && KB <= 8) {
        if (a.N == 128) return launch_blk_nt<KB, 128>(a, Acur, Anext, sc, st);
        if (a.N == 256) return launch_blk_nt<KB, 256>(a, Acur, Anext, sc, st);
        if (a.N == 512) return launch_blk_nt<KB, 512>(a, Acur, Anext, sc, st);
    }
    return launch_blk_nt<KB, 0>(a, Acur, Anext, sc, st);
}

cudaError_t launch_update_blk(const StepArgs& a, const uint32_t* Acur, uint32_t* Anext, const StepScalars* sc,
                              cudaStream_t st) {
    if (a.V == 0) return cudaGetLastError();
    if (a.KB == 4) return launch_blk_kb<4>(a, Acur, Anext, sc, st);
    if (a.KB == 8) return launch_blk_kb<8>(a, Acur, Anext, sc, st);
    return launch_blk_kb<16>(a, Acur, Anext, sc, st);
}

}  // namespace tsat
