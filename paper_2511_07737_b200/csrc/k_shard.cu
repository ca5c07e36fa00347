// k_shard.cu - the candidate-sharded iteration.
//
// Each rank holds N_l = N/W candidates; the exchanges Eq. 5 needs are done
// by three exact collectives between these kernels:
//   k_gtable -> k_pack_max -> [MAX u64 (~best key, gmax, thmax)] -> k_unpack_max
//   k_update<mode A> (G -> Gbuf, J partials) -> [SUM int64 J[V]]
//   k_update_b (AdamW, Q partials, sign planes) -> [SUM int64 Q[V] + loss]
//   k_rows_finish (Eq. 5 statistics, bits of the next state) -> k_step_end_sharded
// All reduced quantities are integers (or maxima), so every rank sees the
// same values and the result is bit-identical for any W (and to W = 1).
#include "device_common.cuh"
#include "peer.cuh"

namespace tsat {

__global__ void k_pack_max(DevScalars* __restrict__ ds, const StepScalars* __restrict__ sc,
                           unsigned long long* __restrict__ buf) {
    const long long t = sc->t;
    buf[0] = ~ds->best_key;                       // min key -> max of its complement
    buf[1] = ds->gmax_bits;
    buf[2] = ds->thmax_bits[t & 1];
}

// key_only (normalize 2, per shard): gmax and max|theta| of J's scale stay local.
__global__ void k_unpack_max(DevScalars* __restrict__ ds, const StepScalars* __restrict__ sc,
                             const unsigned long long* __restrict__ buf, int key_only) {
    const long long t = sc->t;
    ds->best_key = ~buf[0];
    if (key_only) return;
    ds->gmax_bits = buf[1];
    ds->thmax_bits[t & 1] = (unsigned int)buf[2];
}

// Phase B of one row (one CTA per row): c_v from the global J, grad, AdamW
// (PyTorch order, R6-R6c), Q partial, max |theta|, sign planes of theta_{t+1}.
// Identical arithmetic to the fused k_update.
template <bool MAG>           // normalize 3 (R28), as k_update's MAG
__global__ void __launch_bounds__(256) k_update_b(StepArgs a, const uint32_t* __restrict__ Acur,
                                                  const StepScalars* __restrict__ sc) {
    __shared__ long long sh_s[32];
    __shared__ float sh_m[32];
    const int v = blockIdx.x;
    const int N = a.N, NW = N >> 5;
    const MethodConsts& mc = a.mc;
    const long long t = sc->t;
    const double gmax = __longlong_as_double((long long)a.ds->gmax_bits);
    const float thmax = __uint_as_float(a.ds->thmax_bits[t & 1]);
    const int2 pn = a.occ_pn[v];
    const int occ = pn.x + pn.y;
    int s;
    float p2;
    const bool jvalid = jscale(mc.Nnorm, occ, gmax, thmax, &s, &p2);
    const double rho = a.rowRho[v];
    double c = 0.0;
    if (mc.normalize && !a.rowGuard[v]) {
        const double J = jvalid ? scalbn((double)a.Jbuf[v], -s) : 0.0;
        c = J / (double)mc.Nnorm;
        c = c * rho;
        c = c * rho;
    }
    const float rhof = __double2float_rn(rho), ncf = -__double2float_rn(c);     // R27b: fp32 operands
    const float wdf = sc->wdf, a1 = sc->a1, b2f = sc->b2f, a2 = sc->a2, nss = sc->nss, rbc2 = sc->rbc2,
                epsf = sc->epsf, nz = sc->nz;
    float* trow = a.theta + (size_t)v * N;
    float* mrow = a.m + (size_t)v * N;
    float* vrow = a.v + (size_t)v * N;
    const float* grow = a.Gbuf + (size_t)v * N;
    const int lane = threadIdx.x & 31;
    long long Qn = 0;
    float mx = 0.0f;
    for (int base = 0; base < N; base += 4 * blockDim.x) {
        const int n = base + 4 * threadIdx.x;
        unsigned pnib = 0, nnib = 0;
        if (n < N) {
            const float4 th4 = *reinterpret_cast<const float4*>(trow + n);
            const float4 m4 = *reinterpret_cast<const float4*>(mrow + n);
            const float4 v4 = *reinterpret_cast<const float4*>(vrow + n);
            const float4 g4 = *reinterpret_cast<const float4*>(grow + n);
            float th[4] = {th4.x, th4.y, th4.z, th4.w};
            float mm[4] = {m4.x, m4.y, m4.z, m4.w};
            float vv[4] = {v4.x, v4.y, v4.z, v4.w};
            const float G[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float g = __fmaf_rn(G[q], rhof, jac_addend(ncf, th[q], MAG));   // R27b, R28
                float x = th[q] * wdf;
                const float m0 = mm[q] * sc->mkeep;
                const float mn = __fmaf_rn(a1, g - m0, m0);
                const float vb = vv[q] * b2f;
                const float vn = __fmaf_rn(a2 * g, g, vb);
                const float den = __fmul_rn(__fsqrt_rn(vn), rbc2) + epsf;
                x = x + (nss * mn) / den;
                if (mc.noise) {
                    const long long ng = mc.n0 + n + q;
                    uint32_t xr[4] = {(uint32_t)(ng >> 2), (uint32_t)v, (uint32_t)(1 + t), 0u};
                    philox4x32_10(xr, (uint32_t)mc.seed, (uint32_t)(mc.seed >> 32));
                    const float xi = (float)(xr[ng & 3] >> 8) * 5.9604644775390625e-08f - 0.5f;
                    x = x + nz * xi;
                }
                th[q] = x; mm[q] = mn; vv[q] = vn;
                Qn += __float2ll_rn((MAG ? fabsf(x) : x) * 4294967296.0f);
                mx = fmaxf(mx, fabsf(x));
                pnib |= (x > 0.0f ? 1u : 0u) << q;
                nnib |= (x < 0.0f ? 1u : 0u) << q;
            }
            *reinterpret_cast<float4*>(trow + n) = make_float4(th[0], th[1], th[2], th[3]);
            *reinterpret_cast<float4*>(mrow + n) = make_float4(mm[0], mm[1], mm[2], mm[3]);
            *reinterpret_cast<float4*>(vrow + n) = make_float4(vv[0], vv[1], vv[2], vv[3]);
        }
        unsigned pw = pnib << (4 * (lane & 7)), nw = nnib << (4 * (lane & 7));
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            pw |= __shfl_xor_sync(0xffffffffu, pw, o);
            nw |= __shfl_xor_sync(0xffffffffu, nw, o);
        }
        if ((lane & 7) == 0 && n < N) {
            a.Pbuf[(size_t)v * NW + (n >> 5)] = pw;
            a.Nbuf[(size_t)v * NW + (n >> 5)] = nw;
        }
    }
    block_sum_max(Qn, mx, sh_s, sh_m);
    if (threadIdx.x == 0) {
        a.Qbuf[v] = Qn;
        atomicMax(&a.ds->thmax_bits[(t + 1) & 1], __float_as_uint(mx));
        const unsigned long long bk = a.ds->best_key;               // global after the MAX exchange
        if ((bk >> 32) == 0ull && a.ds->sol_step < 0) {
            const long long idx = (long long)(bk & 0xffffffffull) - mc.n0;
            if (idx >= 0 && idx < N) a.sol[v] = (unsigned char)((Acur[(size_t)v * NW + (idx >> 5)] >> (idx & 31)) & 1u);
        }
        if (v == 0) a.Qbuf[a.V] = a.ds->loss_fx;                   // this rank's loss (fixed point)
    }
}

// Row statistics of a given state, partial over this rank's candidates
// (init / set_state): Q partial, sign planes, max |theta|.
__global__ void __launch_bounds__(256) k_rows_partial(StepArgs a, const float* __restrict__ theta,
                                                      unsigned int* __restrict__ thmax_bits) {
    __shared__ long long sh_s[32];
    __shared__ float sh_m[32];
    const int v = blockIdx.x;
    const int N = a.N, NW = N >> 5;
    const float* row = theta + (size_t)v * N;
    long long s = 0;
    float mx = 0.0f;
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
        const float x = row[n];
        s += __float2ll_rn((a.mc.normalize == 3 ? fabsf(x) : x) * 4294967296.0f);
        mx = fmaxf(mx, fabsf(x));
        const unsigned pw = __ballot_sync(0xffffffffu, x > 0.0f), nw = __ballot_sync(0xffffffffu, x < 0.0f);
        if ((threadIdx.x & 31) == 0) {
            a.Pbuf[(size_t)v * NW + (n >> 5)] = pw;
            a.Nbuf[(size_t)v * NW + (n >> 5)] = nw;
        }
    }
    block_sum_max(s, mx, sh_s, sh_m);
    if (threadIdx.x == 0) {
        a.Qbuf[v] = s;
        atomicMax(thmax_bits, __float_as_uint(mx));
        if (v == 0) a.Qbuf[a.V] = 0;
    }
}

// After the Q exchange: Eq. 5 statistics of every row and the bit planes of
// the new state (one warp per row); the global loss from slot V.
__global__ void __launch_bounds__(256) k_rows_finish(StepArgs a, uint32_t* __restrict__ Anext) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) a.ds->loss = -((double)a.Qbuf[a.V] * a.mc.loss_unscale);   // * 2^-e
    if (warp >= a.V) return;
    const int v = warp, NW = a.N >> 5;
    double dn = 0.0;
    if (lane == 0) {
        double rhon;
        unsigned char gn;
        const long long Q = a.Qbuf[v];
        row_finish(Q, a.mc, &dn, &rhon, &gn);
        a.rowQ[v] = Q; a.rowD[v] = dn; a.rowRho[v] = rhon; a.rowGuard[v] = gn;
    }
    dn = __shfl_sync(0xffffffffu, dn, 0);
    const bool dpos = dn > 0.0;
    for (int w = lane; w < NW; w += 32)
        Anext[(size_t)v * NW + w] = dpos ? a.Pbuf[(size_t)v * NW + w] : a.Nbuf[(size_t)v * NW + w];
}

// Peer path, init / set_state: exchange of the Q row partials in Qbuf.  Two
// kernels (all sends, then all receives) so no CTA waits on a CTA of its own
// grid that may not be resident.
__global__ void k_peer_send_rows(StepArgs a, unsigned gen) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= a.V) return;
    peer_row_send(a.px, 1, v, a.Qbuf[v], gen);
}
__global__ void k_peer_recv_rows(StepArgs a, unsigned gen) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= a.V) return;
    a.Qbuf[v] = peer_row_recv(a.px, 1, v, gen, a.ds, a.Qbuf[v]);
}

// End of a sharded iteration: first-model bookkeeping (global best), step
// info and accumulator reset; the loss was reduced exactly with Q.
__global__ void k_step_end_sharded(DevScalars* __restrict__ ds, const StepScalars* __restrict__ sc) {
    const long long t = sc->t;
    const unsigned long long bk = ds->best_key;
    const int bu = (int)(bk >> 32);
    const long long bi = (long long)(bk & 0xffffffffull);
    if (bu == 0 && ds->sol_step < 0) { ds->sol_step = t; ds->sol_idx = bi; }
    ds->info_t = t + 1;
    ds->info_best_unsat = bu;
    ds->info_best_idx = bi;
    ds->info_loss = ds->loss;
    ds->best_key = ~0ull;
    ds->gmax_bits = 0ull;
    ds->thmax_bits[t & 1] = 0u;
    ds->row_counter = 0;
    ds->loss_fx = 0;
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_shard_pack_max(const StepArgs& a, const StepScalars* sc, cudaStream_t st) {
    k_pack_max<<<1, 1, 0, st>>>(a.ds, sc, a.maxbuf);
    return cudaGetLastError();
}
cudaError_t launch_shard_unpack_max(const StepArgs& a, const StepScalars* sc, cudaStream_t st, bool key_only) {
    k_unpack_max<<<1, 1, 0, st>>>(a.ds, sc, a.maxbuf, key_only ? 1 : 0);
    return cudaGetLastError();
}
cudaError_t launch_update_b(const StepArgs& a, const uint32_t* Acur, const StepScalars* sc, cudaStream_t st) {
    if (a.V == 0) return cudaGetLastError();
    int threads = a.N / 4;
    threads = threads < 32 ? 32 : (threads > 256 ? 256 : (threads + 31) / 32 * 32);
    if (a.mc.normalize == 3) k_update_b<true><<<a.V, threads, 0, st>>>(a, Acur, sc);
    else k_update_b<false><<<a.V, threads, 0, st>>>(a, Acur, sc);
    return cudaGetLastError();
}
cudaError_t launch_rows_partial(const StepArgs& a, const float* theta, unsigned int* thmax_bits, cudaStream_t st) {
    if (a.V > 0) k_rows_partial<<<a.V, 256, 0, st>>>(a, theta, thmax_bits);
    return cudaGetLastError();
}
cudaError_t launch_rows_finish(const StepArgs& a, uint32_t* Anext, cudaStream_t st) {
    const long long threads = (long long)(a.V > 0 ? a.V : 1) * 32;
    k_rows_finish<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(a, Anext);
    return cudaGetLastError();
}
cudaError_t launch_step_end_sharded(const StepArgs& a, const StepScalars* sc, cudaStream_t st) {
    k_step_end_sharded<<<1, 1, 0, st>>>(a.ds, sc);
    return cudaGetLastError();
}

// Export all-gather over peer memory (tsat_export_best): every rank stores its
// n words into its slot of every rank's phase region, then publishes the slot
// with a release store of the generation; after acquiring the W flags the CTA
// copies the W slots (rank order) to recv.  Phases 0 (keys) and 1 (entries)
// use separate regions: a rank writes phase p of call c + 1 only after every
// rank has sent data that it produces after reading phase p of call c.
__global__ void __launch_bounds__(256) k_peer_allgather(PeerArgs px, int phase, const unsigned long long* __restrict__ send,
                                                        int n, unsigned long long* __restrict__ recv, unsigned gen,
                                                        DevScalars* ds) {
    __shared__ int ok;
    const size_t slot_words = (size_t)kExportCap;
    auto region = [&](int p) {
        return reinterpret_cast<unsigned long long*>(px.xb[p] + px.L.ex) + (size_t)phase * px.W * slot_words;
    };
    for (int p = 0; p < px.W; ++p) {
        if (p == px.rank) continue;
        unsigned long long* d = region(p) + (size_t)px.rank * slot_words;
        for (int i = threadIdx.x; i < n; i += blockDim.x) st_relaxed_sys_u64(d + i, send[i]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (int p = 0; p < px.W; ++p)
            if (p != px.rank)
                st_release_sys(reinterpret_cast<unsigned*>(px.xb[p] + px.L.ef) + (size_t)phase * px.W + px.rank, gen);
        int good = 1;
        const unsigned* fs = reinterpret_cast<const unsigned*>(px.xb[px.rank] + px.L.ef) + (size_t)phase * px.W;
        for (int r = 0; r < px.W && good; ++r)
            if (r != px.rank && !peer_wait(fs + r, gen, ds)) good = 0;
        ok = good;
    }
    __syncthreads();
    if (!ok) return;
    for (int r = 0; r < px.W; ++r) {
        const unsigned long long* s = r == px.rank ? send : region(px.rank) + (size_t)r * slot_words;
        for (int i = threadIdx.x; i < n; i += blockDim.x)
            recv[(size_t)r * n + i] = r == px.rank ? s[i] : ld_relaxed_sys_u64(s + i);
    }
}

cudaError_t launch_peer_allgather(const StepArgs& a, int phase, const unsigned long long* send, int n,
                                  unsigned long long* recv, unsigned gen, cudaStream_t st) {
    k_peer_allgather<<<1, 256, 0, st>>>(a.px, phase, send, n, recv, gen, a.ds);
    return cudaGetLastError();
}

cudaError_t launch_peer_rows_exchange(const StepArgs& a, unsigned gen, cudaStream_t st) {
    if (a.V == 0) return cudaGetLastError();
    const unsigned blocks = (unsigned)((a.V + 255) / 256);
    k_peer_send_rows<<<blocks, 256, 0, st>>>(a, gen);
    k_peer_recv_rows<<<blocks, 256, 0, st>>>(a, gen);
    return cudaGetLastError();
}

}  // namespace tsat
