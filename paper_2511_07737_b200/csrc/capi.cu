// capi.cu - the extern "C" boundary of libturbosat (include/turbosat.h) and
// the host runtime behind it: context, CNF upload, workspace layout, per-call
// step-scalar tables, CUDA-graph capture of k-iteration sequences, kernel
// timing, export.
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges visible to nsys / ncu --nvtx
#include <cuda_runtime.h>

#include <algorithm>
#include <new>
#include <stdexcept>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <string>
#include <vector>

#include "../../include/turbosat.h"
#include "tsat_internal.h"


using namespace tsat;

#ifndef TSAT_SEG
#define TSAT_SEG 1                      // length-segmented clause evaluation (k_clause_seg)
#endif

struct DevCnf {
    void* arena = nullptr;              // one allocation holding every array below
    uint32_t *cptr = nullptr, *clit = nullptr, *occ_ptr = nullptr, *occ_rec = nullptr, *occ_cnt = nullptr;
    uint32_t *bat_ptr = nullptr, *bat_rec = nullptr;
    uint32_t* seg_lit = nullptr;        // clause length segments (k_clause_seg), K <= 7
    int2* occ_pn = nullptr;
    int* hub_of = nullptr;
    int4* hub_sc = nullptr;
};

struct tsat_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;      // caller's stream: every launch / copy
    cudaStream_t cap_stream = nullptr;  // private stream used only to capture graphs
    cudaStream_t cap_side = nullptr;    // capture fork: k_hub beside k_clause / k_gtable
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool sharded = false;               // candidate-sharded path (NCCL communicator)
    void* comm = nullptr;               // ncclComm_t
    // peer-exchange path (tsat_create_peer): exchanges inside the kernels over
    // NVLink peer memory, buffers shared by CUDA IPC
    bool peer = false;
    void* xbuf = nullptr;               // this rank's exchange buffer (PeerLayout)
    cudaIpcMemHandle_t xhandle{};
    char* peer_ptr[kMaxPeers] = {};
    bool peer_ipc[kMaxPeers] = {};      // opened with cudaIpcOpenMemHandle (close on destroy)
    bool peers_ready = false;
    unsigned xgen = 0;                  // exchange generation (same sequence on every rank)
    int rank = 0, world = 1;
    tsat_status poisoned = TSAT_OK;
    std::string err;
    // CNF
    bool have_cnf = false;
    HostCnf cnf;
    DevCnf dcnf;
    // batch
    bool have_batch = false;
    int64_t N_global = 0;
    int N = 0;                 // local
    long long n0 = 0;
    int KB = 4;
    uint64_t seed = 0;
    tsat_config cfg{};
    MethodConsts mc{};
    Layout L{};
    char* ws = nullptr;
    size_t ws_bytes = 0;
    int64_t t = 0;             // iterations completed
    int64_t steps_done = 0;    // >= 1 once a state has been evaluated
    StepScalars* h_steptab = nullptr;   // pinned, 2 slots of kMaxStepsPerCall (alternating tsat_step calls)
    cudaEvent_t tab_ev[2] = {nullptr, nullptr};   // slot's upload done (the host may rewrite it)
    int tab_slot = 0;
    DevScalars* h_scal = nullptr;       // pinned readback
    std::map<int, cudaGraphExec_t> graphs;
    // profiling
    bool profiling = false;
    std::vector<cudaEvent_t> events;    // (kKernelsPerStep+1) per step of the largest k
    double prof_ms[kKernelsPerStep] = {0, 0, 0, 0, 0};
    // k_update launch geometry (configure_kernels)
    int upd_mode = 0, upd_GT = 0, upd_NG = 0, upd_grid = 0, num_sms = 0, upd_recbufs = 2;
    int upd_RB = 1, upd_blk_cap = 0;    // row-block k_update (small shards, k_update_blk.cu)
    int upd_cw6 = 0;                    // per-row k_update with 6-plane counters (configure)
    int* blk_rows = nullptr;            // device [V]: rows in block order (library-owned)
    // dense tensor-core clause evaluation (config.clause_eval = 1, k_dense.cu): library-owned
    uint8_t* dP = nullptr;
    uint8_t* dAL = nullptr;
    int dKp = 0, dCp = 0;
    // fp64 state (config.state_fp64 = 1, k_fp64.cu): library-owned
    double *th64 = nullptr, *m64 = nullptr, *v64 = nullptr, *G64 = nullptr, *gt64 = nullptr;
    long long* J64 = nullptr;
    unsigned long long* Qp64 = nullptr;
    uint32_t *Pw64 = nullptr, *Nw64 = nullptr;
    int upd_chunk = 0, upd_gs_global = 0;
    bool chunked = false;               // N too large for the fused kernel: split sequence, no collectives at W = 1
    int upd_cl = 0;                     // > 1: cluster-split rows (k_update MODE 3) instead of chunking
    int upd_prefetch = 1;               // k_update L2 row prefetch (configure_update)
    bool use_seg = false;               // length-segmented clause evaluation (k_clause_seg)
    size_t upd_smem = 0;
    int64_t prof_steps = 0;
    int prof_pending_k = 0;
};

namespace {

tsat_status fail(tsat_ctx c, tsat_status s, const std::string& msg) {
    if (c) c->err = msg;
    return s;
}

tsat_status cuda_fail(tsat_ctx c, cudaError_t e, const char* where) {
    if (c) {
        c->poisoned = TSAT_E_CUDA;
        c->err = std::string(where) + ": " + cudaGetErrorString(e);
    }
    return TSAT_E_CUDA;
}

#define CK(call)                                                  \
    do {                                                          \
        cudaError_t e_ = (call);                                  \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call);  \
    } while (0)

// Makes ctx->device current for the duration of an entry point and restores
// the caller's current device on return (calls on a context whose
// device is not current, and callers that switch devices).
struct DevGuard {
    int prev = -1;
    explicit DevGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DevGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

#define GUARD_CTX()                                    \
    if (!ctx) return TSAT_E_ARG;                       \
    if (ctx->poisoned != TSAT_OK) return ctx->poisoned; \
    DevGuard dev_guard_(ctx->device)

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

float __uint_as_float_host(uint32_t u) {
    float f;
    memcpy(&f, &u, 4);
    return f;
}

// No C++ exception crosses the C ABI: host allocation failures map to
// TSAT_E_OOM, anything else to TSAT_E_ARG.
template <class F>
tsat_status no_throw(tsat_ctx ctx, F&& f) {
    try {
        return f();
    } catch (const std::bad_alloc&) {
        if (ctx) ctx->err = "host allocation failed";
        return TSAT_E_OOM;
    } catch (const std::exception& ex) {
        if (ctx) ctx->err = std::string("exception: ") + ex.what();
        return TSAT_E_ARG;
    } catch (...) {
        if (ctx) ctx->err = "unknown exception";
        return TSAT_E_ARG;
    }
}

// Exchange buffers created in this process, by IPC handle: a rank whose peer
// lives in the same process (tests: several ranks on one GPU) maps it directly
// (cudaIpcOpenMemHandle refuses handles of its own process).
std::mutex g_xreg_mu;
std::map<std::string, void*> g_xreg;
std::string handle_key(const cudaIpcMemHandle_t& h) { return std::string(h.reserved, sizeof(h.reserved)); }

void peer_release(tsat_ctx ctx) {
    for (int r = 0; r < kMaxPeers; ++r) {
        if (ctx->peer_ipc[r] && ctx->peer_ptr[r]) cudaIpcCloseMemHandle(ctx->peer_ptr[r]);
        ctx->peer_ipc[r] = false;
        ctx->peer_ptr[r] = nullptr;
    }
    ctx->peers_ready = false;
    if (ctx->xbuf) {
        {
            std::lock_guard<std::mutex> lk(g_xreg_mu);
            g_xreg.erase(handle_key(ctx->xhandle));
        }
        cudaFree(ctx->xbuf);
        ctx->xbuf = nullptr;
    }
}

Layout make_layout(int V, int N, int KB, int n_hubs, bool sharded, bool peer) {
    Layout L{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off = align_up(off + bytes);
        return o;
    };
    size_t VN = (size_t)V * N, NW = (size_t)N / 32;
    L.theta = take(VN * 4);
    L.m = take(VN * 4);
    L.v = take(VN * 4);
    L.A0 = take((size_t)(V + 1) * NW * 4);            // + row V: all-zero padding row (k_clause)
    L.A1 = take((size_t)(V + 1) * NW * 4);
    L.hist = take((size_t)N * KB * 4);
    L.gtab = take((size_t)N * KB * 4);
    L.S = take((size_t)N * 8);
    L.lossp = take((size_t)((N + 255) / 256) * 8);
    L.unsat = take((size_t)N * 4);
    L.rowQ = take((size_t)V * 8);
    L.rowD = take((size_t)V * 8);
    L.rowRho = take((size_t)V * 8);
    L.rowGuard = take((size_t)V);
    L.scal = take(sizeof(DevScalars));
    L.steptab = take(sizeof(StepScalars) * kMaxStepsPerCall);
    L.sol = take((size_t)V);
    L.hubD = take((size_t)n_hubs * (KB - 1) * N * 4);
    const size_t sv = sharded ? 1 : 0;
    const size_t sr = (sharded || peer) ? 1 : 0;      // row-statistics buffers (init / set_state)
    L.Gbuf = take(sv * VN * 4);
    L.Jbuf = take(sv * (size_t)V * 8);
    L.Qbuf = take(sr * ((size_t)V + 1) * 8);
    L.Pbuf = take(sr * (size_t)V * NW * 4);
    L.Nbuf = take(sr * (size_t)V * NW * 4);
    L.maxbuf = take(sv * 3 * 8);
    L.total = off;
    return L;
}

// Whether N candidates per GPU need the chunked split sequence (the fused
// k_update's shared memory would not hold the batch's g table + 2 groups),
// or (W = 1, *cl > 1) run as cluster-split rows instead.
tsat_status batch_chunked(tsat_ctx ctx, int N, int KB, bool* out, int* cl = nullptr) {
    int optin = 0;
    CK(cudaSetDevice(ctx->device));
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    const int rec_cap = std::max(64, (ctx->cnf.max_rec_words + 63) / 64 * 64);
    const bool w1 = !ctx->sharded && !ctx->peer && ctx->world == 1 && N >= 1024;
    const int c = w1 ? update_cluster_size(KB, N, rec_cap, optin) : 0;
    if (cl) *cl = c;
    *out = c == 0 && !update_fits_fused(KB, N, rec_cap, optin);
    return TSAT_OK;
}

StepArgs step_args(tsat_ctx ctx) {
    StepArgs a{};
    char* w = ctx->ws;
    const Layout& L = ctx->L;
    a.theta = (float*)(w + L.theta);
    a.m = (float*)(w + L.m);
    a.v = (float*)(w + L.v);
    a.A0 = (uint32_t*)(w + L.A0);
    a.A1 = (uint32_t*)(w + L.A1);
    a.hist = (int*)(w + L.hist);
    a.unsat = (int*)(w + L.unsat);
    a.gtab = (float*)(w + L.gtab);
    a.hubD = (int*)(w + L.hubD);
    a.S = (double*)(w + L.S);
    a.lossp = (double*)(w + L.lossp);
    a.rowQ = (long long*)(w + L.rowQ);
    a.rowD = (double*)(w + L.rowD);
    a.rowRho = (double*)(w + L.rowRho);
    a.rowGuard = (unsigned char*)(w + L.rowGuard);
    a.sol = (unsigned char*)(w + L.sol);
    a.ds = (DevScalars*)(w + L.scal);
    a.cptr = ctx->dcnf.cptr;
    a.clit = ctx->dcnf.clit;
    a.occ_ptr = ctx->dcnf.occ_ptr;
    a.occ_rec = ctx->dcnf.occ_rec;
    a.occ_cnt = ctx->dcnf.occ_cnt;
    a.upd_ptr = ctx->cnf.batched ? ctx->dcnf.bat_ptr : ctx->dcnf.occ_ptr;
    a.upd_rec = ctx->cnf.batched ? ctx->dcnf.bat_rec : ctx->dcnf.occ_rec;
    a.occ_pn = ctx->dcnf.occ_pn;
    a.hub_of = ctx->dcnf.hub_of;
    a.hub_sc = ctx->dcnf.hub_sc;
    a.n_hubs = ctx->cnf.n_hubs;
    a.n_hub_sc = ctx->cnf.n_hub_sc;
    a.uniform_len = ctx->cnf.uniform_len;
    a.num_sms = ctx->num_sms;
    a.upd_mode = ctx->upd_mode;
    a.upd_chunk = ctx->upd_chunk;
    a.upd_gs_global = ctx->upd_gs_global;
    a.upd_GT = ctx->upd_GT;
    a.upd_recbufs = ctx->upd_recbufs;
#ifndef TSAT_PDL
#define TSAT_PDL 1
#endif
    // PDL on the fused W = 1 sequence (one stream, no forked k_hub branch)
    a.pdl = TSAT_PDL && !ctx->profiling && !ctx->sharded && !ctx->chunked && !ctx->peer && ctx->cnf.n_hub_sc == 0 &&
            ctx->upd_cl <= 1 &&
            ctx->th64 == nullptr;
    a.upd_NG = ctx->upd_NG;
    a.upd_grid = ctx->upd_grid;
    a.upd_smem = ctx->upd_smem;
    a.upd_rec_cap = std::max(64, (ctx->cnf.max_rec_words + 63) / 64 * 64);
    a.upd_RB = ctx->upd_RB;
    a.upd_blk_cap = ctx->upd_blk_cap;
    a.upd_cw6 = ctx->upd_cw6;
    a.upd_cl = ctx->upd_cl;
    a.upd_prefetch = ctx->upd_prefetch;
    a.blk_rows = ctx->blk_rows;
    a.use_seg = ctx->use_seg ? 1 : 0;
    a.seg_lit = ctx->dcnf.seg_lit;
    for (int L = 0; L < 8; ++L) {
        a.seg_C[L] = ctx->cnf.seg_C.size() == 8 ? ctx->cnf.seg_C[L] : 0;
        a.seg_off[L] = ctx->cnf.seg_off.size() == 8 ? ctx->cnf.seg_off[L] : 0;
    }
    a.fp64 = ctx->th64 != nullptr;
    a.th64 = ctx->th64; a.m64 = ctx->m64; a.v64 = ctx->v64; a.G64 = ctx->G64; a.gt64 = ctx->gt64;
    a.J64 = ctx->J64; a.Qp64 = ctx->Qp64; a.Pw64 = ctx->Pw64; a.Nw64 = ctx->Nw64;
    a.dense = ctx->dP != nullptr;
    a.dP = ctx->dP;
    a.dAL = ctx->dAL;
    a.dKp = ctx->dKp;
    a.dCp = ctx->dCp;
    a.sharded = (ctx->sharded || ctx->chunked) ? 1 : 0;     // kernels: the split (phase A / B) sequence
    a.Gbuf = (float*)(w + L.Gbuf);
    a.Jbuf = (long long*)(w + L.Jbuf);
    a.Qbuf = (long long*)(w + L.Qbuf);
    a.Pbuf = (uint32_t*)(w + L.Pbuf);
    a.Nbuf = (uint32_t*)(w + L.Nbuf);
    a.maxbuf = (unsigned long long*)(w + L.maxbuf);
    a.peer = ctx->peer ? 1 : 0;
    if (ctx->peer) {
        for (int r = 0; r < ctx->world; ++r) a.px.xb[r] = ctx->peer_ptr[r];
        a.px.W = ctx->world;
        a.px.rank = ctx->rank;
        a.px.V = ctx->cnf.V;
        a.px.exchange_rows = ctx->cfg.normalize != 2 && !(ctx->world == 1 && std::getenv("TSAT_PEER_NOX"));   // A/B hook
        a.px.L = peer_layout(ctx->cnf.V, ctx->world);
    }
    a.V = ctx->cnf.V;
    a.N = ctx->N;
    a.C = ctx->cnf.C;
    a.KB = ctx->KB;
    a.mc = ctx->mc;
    return a;
}

// Host-side canonical per-iteration scalars (libm; R6, R9).
double lr_at(const tsat_config& c, int64_t t) {
    int64_t i = (t % c.restart_every) / c.decay_every;
    double p = 1.0;
    for (int64_t k = 0; k < i; ++k) p = p * c.decay_factor;
    double lr = c.lr0 / p;
    return lr < c.lr_min ? c.lr_min : lr;
}

StepScalars step_scalars(const tsat_config& c, int64_t t) {
    StepScalars s{};
    double lr = lr_at(c, t);
    // AdamW bias-correction step; a moment reset re-creates the optimizer
    const bool reset = c.reset_moments_on_restart && t > 0 && t % c.restart_every == 0;
    double st = (double)((c.reset_moments_on_restart ? t % c.restart_every : t) + 1);
    s.t = t;
    s.lr = lr;
    s.wdf = (float)(1.0 - lr * c.weight_decay);
    s.a1 = (float)(1.0 - c.beta1);
    s.b2f = reset ? 0.0f : (float)c.beta2;
    s.mkeep = reset ? 0.0f : 1.0f;
    s.a2 = (float)(1.0 - c.beta2);
    double bc1 = 1.0 - std::pow(c.beta1, st);
    double bc2 = 1.0 - std::pow(c.beta2, st);
    s.nss = (float)(-(lr / bc1));
    s.rbc2 = (float)(1.0 / std::sqrt(bc2));
    s.epsf = (float)c.eps;
    s.nz = (float)(lr * c.noise_sigma);
    // SmoothMin temperature of this iteration and its table E[d] = exp(-tau d)
    // (host libm, R11); annealed within each LR cycle when tau_final > 0 (R29)
    double tau = c.tau;
    if (c.tau_final > 0 && c.restart_every > 1)
        tau = c.tau * std::pow(c.tau_final / c.tau, (double)(t % c.restart_every) / (double)(c.restart_every - 1));
    s.tau = tau;
    for (int d = 0; d < 16; ++d) s.E[d] = std::exp(-tau * (double)d);
    // fp64 state (R30): the same AdamW scalars unrounded
    s.wdf64 = 1.0 - lr * c.weight_decay;
    s.a1_64 = 1.0 - c.beta1;
    s.b2_64 = reset ? 0.0 : c.beta2;
    s.a2_64 = 1.0 - c.beta2;
    s.nss64 = -(lr / bc1);
    s.rbc2_64 = 1.0 / std::sqrt(bc2);
    s.eps64 = c.eps;
    s.nz64 = lr * c.noise_sigma;
    return s;
}

void free_fp64(tsat_ctx ctx) {
    for (void* p : {(void*)ctx->th64, (void*)ctx->m64, (void*)ctx->v64, (void*)ctx->G64, (void*)ctx->gt64,
                    (void*)ctx->J64, (void*)ctx->Qp64, (void*)ctx->Pw64, (void*)ctx->Nw64})
        cudaFree(p);
    ctx->th64 = ctx->m64 = ctx->v64 = ctx->G64 = ctx->gt64 = nullptr;
    ctx->J64 = nullptr;
    ctx->Qp64 = nullptr;
    ctx->Pw64 = ctx->Nw64 = nullptr;
}

void free_cnf(tsat_ctx ctx) {
    if (ctx->dcnf.arena) cudaFreeAsync(ctx->dcnf.arena, ctx->stream);
    ctx->dcnf = DevCnf{};
    ctx->have_cnf = false;
}

void drop_graphs(tsat_ctx ctx) {
    for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
    ctx->graphs.clear();
}

void fill_info(const HostCnf& h, tsat_cnf_info* info) {
    if (!info) return;
    info->V = h.V;
    info->C = h.C;
    info->nnz = h.nnz;
    info->K = h.K;
    info->header_C = h.header_C;
    info->n_warnings = h.n_warnings;
    info->n_tautologies = h.n_tautologies;
    info->n_duplicates = h.n_duplicates;
    info->has_empty = h.has_empty;
    info->n_hub_rows = h.n_hubs;
}

tsat_status upload_cnf(tsat_ctx ctx, HostCnf&& h) {
    drop_graphs(ctx);
    free_cnf(ctx);
    ctx->have_batch = false;
    ctx->cnf = std::move(h);
    const HostCnf& c = ctx->cnf;
    // every device array of the CNF in one allocation, filled by one copy from
    // one host staging buffer (per-array cudaMalloc + pageable copies cost
    // milliseconds of the end-to-end setup)
    struct Part { void** dst; const void* src; size_t bytes, alloc; };
    std::vector<Part> parts;
    auto add = [&](void** dst, const void* src, size_t n, size_t min_n) {
        parts.push_back({dst, src, n * 4, ((std::max(n, min_n) * 4) + 255) / 256 * 256});
    };
    add((void**)&ctx->dcnf.cptr, c.clause_ptr.data(), c.clause_ptr.size(), 1);
    add((void**)&ctx->dcnf.clit, c.clause_lit.data(), c.clause_lit.size(), 1);
    if (c.K <= 7 && !c.seg_lit.empty()) add((void**)&ctx->dcnf.seg_lit, c.seg_lit.data(), c.seg_lit.size(), 1);
    add((void**)&ctx->dcnf.occ_ptr, c.occ_ptr.data(), c.occ_ptr.size(), 1);
    add((void**)&ctx->dcnf.occ_rec, c.occ_rec.data(), c.occ_rec.size(), 1);
    add((void**)&ctx->dcnf.occ_cnt, c.occ_cnt.data(), c.occ_cnt.size(), 1);
    if (c.batched) {
        add((void**)&ctx->dcnf.bat_ptr, c.bat_ptr.data(), c.bat_ptr.size(), 1);
        add((void**)&ctx->dcnf.bat_rec, c.bat_rec.data(), c.bat_rec.size(), 1);
    }
    add((void**)&ctx->dcnf.occ_pn, c.occ_pn.data(), c.occ_pn.size(), 4);
    add((void**)&ctx->dcnf.hub_of, c.hub_of.data(), c.hub_of.size(), 4);
    add((void**)&ctx->dcnf.hub_sc, c.hub_sc.data(), c.hub_sc.size(), 4);
    size_t total = 0;
    for (const Part& p : parts) total += p.alloc;
    CK(cudaSetDevice(ctx->device));
    // stream-ordered, from the device's default pool kept reserved across
    // frees (a plain cudaMalloc after another context's frees measured 3-22 ms)
    {
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, ctx->device));
        unsigned long long keep = ~0ull;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    CK(cudaMallocAsync(&ctx->dcnf.arena, total, ctx->stream));
    std::vector<unsigned char> stage(total);
    size_t off = 0;
    for (const Part& p : parts) {
        *p.dst = (char*)ctx->dcnf.arena + off;
        if (p.bytes) std::memcpy(stage.data() + off, p.src, p.bytes);
        off += p.alloc;
    }
    CK(cudaMemcpyAsync(ctx->dcnf.arena, stage.data(), total, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));        // `stage` is pageable and local
    if (ctx->peer) {                    // a fresh, zeroed exchange buffer for this V; peers must reconnect
        peer_release(ctx);
        const size_t xb = peer_layout(c.V, ctx->world).total;
        CK(cudaMalloc(&ctx->xbuf, xb));
        CK(cudaMemsetAsync(ctx->xbuf, 0, xb, ctx->stream));
        CK(cudaIpcGetMemHandle(&ctx->xhandle, ctx->xbuf));
        std::lock_guard<std::mutex> lk(g_xreg_mu);
        g_xreg[handle_key(ctx->xhandle)] = ctx->xbuf;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->have_cnf = true;
    return TSAT_OK;
}

tsat_status check_batch(tsat_ctx ctx, bool need_step) {
    if (!ctx->have_cnf || !ctx->have_batch) return fail(ctx, TSAT_E_STATE, "no batch: call tsat_init_batch first");
    if (need_step && ctx->steps_done == 0) return fail(ctx, TSAT_E_STATE, "no evaluated state: call tsat_step first");
    return TSAT_OK;
}

// Eq. 5 row statistics and bit planes of the state theta_t (init / set_state):
// one kernel for W = 1; partial sums + exact int64 exchange when sharded.
tsat_status state_stats(tsat_ctx ctx, const StepArgs& a, int64_t t) {
    uint32_t* A = (t & 1) ? a.A1 : a.A0;
    unsigned int* thm = &a.ds->thmax_bits[t & 1];
    if (a.fp64) {                                  // R30 (one GPU)
        CK(launch_rowstats64(a, t, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        return TSAT_OK;
    }
    if (ctx->peer) {
        const unsigned gen = ++ctx->xgen;
        CK(launch_rows_partial(a, a.theta, thm, ctx->stream));
        if (ctx->cfg.normalize != 2) CK(launch_peer_rows_exchange(a, gen, ctx->stream));
        CK(launch_rows_finish(a, A, ctx->stream));
        CK(cudaMemcpyAsync(ctx->h_scal, ctx->ws + ctx->L.scal, sizeof(DevScalars), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (ctx->h_scal->xerr) {
            ctx->poisoned = TSAT_E_NCCL;
            return fail(ctx, TSAT_E_NCCL, "peer exchange timed out (row statistics)");
        }
    } else if (!ctx->sharded) {
        CK(launch_rowstats(a.theta, a.V, a.N, ctx->mc, a.rowQ, a.rowD, a.rowRho, a.rowGuard, A, thm, ctx->stream));
    } else {
        std::string err;
        CK(launch_rows_partial(a, a.theta, thm, ctx->stream));
        if (ctx->cfg.normalize != 2 && comm_allreduce_sum_i64(ctx->comm, a.Qbuf, (size_t)a.V + 1, ctx->stream, &err)) {
            ctx->poisoned = TSAT_E_NCCL;
            ctx->err = err;
            return TSAT_E_NCCL;
        }
        CK(launch_rows_finish(a, A, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return TSAT_OK;
}

// One profiling segment of an iteration.  W = 1: one kernel per segment.
// Sharded: the segments also hold the collectives:
//   0 clause | 1 gtable, MAX(best, gmax, thmax) | 2 hub |
//   3 update A, SUM J, update B, SUM Q+loss, rows finish | 4 step end.
// Returns 0, 6 (CUDA) or 7 (NCCL) with *err.
int launch_segment(tsat_ctx ctx, const StepArgs& a, int seg, const StepScalars* sc, long long t, cudaStream_t st,
                   std::string* err) {
    auto ck = [&](cudaError_t e, const char* what) {
        if (e == cudaSuccess) return 0;
        *err = std::string(what) + ": " + cudaGetErrorString(e);
        return 6;
    };
    if (!ctx->sharded && !ctx->chunked) return ck(launch_step_kernel(seg, a, sc, t, st), "step kernel");
    const bool comm = ctx->sharded;           // chunked at W = 1: the same sequence without exchanges
    const uint32_t* Acur = (t & 1) ? a.A1 : a.A0;
    uint32_t* Anext = (t & 1) ? a.A0 : a.A1;
    int r = 0;
    switch (seg) {
        case 0: return ck(launch_step_kernel(0, a, sc, t, st), "k_clause");
        case 1:
            if ((r = ck(launch_step_kernel(1, a, sc, t, st), "k_gtable"))) return r;
            if (!comm) return 0;
            if ((r = ck(launch_shard_pack_max(a, sc, st), "k_pack_max"))) return r;
            if ((r = comm_allreduce_max_u64(ctx->comm, a.maxbuf, 3, st, err))) return r;
            return ck(launch_shard_unpack_max(a, sc, st, a.mc.normalize == 2), "k_unpack_max");
        case 2: return ck(launch_step_kernel(2, a, sc, t, st), "k_hub");
        case 3:
            if (ctx->chunked && (r = ck(cudaMemsetAsync(a.Jbuf, 0, (size_t)a.V * 8, st), "J reset"))) return r;
            if ((r = ck(launch_update_a(a, Acur, sc, st), "k_update(A)"))) return r;
            // normalize 2 (per shard): J and the row sums stay local, only the loss slot is summed
            if (comm && a.mc.normalize != 2 && (r = comm_allreduce_sum_i64(ctx->comm, a.Jbuf, (size_t)a.V, st, err)))
                return r;
            if ((r = ck(launch_update_b(a, Acur, sc, st), "k_update_b"))) return r;
            if (!comm) {
            } else if (a.mc.normalize == 2) {
                if ((r = comm_allreduce_sum_i64(ctx->comm, a.Qbuf + a.V, 1, st, err))) return r;
            } else if ((r = comm_allreduce_sum_i64(ctx->comm, a.Qbuf, (size_t)a.V + 1, st, err))) {
                return r;
            }
            return ck(launch_rows_finish(a, Anext, st), "k_rows_finish");
        case 4: return ck(launch_step_end_sharded(a, sc, st), "k_step_end");
    }
    return 0;
}

// Launch the k-iteration sequence (graph or direct).
tsat_status launch_steps(tsat_ctx ctx, int k) {
    StepArgs a = step_args(ctx);
    const StepScalars* sc = (const StepScalars*)(ctx->ws + ctx->L.steptab);
    if (ctx->profiling) {
        size_t need = (size_t)k * (kKernelsPerStep + 1);
        while (ctx->events.size() < need) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            ctx->events.push_back(e);
        }
    }
    // k_hub reads only the evaluated state's bit planes, so (unless every
    // kernel is being timed) it runs on a forked capture branch beside
    // k_clause and k_gtable and joins before k_update
    const bool fork_hub = !ctx->profiling && ctx->cnf.n_hub_sc > 0 && ctx->th64 == nullptr;
    if (fork_hub && !ctx->cap_side) {
        CK(cudaStreamCreateWithFlags(&ctx->cap_side, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
    }
    std::string serr;
    int sstat = 0;
    auto body = [&](bool capture) -> cudaError_t {
        for (int i = 0; i < k; ++i) {
            long long t = ctx->t + i;
            if (fork_hub) {
                cudaError_t e = cudaEventRecord(ctx->ev_fork, ctx->cap_stream);
                if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->cap_side, ctx->ev_fork, 0);
                if (e != cudaSuccess) return e;
                sstat = launch_segment(ctx, a, 2, sc + i, t, ctx->cap_side, &serr);
                if (sstat) return cudaErrorUnknown;
                if ((e = cudaEventRecord(ctx->ev_join, ctx->cap_side)) != cudaSuccess) return e;
            }
            for (int kk = 0; kk < kKernelsPerStep; ++kk) {
                if (fork_hub && kk == 2) {
                    cudaError_t e = cudaStreamWaitEvent(ctx->cap_stream, ctx->ev_join, 0);
                    if (e != cudaSuccess) return e;
                    continue;
                }
                if (ctx->profiling) {
                    cudaError_t e = cudaEventRecordWithFlags(ctx->events[(size_t)i * (kKernelsPerStep + 1) + kk], ctx->cap_stream,
                                                            cudaEventRecordExternal);
                    if (e != cudaSuccess) return e;
                }
                // kernels read t from the step table; the parity of t selects
                // the A buffers, so the graph is keyed by (k, t parity).
                sstat = launch_segment(ctx, a, kk, sc + i, t, ctx->cap_stream, &serr);
                if (sstat) return cudaErrorUnknown;
            }
            if (ctx->profiling) {
                cudaError_t e = cudaEventRecordWithFlags(ctx->events[(size_t)i * (kKernelsPerStep + 1) + kKernelsPerStep],
                                                        ctx->cap_stream, cudaEventRecordExternal);
                if (e != cudaSuccess) return e;
            }
        }
        (void)capture;
        return cudaSuccess;
    };
    int key = k * 4 + (int)(ctx->t & 1) * 2 + (ctx->profiling ? 1 : 0);
    auto it = ctx->graphs.find(key);
    if (it == ctx->graphs.end()) {
        cudaGraph_t g;
        // capture on the private stream (the caller's may be the legacy
        // default stream, which cannot be captured); replay on the caller's
        CK(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
        cudaError_t e = body(true);
        cudaError_t e2 = cudaStreamEndCapture(ctx->cap_stream, &g);
        if (sstat) {
            if (e2 == cudaSuccess) cudaGraphDestroy(g);
            ctx->poisoned = sstat == 7 ? TSAT_E_NCCL : TSAT_E_CUDA;
            ctx->err = serr;
            return ctx->poisoned;
        }
        if (e != cudaSuccess) return cuda_fail(ctx, e, "capture step kernels");
        if (e2 != cudaSuccess) return cuda_fail(ctx, e2, "cudaStreamEndCapture");
        cudaGraphExec_t ex;
        CK(cudaGraphInstantiate(&ex, g, 0));
        cudaGraphDestroy(g);
        it = ctx->graphs.emplace(key, ex).first;
    }
    CK(cudaGraphLaunch(it->second, ctx->stream));
    if (ctx->profiling) ctx->prof_pending_k = k;
    return TSAT_OK;
}

tsat_status collect_profile(tsat_ctx ctx) {
    if (!ctx->profiling || ctx->prof_pending_k == 0) return TSAT_OK;
    int k = ctx->prof_pending_k;
    for (int i = 0; i < k; ++i)
        for (int kk = 0; kk < kKernelsPerStep; ++kk) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, ctx->events[(size_t)i * (kKernelsPerStep + 1) + kk],
                                    ctx->events[(size_t)i * (kKernelsPerStep + 1) + kk + 1]));
            ctx->prof_ms[kk] += ms;
        }
    ctx->prof_steps += k;
    ctx->prof_pending_k = 0;
    return TSAT_OK;
}

tsat_status read_info(tsat_ctx ctx, tsat_step_info* out) {
    CK(cudaMemcpyAsync(ctx->h_scal, ctx->ws + ctx->L.scal, sizeof(DevScalars), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    tsat_status s = collect_profile(ctx);
    if (s != TSAT_OK) return s;
    const DevScalars& d = *ctx->h_scal;
    if (d.xerr) {
        ctx->poisoned = TSAT_E_NCCL;
        return fail(ctx, TSAT_E_NCCL, "peer exchange timed out");
    }
    if (out) {
        out->t = ctx->t;
        out->best_unsat = d.info_best_unsat;
        out->best_idx = d.info_best_idx;
        out->solved = d.sol_step >= 0 ? 1 : 0;
        out->solved_step = d.sol_step;
        out->solved_idx = d.sol_step >= 0 ? d.sol_idx : -1;
        out->loss = d.info_loss;
    }
    return TSAT_OK;
}

}  // namespace

// =====================================================================
extern "C" {

tsat_status tsat_config_default(tsat_config* out) {
    if (!out) return TSAT_E_ARG;
    out->tau = 1.0;
    out->normalize = 1;
    out->beta1 = 0.9;
    out->beta2 = 0.999;
    out->eps = 1e-8;
    out->weight_decay = 1e-2;
    out->lr0 = 1e-1;
    out->lr_min = 1e-15;
    out->decay_factor = 10.0;
    out->decay_every = 30;
    out->restart_every = 360;
    out->noise_sigma = 0.0;
    out->reset_moments_on_restart = 0;
    out->tau_final = 0.0;
    out->clause_eval = 0;
    out->state_fp64 = 0;
    out->eps_norm = 1e-8;
    return TSAT_OK;
}

const char* tsat_status_string(tsat_status s) {
    switch (s) {
        case TSAT_OK: return "TSAT_OK";
        case TSAT_E_ARG: return "TSAT_E_ARG";
        case TSAT_E_PARSE: return "TSAT_E_PARSE";
        case TSAT_E_RANGE: return "TSAT_E_RANGE";
        case TSAT_E_STATE: return "TSAT_E_STATE";
        case TSAT_E_OOM: return "TSAT_E_OOM";
        case TSAT_E_CUDA: return "TSAT_E_CUDA";
        case TSAT_E_NCCL: return "TSAT_E_NCCL";
        case TSAT_E_UNSUPPORTED: return "TSAT_E_UNSUPPORTED";
    }
    return "TSAT_E_?";
}

tsat_status tsat_parse_dimacs(const char* text, size_t len, tsat_cnf_info* info) {
    return no_throw(nullptr, [&]() -> tsat_status {
        if (!text && len) return TSAT_E_ARG;
        int32_t V;
        std::vector<int64_t> ptr;
        std::vector<int32_t> lits;
        int64_t hc, nw;
        std::string msg;
        if (parse_dimacs(text, len, &V, &ptr, &lits, &hc, &nw, &msg)) return TSAT_E_PARSE;
        HostCnf h;
        int r = build_cnf(V, (int64_t)ptr.size() - 1, ptr.data(), lits.data(), &h, &msg);
        if (r) return r == 3 ? TSAT_E_RANGE : TSAT_E_ARG;
        h.header_C = hc;
        h.n_warnings = nw;
        fill_info(h, info);
        return TSAT_OK;
    });
}

tsat_status tsat_create(tsat_ctx* out, int cuda_device, void* cuda_stream, const void* nccl_unique_id, int rank,
                        int world) {
    return no_throw(nullptr, [&]() -> tsat_status {
        if (!out) return TSAT_E_ARG;
        *out = nullptr;
        if (world < 1 || rank < 0 || rank >= world) return TSAT_E_ARG;
        if (world > 1 && !nccl_unique_id) return TSAT_E_ARG;
        DevGuard dev_guard_(cuda_device);
        std::unique_ptr<tsat_ctx_s> c(new tsat_ctx_s());
        c->device = cuda_device;
        c->stream = (cudaStream_t)cuda_stream;
        c->rank = rank;
        c->world = world;
        tsat_ctx ctx = c.get();
        CK(cudaSetDevice(cuda_device));
        CK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
        CK(cudaMallocHost(&c->h_steptab, 2 * sizeof(StepScalars) * kMaxStepsPerCall));
        for (auto& e : c->tab_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaMallocHost(&c->h_scal, sizeof(DevScalars)));
        tsat_config_default(&c->cfg);
        if (nccl_unique_id) {           // candidate-sharded path (also with a 1-rank communicator)
            std::string err;
            if (comm_init(&c->comm, nccl_unique_id, rank, world, &err)) {
                cudaStreamDestroy(c->cap_stream);
                cudaFreeHost(c->h_steptab);
                cudaFreeHost(c->h_scal);
                return TSAT_E_NCCL;
            }
            c->sharded = true;
        }
        *out = c.release();
        return TSAT_OK;
    });
}

tsat_status tsat_create_peer(tsat_ctx* out, int cuda_device, void* cuda_stream, int rank, int world) {
    return no_throw(nullptr, [&]() -> tsat_status {
        if (!out) return TSAT_E_ARG;
        *out = nullptr;
        if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world) return TSAT_E_ARG;
        DevGuard dev_guard_(cuda_device);
        std::unique_ptr<tsat_ctx_s> c(new tsat_ctx_s());
        c->device = cuda_device;
        c->stream = (cudaStream_t)cuda_stream;
        c->rank = rank;
        c->world = world;
        c->peer = true;
        tsat_ctx ctx = c.get();
        CK(cudaSetDevice(cuda_device));
        CK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
        CK(cudaMallocHost(&c->h_steptab, 2 * sizeof(StepScalars) * kMaxStepsPerCall));
        for (auto& e : c->tab_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaMallocHost(&c->h_scal, sizeof(DevScalars)));
        tsat_config_default(&c->cfg);
        *out = c.release();
        return TSAT_OK;
    });
}

tsat_status tsat_peer_handle(tsat_ctx ctx, void* out, size_t bytes) {
    GUARD_CTX();
    if (!ctx->peer) return fail(ctx, TSAT_E_STATE, "not a peer context (tsat_create_peer)");
    if (!out || bytes < TSAT_PEER_HANDLE_BYTES) return fail(ctx, TSAT_E_ARG, "handle buffer too small");
    if (!ctx->xbuf) return fail(ctx, TSAT_E_STATE, "no CNF loaded (the exchange buffer is sized by V)");
    static_assert(sizeof(cudaIpcMemHandle_t) == TSAT_PEER_HANDLE_BYTES, "IPC handle size");
    memcpy(out, &ctx->xhandle, sizeof(cudaIpcMemHandle_t));
    return TSAT_OK;
}

tsat_status tsat_peer_open(tsat_ctx ctx, const void* handles, size_t bytes) {
    GUARD_CTX();
    if (!ctx->peer) return fail(ctx, TSAT_E_STATE, "not a peer context (tsat_create_peer)");
    if (!handles || bytes != (size_t)ctx->world * TSAT_PEER_HANDLE_BYTES)
        return fail(ctx, TSAT_E_ARG, "expected world * TSAT_PEER_HANDLE_BYTES bytes of handles");
    if (!ctx->xbuf) return fail(ctx, TSAT_E_STATE, "no CNF loaded");
    CK(cudaSetDevice(ctx->device));
    for (int r = 0; r < kMaxPeers; ++r) {
        if (ctx->peer_ipc[r] && ctx->peer_ptr[r]) cudaIpcCloseMemHandle(ctx->peer_ptr[r]);
        ctx->peer_ipc[r] = false;
        ctx->peer_ptr[r] = nullptr;
    }
    for (int r = 0; r < ctx->world; ++r) {
        cudaIpcMemHandle_t h;
        memcpy(&h, (const char*)handles + (size_t)r * TSAT_PEER_HANDLE_BYTES, sizeof(h));
        if (r == ctx->rank) {
            if (memcmp(&h, &ctx->xhandle, sizeof(h)) != 0)
                return fail(ctx, TSAT_E_ARG, "handle of this rank does not match tsat_peer_handle");
            ctx->peer_ptr[r] = (char*)ctx->xbuf;
            continue;
        }
        void* p = nullptr;
        {
            std::lock_guard<std::mutex> lk(g_xreg_mu);
            auto it = g_xreg.find(handle_key(h));
            if (it != g_xreg.end()) p = it->second;
        }
        if (!p) {
            CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            ctx->peer_ipc[r] = true;
        }
        ctx->peer_ptr[r] = (char*)p;
    }
    ctx->peers_ready = true;
    return TSAT_OK;
}

tsat_status tsat_nccl_unique_id(void* out, size_t bytes) {
    if (!out || bytes < 128) return TSAT_E_ARG;
    std::string err;
    return comm_unique_id(out, &err) ? TSAT_E_NCCL : TSAT_OK;
}

tsat_status tsat_load_dimacs(tsat_ctx ctx, const char* text, size_t len, tsat_cnf_info* info) {
    return no_throw(ctx, [&]() -> tsat_status {
        GUARD_CTX();
        if (!text && len) return fail(ctx, TSAT_E_ARG, "null text");
        int32_t V;
        std::vector<int64_t> ptr;
        std::vector<int32_t> lits;
        int64_t hc, nw;
        std::string msg;
        if (parse_dimacs(text, len, &V, &ptr, &lits, &hc, &nw, &msg)) return fail(ctx, TSAT_E_PARSE, msg);
        HostCnf h;
        int r = build_cnf(V, (int64_t)ptr.size() - 1, ptr.data(), lits.data(), &h, &msg);
        if (r) return fail(ctx, r == 3 ? TSAT_E_RANGE : TSAT_E_ARG, msg);
        h.header_C = hc;
        h.n_warnings = nw;
        fill_info(h, info);
        return upload_cnf(ctx, std::move(h));
    });
}

tsat_status tsat_load_clauses(tsat_ctx ctx, int32_t V, int64_t C, const int64_t* clause_ptr, const int32_t* lits,
                              tsat_cnf_info* info) {
    return no_throw(ctx, [&]() -> tsat_status {
        GUARD_CTX();
        std::string msg;
        HostCnf h;
        int r = build_cnf(V, C, clause_ptr, lits, &h, &msg);
        if (r) return fail(ctx, r == 3 ? TSAT_E_RANGE : TSAT_E_ARG, msg);
        fill_info(h, info);
        return upload_cnf(ctx, std::move(h));
    });
}

tsat_status tsat_workspace_bytes(tsat_ctx ctx, int64_t N_global, size_t* bytes) {
    GUARD_CTX();
    if (!bytes) return fail(ctx, TSAT_E_ARG, "null bytes");
    if (!ctx->have_cnf) return fail(ctx, TSAT_E_STATE, "no CNF loaded");
    if (N_global <= 0 || N_global % (32LL * ctx->world) != 0)
        return fail(ctx, TSAT_E_ARG, "N_global must be a positive multiple of 32 * world");
    int64_t N = N_global / ctx->world;
    if (N_global >= (1LL << 32)) return fail(ctx, TSAT_E_RANGE, "N_global >= 2^32");
    if ((int64_t)ctx->cnf.V * (N / 32) >= (1LL << 31))
        return fail(ctx, TSAT_E_RANGE, "V * N / 32 >= 2^31 (32-bit bit-plane offsets)");
    int KB = bins_for_K(ctx->cnf.K);
    bool chunked = false;
    tsat_status s = batch_chunked(ctx, (int)N, KB, &chunked);
    if (s != TSAT_OK) return s;
    if (chunked && ctx->peer)
        return fail(ctx, TSAT_E_RANGE, "peer path: N per GPU too large for the fused kernel (use more GPUs)");
    *bytes = make_layout(ctx->cnf.V, (int)N, KB, ctx->cnf.n_hubs, ctx->sharded || chunked, ctx->peer).total;
    return TSAT_OK;
}

tsat_status tsat_init_batch(tsat_ctx ctx, int64_t N_global, uint64_t seed, const tsat_config* cfg, void* ws,
                            size_t bytes) {
    nvtxRangePushA("tsat_init_batch");
    struct PopOnExit { ~PopOnExit() { nvtxRangePop(); } } pop_;
    return no_throw(ctx, [&]() -> tsat_status {
        GUARD_CTX();
        size_t need;
        tsat_status s = tsat_workspace_bytes(ctx, N_global, &need);
        if (s != TSAT_OK) return s;
        if (!ws || bytes < need) return fail(ctx, TSAT_E_OOM, "workspace too small");
        if ((uintptr_t)ws % 256) return fail(ctx, TSAT_E_ARG, "workspace must be 256-byte aligned");
        if (ctx->peer && !ctx->peers_ready) return fail(ctx, TSAT_E_STATE, "peer context: call tsat_peer_open first");
        tsat_config c;
        if (cfg) c = *cfg; else tsat_config_default(&c);
        if (!(c.tau > 0) || !(c.tau_final >= 0) || c.decay_every < 1 || c.restart_every < 1 || !(c.decay_factor > 0) || !(c.eps_norm > 0) ||
            c.normalize < 0 || c.normalize > 3 || (c.reset_moments_on_restart & ~1))
            return fail(ctx, TSAT_E_ARG, "invalid config");
        drop_graphs(ctx);
        ctx->cfg = c;
        ctx->N_global = N_global;
        ctx->N = (int)(N_global / ctx->world);
        ctx->n0 = (long long)ctx->rank * ctx->N;
        ctx->KB = bins_for_K(ctx->cnf.K);
        ctx->seed = seed;
        ctx->ws = (char*)ws;
        ctx->ws_bytes = bytes;
        {
            bool ch = false;
            int cl = 0;
            tsat_status s2 = batch_chunked(ctx, ctx->N, ctx->KB, &ch, &cl);
            if (s2 != TSAT_OK) return s2;
            ctx->chunked = ch;
            ctx->upd_cl = cl;
            // length-segmented clause evaluation: every K <= 7 instance but
            // uniform 3-SAT (its tuned kernel reads the CSR directly), >= 1024
            // candidates per GPU (the padded kernel's sub-groups serve below)
            ctx->use_seg = TSAT_SEG && ctx->dcnf.seg_lit && ctx->cnf.K <= 7 &&
                           !(ctx->cnf.uniform_len && ctx->cnf.K <= 3) && ctx->N >= 1024 && !std::getenv("TSAT_NO_SEG");
        }
        if (ctx->chunked && ctx->peer)
            return fail(ctx, TSAT_E_RANGE, "peer path: N per GPU too large for the fused kernel (use more GPUs)");
        ctx->L = make_layout(ctx->cnf.V, ctx->N, ctx->KB, ctx->cnf.n_hubs, ctx->sharded || ctx->chunked, ctx->peer);
        MethodConsts& mc = ctx->mc;
        mc = MethodConsts{};
        for (int d = 0; d < 16; ++d) mc.E[d] = std::exp(-c.tau * (double)d);
        mc.tau = c.tau;
        mc.eps_norm = c.eps_norm;
        mc.normalize = c.normalize;                 // 0 off, 1 global, 2 per shard, 3 global mean magnitude (R28)
        mc.K = ctx->cnf.K;
        mc.Nnorm = c.normalize == 2 ? N_global / ctx->world : N_global;
        mc.n0 = ctx->n0;
        mc.seed = seed;
        mc.noise = c.noise_sigma != 0.0;
        {   // fixed-point loss scale: N_global * K * 2^e < 2^61, e <= 40
            int e = 40;
            const double bound = (double)N_global * (double)std::max(ctx->cnf.K, 1);
            while (e > -60 && std::ldexp(bound, e) >= std::ldexp(1.0, 61)) --e;
            mc.loss_scale = std::ldexp(1.0, e);
            mc.loss_unscale = std::ldexp(1.0, -e);
        }
        ctx->t = 0;
        ctx->steps_done = 0;
        CK(cudaSetDevice(ctx->device));
        // fp64 state (f2, R30): library-owned 48 B per (v, n) + G, fp64 g table, row partials
        free_fp64(ctx);
        if (c.state_fp64) {
            if (c.state_fp64 != 1) return fail(ctx, TSAT_E_ARG, "state_fp64 must be 0 or 1");
            if (ctx->world > 1 || ctx->sharded || ctx->peer || ctx->chunked)
                return fail(ctx, TSAT_E_UNSUPPORTED, "state_fp64: one GPU, fused path only");
            const size_t VN = (size_t)ctx->cnf.V * ctx->N, nb = (size_t)fp64_blocks_per_row(ctx->N);
            const size_t V1 = (size_t)std::max(ctx->cnf.V, 1);
            CK(cudaMalloc(&ctx->th64, std::max<size_t>(VN, 1) * 8));
            CK(cudaMalloc(&ctx->m64, std::max<size_t>(VN, 1) * 8));
            CK(cudaMalloc(&ctx->v64, std::max<size_t>(VN, 1) * 8));
            CK(cudaMalloc(&ctx->G64, std::max<size_t>(VN, 1) * 8));
            CK(cudaMalloc(&ctx->gt64, (size_t)ctx->KB * ctx->N * 8));
            CK(cudaMalloc(&ctx->J64, V1 * 8));
            CK(cudaMalloc(&ctx->Qp64, V1 * nb * 16));
            CK(cudaMalloc(&ctx->Pw64, V1 * (ctx->N / 32) * 4));
            CK(cudaMalloc(&ctx->Nw64, V1 * (ctx->N / 32) * 4));
            CK(cudaMemset(ctx->J64, 0, V1 * 8));
            CK(cudaMemset(ctx->G64, 0, std::max<size_t>(VN, 1) * 8));
        }
        // dense clause evaluation (f4 experiment): P (C x 2V) and A (N x 2V) as uint8, K-major
        cudaFree(ctx->dP);
        cudaFree(ctx->dAL);
        ctx->dP = ctx->dAL = nullptr;
        if (c.clause_eval == 1 && ctx->cnf.C > 0) {
            const long long Kp = ((2LL * ctx->cnf.V + 31) / 32) * 32;
            const long long Cp = (ctx->cnf.C + dense_tile_m() - 1) / dense_tile_m() * dense_tile_m();
            const long long Np = ((long long)ctx->N + dense_tile_n() - 1) / dense_tile_n() * dense_tile_n();
            if (Kp * Cp >= (1LL << 31) || Kp * Np >= (1LL << 31))
                return fail(ctx, TSAT_E_RANGE, "clause_eval = 1: dense P or A above 2^31 bytes");
            std::vector<uint8_t> hp((size_t)(Kp * Cp), 0);
            for (int64_t cc = 0; cc < ctx->cnf.C; ++cc)
                for (uint32_t i = ctx->cnf.clause_ptr[cc]; i < ctx->cnf.clause_ptr[cc + 1]; ++i)
                    hp[(size_t)cc * Kp + ctx->cnf.clause_lit[i]] = 1;     // column = literal code 2v + neg
            CK(cudaMalloc(&ctx->dP, hp.size()));
            CK(cudaMalloc(&ctx->dAL, (size_t)(Kp * Np)));
            CK(cudaMemcpy(ctx->dP, hp.data(), hp.size(), cudaMemcpyHostToDevice));
            CK(cudaMemset(ctx->dAL, 0, (size_t)(Kp * Np)));
            ctx->dKp = (int)Kp;
            ctx->dCp = (int)Cp;
        } else if (c.clause_eval != 0 && c.clause_eval != 1) {
            return fail(ctx, TSAT_E_ARG, "clause_eval must be 0 or 1");
        }
        // 6-plane counters for the K <= 3 fused kernel when no row has more than
        // 31 same-sign occurrences (the counters hold cneg - cpos per bin)
        // (measured: c2 k_update -2.4 %; where the bit planes exceed L2 - c3,
        // c5 - the extra warps' HBM gathers make it slower, so only when the
        // planes are L2-resident: both buffers below 48 MB)
        ctx->upd_cw6 = 0;
        const bool planes_l2 = 2.0 * 4.0 * ((double)ctx->cnf.V + 1.0) * (double)(ctx->N / 32) <= 48.0e6;
#ifndef TSAT_PEER_CW6
#define TSAT_PEER_CW6 0                 // 1: the peer kernel with 6-plane counters too (c2 peer k_update 0.278 -> 0.281 ms: not used)
#endif
        if (ctx->cnf.K <= 3 && planes_l2 && !ctx->sharded && !ctx->chunked && (TSAT_PEER_CW6 || !ctx->peer) &&
            !std::getenv("TSAT_NO_CW6")) {
            int mx = 0;
            for (int v = 0; v < ctx->cnf.V; ++v)
                if (ctx->cnf.hub_of[v] < 0) mx = std::max({mx, ctx->cnf.occ_pn[2 * v], ctx->cnf.occ_pn[2 * v + 1]});
            ctx->upd_cw6 = mx <= 31 ? 1 : 0;
        }
        // row blocks for small shards (fused W = 1 and peer paths): RB rows per
        // work item, staging capacity = max over blocks of the non-hub rows' records
        ctx->upd_RB = 1;
        ctx->upd_blk_cap = 0;
        if (!ctx->sharded && !ctx->chunked && !std::getenv("TSAT_NO_BLK")) {
            const int RB = update_block_rows(ctx->N);
            if (RB > 1) {
                // block order: consecutive variables (the kernel then needs no
                // row list).  TSAT_BLK_SORT=1: rows grouped by their gather
                // length (the RB rows a warp gathers at once finish together)
                // through a row list - measured slower (c3 N = 128 k_update
                // 1.16 vs 1.11 ms, N = 256 2.04 vs 1.95 ms): the indirection and
                // lost row locality cost more than the divergence it removes.
                const HostCnf& h = ctx->cnf;
                const std::vector<uint32_t>& ptr = h.batched ? h.bat_ptr : h.occ_ptr;
                const int V = h.V;
                std::vector<int> order((size_t)V);
                for (int v = 0; v < V; ++v) order[v] = v;
                auto glen = [&](int v) -> long long {
                    if (h.hub_of[v] >= 0) return -1;
                    if (!h.batched) return (h.occ_pn[2 * v] + 3) / 4 + (h.occ_pn[2 * v + 1] + 3) / 4;
                    return (long long)(ptr[v + 1] - ptr[v]);
                };
                const bool sorted = std::getenv("TSAT_BLK_SORT") != nullptr;
                if (sorted)
                    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return glen(x) < glen(y); });
                long long cap = 0;
                for (int b0 = 0; b0 < V; b0 += RB) {
                    long long w = 0;
                    for (int i = b0; i < std::min(V, b0 + RB); ++i) {
                        const int v = order[i];
                        if (h.hub_of[v] < 0) w += ptr[v + 1] - ptr[v];
                    }
                    cap = std::max(cap, w);
                }
                cudaFree(ctx->blk_rows);
                ctx->blk_rows = nullptr;
                if (sorted) {
                    CK(cudaMalloc(&ctx->blk_rows, (size_t)std::max(V, 1) * sizeof(int)));
                    CK(cudaMemcpy(ctx->blk_rows, order.data(), (size_t)V * sizeof(int), cudaMemcpyHostToDevice));
                }
                ctx->upd_RB = RB;
                ctx->upd_blk_cap = (int)std::max(64LL, (cap + 63) / 64 * 64);
            }
        }
        {
            StepArgs g = step_args(ctx);
            CK(configure_kernels(&g));
            ctx->upd_mode = g.upd_mode;
            ctx->upd_GT = g.upd_GT;
            ctx->upd_recbufs = g.upd_recbufs;
            ctx->upd_NG = g.upd_NG;
            ctx->upd_grid = g.upd_grid;
            ctx->upd_prefetch = g.upd_prefetch;
            ctx->upd_smem = g.upd_smem;
            ctx->num_sms = g.num_sms;
            ctx->upd_chunk = g.upd_chunk;
            ctx->upd_gs_global = g.upd_gs_global;
        }
        if (ctx->chunked != (ctx->upd_chunk < ctx->N && ctx->upd_cl <= 1))
            return fail(ctx, TSAT_E_STATE, "internal: chunking decision changed between layout and launch");
        StepArgs a = step_args(ctx);
        if (ctx->L.hubD != ctx->L.total)
            CK(cudaMemsetAsync(ctx->ws + ctx->L.hubD, 0, ctx->L.total - ctx->L.hubD, ctx->stream));
        CK(cudaMemsetAsync(ctx->ws + ctx->L.hist, 0, (size_t)ctx->N * ctx->KB * 4, ctx->stream));
        CK(cudaMemsetAsync(ctx->ws + ctx->L.scal, 0, sizeof(DevScalars), ctx->stream));
        {
            const size_t rowb = (size_t)(ctx->N / 32) * 4, zoff = (size_t)ctx->cnf.V * rowb;
            CK(cudaMemsetAsync(ctx->ws + ctx->L.A0 + zoff, 0, rowb, ctx->stream));
            CK(cudaMemsetAsync(ctx->ws + ctx->L.A1 + zoff, 0, rowb, ctx->stream));
        }
        DevScalars init{};
        init.best_key = ~0ull;
        init.sol_step = -1;
        init.sol_idx = -1;
        init.info_best_unsat = -1;
        init.info_best_idx = -1;
        *ctx->h_scal = init;
        CK(cudaMemcpyAsync(a.ds, ctx->h_scal, sizeof(DevScalars), cudaMemcpyHostToDevice, ctx->stream));
        if (a.fp64) CK(launch_init64(a, seed, ctx->stream));
        else CK(launch_init(a.theta, a.m, a.v, a.V, a.N, ctx->n0, seed, ctx->stream));
        s = state_stats(ctx, a, 0);
        if (s != TSAT_OK) return s;
        ctx->have_batch = true;
        return TSAT_OK;
    });
}

tsat_status tsat_step(tsat_ctx ctx, int32_t k, tsat_step_info* out) {
    return no_throw(ctx, [&]() -> tsat_status {
        GUARD_CTX();
        tsat_status s = check_batch(ctx, false);
        if (s != TSAT_OK) return s;
        if (k < 1) return fail(ctx, TSAT_E_ARG, "k < 1");
        struct NvtxRange {                              // one range per tsat_step call (profiling timelines)
            explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
            ~NvtxRange() { nvtxRangePop(); }
        } nvtx_range_("tsat_step");
        int done = 0;
        while (done < k) {
            int kk = std::min(k - done, kMaxStepsPerCall);
            if (ctx->profiling) {                       // the previous call's kernel events
                CK(cudaStreamSynchronize(ctx->stream));
                s = collect_profile(ctx);
                if (s != TSAT_OK) return s;
            }
            // the device table is rewritten in stream order (after the previous
            // graph has used it); the host slot only once its last upload is done,
            // so consecutive calls queue without draining the GPU
            const int slot = ctx->tab_slot;
            ctx->tab_slot ^= 1;
            CK(cudaEventSynchronize(ctx->tab_ev[slot]));
            StepScalars* tab = ctx->h_steptab + (size_t)slot * kMaxStepsPerCall;
            for (int i = 0; i < kk; ++i) {
                tab[i] = step_scalars(ctx->cfg, ctx->t + i);
                tab[i].xgen = ctx->xgen + 1 + (unsigned)i;
            }
            CK(cudaMemcpyAsync(ctx->ws + ctx->L.steptab, tab, sizeof(StepScalars) * kk, cudaMemcpyHostToDevice,
                               ctx->stream));
            CK(cudaEventRecord(ctx->tab_ev[slot], ctx->stream));
            s = launch_steps(ctx, kk);
            if (s != TSAT_OK) return s;
            ctx->t += kk;
            ctx->steps_done += kk;
            ctx->xgen += (unsigned)kk;
            done += kk;
        }
        if (out) return read_info(ctx, out);
        return TSAT_OK;
    });
}

tsat_status tsat_get_info(tsat_ctx ctx, tsat_step_info* out) {
    GUARD_CTX();
    tsat_status s = check_batch(ctx, false);
    if (s != TSAT_OK) return s;
    return read_info(ctx, out);
}

tsat_status tsat_query_unsat_async(tsat_ctx ctx, int32_t* host_out, size_t n, int64_t* first) {
    GUARD_CTX();
    tsat_status s = check_batch(ctx, true);
    if (s != TSAT_OK) return s;
    if (!host_out) return fail(ctx, TSAT_E_ARG, "null host_out");
    if (n != (size_t)ctx->N) return fail(ctx, TSAT_E_ARG, "host_out must hold exactly N_local counts");
    CK(cudaMemcpyAsync(host_out, ctx->ws + ctx->L.unsat, (size_t)ctx->N * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (first) *first = ctx->n0;
    return TSAT_OK;
}

tsat_status tsat_sync(tsat_ctx ctx) {
    GUARD_CTX();
    CK(cudaStreamSynchronize(ctx->stream));
    return collect_profile(ctx);
}

tsat_status tsat_query_unsat(tsat_ctx ctx, int32_t* host_out, size_t n, int64_t* first) {
    GUARD_CTX();
    tsat_status s = check_batch(ctx, true);
    if (s != TSAT_OK) return s;
    if (!host_out) return fail(ctx, TSAT_E_ARG, "null host_out");
    if (n != (size_t)ctx->N) return fail(ctx, TSAT_E_ARG, "host_out must hold exactly N_local counts");
    CK(cudaMemcpyAsync(host_out, ctx->ws + ctx->L.unsat, (size_t)ctx->N * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (first) *first = ctx->n0;
    return TSAT_OK;
}

tsat_status tsat_export_model(tsat_ctx ctx, int64_t gidx, uint8_t* host_values) {
    return no_throw(ctx, [&]() -> tsat_status {
        GUARD_CTX();
        tsat_status s = check_batch(ctx, true);
        if (s != TSAT_OK) return s;
        if (!host_values) return fail(ctx, TSAT_E_ARG, "null host_values");
        int64_t n = gidx - ctx->n0;
        if (n < 0 || n >= ctx->N) return fail(ctx, TSAT_E_ARG, "candidate not on this rank");
        const int V = ctx->cnf.V, NW = ctx->N / 32;
        size_t Aoff = ((ctx->t - 1) & 1) ? ctx->L.A1 : ctx->L.A0;    // evaluated state theta_{t-1}
        std::vector<uint32_t> words((size_t)V);
        if (V > 0) {
            CK(cudaMemcpy2DAsync(words.data(), 4, ctx->ws + Aoff + (size_t)(n / 32) * 4, (size_t)NW * 4, 4, (size_t)V,
                                 cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
        }
        for (int v = 0; v < V; ++v) host_values[v] = (uint8_t)((words[v] >> (n & 31)) & 1u);
        return TSAT_OK;
    });
}

tsat_status tsat_get_solution(tsat_ctx ctx, uint8_t* host_values, int64_t* idx, int64_t* step) {
    return no_throw(ctx, [&]() -> tsat_status {
        GUARD_CTX();
        tsat_status s = check_batch(ctx, false);
        if (s != TSAT_OK) return s;
        s = read_info(ctx, nullptr);
        if (s != TSAT_OK) return s;
        const DevScalars& d = *ctx->h_scal;
        if (d.sol_step < 0) return fail(ctx, TSAT_E_STATE, "no model found yet");
        if (idx) *idx = d.sol_idx;
        if (step) *step = d.sol_step;
        const bool owner = d.sol_idx >= ctx->n0 && d.sol_idx < ctx->n0 + ctx->N;
        if (host_values && ctx->cnf.V > 0 && owner) {
            CK(cudaMemcpyAsync(host_values, ctx->ws + ctx->L.sol, (size_t)ctx->cnf.V, cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
        }
        return TSAT_OK;
    });
}

tsat_status tsat_get_state64(tsat_ctx ctx, double* theta, double* m, double* v, size_t elems, int64_t* t) {
    GUARD_CTX();
    tsat_status s = check_batch(ctx, false);
    if (s != TSAT_OK) return s;
    if (!ctx->th64) return fail(ctx, TSAT_E_STATE, "the batch has fp32 state: use tsat_get_state");
    if ((theta || m || v) && elems != (size_t)ctx->cnf.V * ctx->N)
        return fail(ctx, TSAT_E_ARG, "state arrays must hold exactly V * N_local elements");
    const size_t bytes = (size_t)ctx->cnf.V * ctx->N * 8;
    if (theta) CK(cudaMemcpyAsync(theta, ctx->th64, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    if (m) CK(cudaMemcpyAsync(m, ctx->m64, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    if (v) CK(cudaMemcpyAsync(v, ctx->v64, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (t) *t = ctx->t;
    return TSAT_OK;
}

tsat_status tsat_set_state64(tsat_ctx ctx, const double* theta, const double* m, const double* v, size_t elems,
                             int64_t t) {
    GUARD_CTX();
    tsat_status s = check_batch(ctx, false);
    if (s != TSAT_OK) return s;
    if (!ctx->th64) return fail(ctx, TSAT_E_STATE, "the batch has fp32 state: use tsat_set_state");
    if (!theta || !m || !v || t < 0) return fail(ctx, TSAT_E_ARG, "null state or t < 0");
    if (elems != (size_t)ctx->cnf.V * ctx->N) return fail(ctx, TSAT_E_ARG, "state arrays must hold exactly V * N_local elements");
    const size_t bytes = (size_t)ctx->cnf.V * ctx->N * 8;
    StepArgs a = step_args(ctx);
    CK(cudaMemcpyAsync(ctx->th64, theta, bytes, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->m64, m, bytes, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->v64, v, bytes, cudaMemcpyHostToDevice, ctx->stream));
    DevScalars init{};
    init.best_key = ~0ull;
    init.sol_step = -1;
    init.sol_idx = -1;
    init.info_best_unsat = -1;
    init.info_best_idx = -1;
    CK(cudaStreamSynchronize(ctx->stream));
    *ctx->h_scal = init;
    CK(cudaMemcpyAsync(a.ds, ctx->h_scal, sizeof(DevScalars), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(a.hist, 0, (size_t)ctx->N * ctx->KB * 4, ctx->stream));
    CK(cudaMemsetAsync(ctx->J64, 0, (size_t)std::max(ctx->cnf.V, 1) * 8, ctx->stream));
    s = state_stats(ctx, a, t);
    if (s != TSAT_OK) return s;
    ctx->t = t;
    ctx->steps_done = 0;
    return TSAT_OK;
}

tsat_status tsat_get_state(tsat_ctx ctx, float* theta, float* m, float* v, size_t elems, int64_t* t) {
    GUARD_CTX();
    tsat_status s = check_batch(ctx, false);
    if (s != TSAT_OK) return s;
    if (ctx->th64) return fail(ctx, TSAT_E_STATE, "the batch has fp64 state: use tsat_get_state64");
    if ((theta || m || v) && elems != (size_t)ctx->cnf.V * ctx->N)
        return fail(ctx, TSAT_E_ARG, "state arrays must hold exactly V * N_local elements");
    size_t bytes = (size_t)ctx->cnf.V * ctx->N * 4;
    if (theta) CK(cudaMemcpyAsync(theta, ctx->ws + ctx->L.theta, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    if (m) CK(cudaMemcpyAsync(m, ctx->ws + ctx->L.m, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    if (v) CK(cudaMemcpyAsync(v, ctx->ws + ctx->L.v, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (t) *t = ctx->t;
    return TSAT_OK;
}

tsat_status tsat_set_state(tsat_ctx ctx, const float* theta, const float* m, const float* v, size_t elems, int64_t t) {
    GUARD_CTX();
    tsat_status s = check_batch(ctx, false);
    if (s != TSAT_OK) return s;
    if (ctx->th64) return fail(ctx, TSAT_E_STATE, "the batch has fp64 state: use tsat_set_state64");
    if (!theta || !m || !v || t < 0) return fail(ctx, TSAT_E_ARG, "null state or t < 0");
    if (elems != (size_t)ctx->cnf.V * ctx->N)
        return fail(ctx, TSAT_E_ARG, "state arrays must hold exactly V * N_local elements (same world size and N)");
    size_t bytes = (size_t)ctx->cnf.V * ctx->N * 4;
    StepArgs a = step_args(ctx);
    CK(cudaMemcpyAsync(a.theta, theta, bytes, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(a.m, m, bytes, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(a.v, v, bytes, cudaMemcpyHostToDevice, ctx->stream));
    DevScalars init{};
    init.best_key = ~0ull;
    init.sol_step = -1;
    init.sol_idx = -1;
    init.info_best_unsat = -1;
    init.info_best_idx = -1;
    CK(cudaStreamSynchronize(ctx->stream));
    *ctx->h_scal = init;
    CK(cudaMemcpyAsync(a.ds, ctx->h_scal, sizeof(DevScalars), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(a.hist, 0, (size_t)ctx->N * ctx->KB * 4, ctx->stream));
    s = state_stats(ctx, a, t);
    if (s != TSAT_OK) return s;
    ctx->t = t;
    ctx->steps_done = 0;
    return TSAT_OK;
}

tsat_status tsat_get_rows(tsat_ctx ctx, const int32_t* rows, int32_t nrows, float* theta, float* m, float* v,
                          size_t row_elems) {
    GUARD_CTX();
    tsat_status s = check_batch(ctx, false);
    if (s != TSAT_OK) return s;
    if (row_elems != (size_t)ctx->N) return fail(ctx, TSAT_E_ARG, "row_elems must equal N_local");
    if (ctx->th64) return fail(ctx, TSAT_E_STATE, "the batch has fp64 state (use tsat_get_state64)");
    if (nrows < 0 || (nrows > 0 && !rows)) return fail(ctx, TSAT_E_ARG, "bad rows");
    const size_t rb = (size_t)ctx->N * 4;
    for (int32_t i = 0; i < nrows; ++i) {
        if (rows[i] < 0 || rows[i] >= ctx->cnf.V) return fail(ctx, TSAT_E_ARG, "row out of range");
        const size_t off = (size_t)rows[i] * rb;
        if (theta) CK(cudaMemcpyAsync((char*)theta + i * rb, ctx->ws + ctx->L.theta + off, rb, cudaMemcpyDeviceToHost, ctx->stream));
        if (m) CK(cudaMemcpyAsync((char*)m + i * rb, ctx->ws + ctx->L.m + off, rb, cudaMemcpyDeviceToHost, ctx->stream));
        if (v) CK(cudaMemcpyAsync((char*)v + i * rb, ctx->ws + ctx->L.v + off, rb, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return TSAT_OK;
}

tsat_status tsat_debug_copy(tsat_ctx ctx, int32_t which, void* dst, size_t bytes) {
    GUARD_CTX();
    tsat_status s = check_batch(ctx, false);
    if (s != TSAT_OK) return s;
    if (!dst) return fail(ctx, TSAT_E_ARG, "null dst");
    size_t off, sz;
    const int N = ctx->N, V = ctx->cnf.V;
    switch (which) {
        case 0: return fail(ctx, TSAT_E_UNSUPPORTED, "histogram is cleared after use; query unsat instead");
        case 1: off = ctx->L.gtab; sz = (size_t)N * ctx->KB * 4; break;
        case 2: off = ctx->L.S; sz = (size_t)N * 8; break;
        case 3: off = ((ctx->t - 1) & 1) ? ctx->L.A1 : ctx->L.A0; sz = (size_t)V * (N / 32) * 4; break;
        case 4: off = ctx->L.rowQ; sz = (size_t)V * 8; break;
        default: return fail(ctx, TSAT_E_ARG, "unknown buffer");
    }
    if (bytes != sz) return fail(ctx, TSAT_E_ARG, "size mismatch: expected " + std::to_string(sz));
    CK(cudaMemcpyAsync(dst, ctx->ws + off, sz, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return TSAT_OK;
}

tsat_status tsat_export_best(tsat_ctx ctx, int32_t M, int32_t k, tsat_partial* out) {
    return no_throw(ctx, [&]() -> tsat_status {
        GUARD_CTX();
        tsat_status s = check_batch(ctx, true);
        if (s != TSAT_OK) return s;
        const int V = ctx->cnf.V, N = ctx->N, W = ctx->world;
        if (M < 1 || (int64_t)M > ctx->N_global || !out) return fail(ctx, TSAT_E_ARG, "need 1 <= M <= N_global and host_out");
        if (k <= 0) k = (int32_t)std::min<int64_t>(V, std::max<int64_t>((V + 9999) / 10000, 20));
        if (k > V) k = V;
        if (k > kTopkMax) return fail(ctx, TSAT_E_RANGE, "k > 2048 not supported");
        if (k < 1) return fail(ctx, TSAT_E_ARG, "V = 0");
        if (W > 1 && ((int64_t)M > kExportCap || (int64_t)M * k > kExportCap))
            return fail(ctx, TSAT_E_RANGE, "multi-GPU export: M and M * k must be <= 65536");
        StepArgs a = step_args(ctx);
        const long long t_eval = ctx->t - 1;
        int n64 = 1;
        while (n64 < std::max(N, M)) n64 <<= 1;
        // device scratch, stream-ordered (cudaMallocAsync / cudaFreeAsync never wait for the
        // device: with several ranks on one GPU a device-synchronising allocation would stall
        // behind a peer's exchange kernel that waits for this rank); freed on every path
        unsigned long long *keys = nullptr, *gk = nullptr, *ent = nullptr, *gent = nullptr;
        int *cols = nullptr, *pos = nullptr, *ov = nullptr;
        double *absG = nullptr, *og = nullptr;
        struct Free {
            cudaStream_t st;
            std::vector<void*> p;
            ~Free() { for (void* x : p) cudaFreeAsync(x, st); }
        } fr{ctx->stream, {}};
        auto dalloc = [&](void** dst, size_t bytes) -> bool {
            if (cudaMallocAsync(dst, std::max<size_t>(bytes, 8), ctx->stream) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            fr.p.push_back(*dst);
            return true;
        };
        const size_t Mk = (size_t)M * k;
        if (!dalloc((void**)&keys, (size_t)n64 * 8) || !dalloc((void**)&gk, (size_t)W * M * 8) ||
            !dalloc((void**)&ent, Mk * 8) || !dalloc((void**)&gent, (size_t)W * Mk * 8) ||
            !dalloc((void**)&cols, (size_t)M * 4) || !dalloc((void**)&pos, (size_t)M * 4) ||
            !dalloc((void**)&ov, Mk * 4) || !dalloc((void**)&og, Mk * 8) || !dalloc((void**)&absG, (size_t)M * V * 8))
            return fail(ctx, TSAT_E_OOM, "export scratch allocation failed");
        // (1) local ranking by (unsat, global index): keys padded with ~0 beyond N_local
        CK(launch_export(a, t_eval, nullptr, M, k, nullptr, keys, n64, nullptr, nullptr, ctx->stream, 0));
        // (2) all ranks' first M keys -> every rank (exact integers: identical merge everywhere)
        std::vector<unsigned long long> hk((size_t)W * M);
        auto gather = [&](int phase, const unsigned long long* send, size_t n, unsigned long long* recv) -> tsat_status {
            if (W == 1) return TSAT_OK;
            if (ctx->peer) {
                CK(launch_peer_allgather(a, phase, send, (int)n, recv, ++ctx->xgen, ctx->stream));
            } else {
                std::string err;
                if (comm_allgather_u64(ctx->comm, send, recv, n, ctx->stream, &err)) {
                    ctx->poisoned = TSAT_E_NCCL;
                    return fail(ctx, TSAT_E_NCCL, err);
                }
            }
            return TSAT_OK;
        };
        s = gather(0, keys, (size_t)M, gk);
        if (s != TSAT_OK) return s;
        CK(cudaMemcpyAsync(hk.data(), W == 1 ? keys : gk, hk.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (ctx->peer) {
            CK(cudaMemcpyAsync(ctx->h_scal, ctx->ws + ctx->L.scal, sizeof(DevScalars), cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            if (ctx->h_scal->xerr) { ctx->poisoned = TSAT_E_NCCL; return fail(ctx, TSAT_E_NCCL, "peer export exchange timed out"); }
        }
        // (3) global top-M: the M smallest keys, ascending (each key is unique: it holds the index)
        {
            std::vector<unsigned long long> sel((size_t)M);
            tsat_merge_keys(reinterpret_cast<const uint64_t*>(hk.data()), hk.size(), M,
                            reinterpret_cast<uint64_t*>(sel.data()));
            hk.swap(sel);
        }
        if (hk.back() == ~0ull) return fail(ctx, TSAT_E_STATE, "fewer than M evaluated candidates");
        // (4) the columns this rank owns: k smallest |G| per column (R14, ties -> lower v) + bits
        std::vector<int> hc, hp;
        for (int i = 0; i < M; ++i) {
            const long long g = (long long)(hk[i] & 0xffffffffull);
            if (g >= ctx->n0 && g < ctx->n0 + N) { hc.push_back((int)(g - ctx->n0)); hp.push_back(i); }
        }
        const int Mo = (int)hc.size();
        CK(cudaMemsetAsync(ent, 0, Mk * 8, ctx->stream));
        if (Mo > 0) {
            CK(cudaMemcpyAsync(cols, hc.data(), (size_t)Mo * 4, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaMemcpyAsync(pos, hp.data(), (size_t)Mo * 4, cudaMemcpyHostToDevice, ctx->stream));
            CK(launch_export(a, t_eval, cols, Mo, k, absG, keys, n64, ov, og, ctx->stream, 1));
            CK(launch_export_pack(a, t_eval, cols, pos, Mo, k, ov, og, ent, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));   // hc / hp stay alive until the copies are done
        }
        // (5) every rank receives every selected column's entries (each position has one owner)
        s = gather(1, ent, Mk, gent);
        if (s != TSAT_OK) return s;
        std::vector<unsigned long long> he((size_t)W * Mk);
        CK(cudaMemcpyAsync(he.data(), W == 1 ? ent : gent, he.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (ctx->peer) {
            CK(cudaMemcpyAsync(ctx->h_scal, ctx->ws + ctx->L.scal, sizeof(DevScalars), cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            if (ctx->h_scal->xerr) { ctx->poisoned = TSAT_E_NCCL; return fail(ctx, TSAT_E_NCCL, "peer export exchange timed out"); }
        }
        const long long Nl = N;
        for (int i = 0; i < M; ++i) {
            const long long g = (long long)(hk[i] & 0xffffffffull);
            const int owner = (int)(g / Nl);
            const unsigned long long* e = he.data() + (size_t)owner * Mk + (size_t)i * k;
            out[i].candidate = g;
            out[i].unsat = (int32_t)(hk[i] >> 32);
            out[i].k = k;
            for (int j = 0; j < k; ++j) {
                const uint32_t lo = (uint32_t)(e[j] & 0xffffffffull);
                const int v = (int)(lo >> 1);
                if (out[i].lits) out[i].lits[j] = (lo & 1u) ? (v + 1) : -(v + 1);
                if (out[i].abs_grad) out[i].abs_grad[j] = __uint_as_float_host((uint32_t)(e[j] >> 32));
            }
        }
        return TSAT_OK;
    });
}

tsat_status tsat_merge_keys(const uint64_t* keys, size_t n, int32_t M, uint64_t* out) {
    if (M < 0 || (M > 0 && (!keys || !out)) || (size_t)M > n) return TSAT_E_ARG;
    return no_throw(nullptr, [&]() -> tsat_status {
        std::vector<uint64_t> v(keys, keys + n);
        std::partial_sort(v.begin(), v.begin() + M, v.end());
        std::copy(v.begin(), v.begin() + M, out);
        return TSAT_OK;
    });
}

tsat_status tsat_export_k(tsat_ctx ctx, int32_t k_req, int32_t* k_out) {
    GUARD_CTX();
    if (!k_out) return fail(ctx, TSAT_E_ARG, "null k_out");
    if (!ctx->have_cnf) return fail(ctx, TSAT_E_STATE, "no CNF loaded");
    const int64_t V = ctx->cnf.V;
    int64_t k = k_req > 0 ? k_req : std::max<int64_t>((V + 9999) / 10000, 20);
    *k_out = (int32_t)std::min<int64_t>(k, V);
    return TSAT_OK;
}

tsat_status tsat_set_profiling(tsat_ctx ctx, int32_t enable) {
    GUARD_CTX();
    ctx->profiling = enable != 0;
    return TSAT_OK;
}

tsat_status tsat_kernel_times(tsat_ctx ctx, double* ms5, int64_t* steps) {
    GUARD_CTX();
    CK(cudaStreamSynchronize(ctx->stream));
    tsat_status s = collect_profile(ctx);
    if (s != TSAT_OK) return s;
    for (int i = 0; i < kKernelsPerStep; ++i) {
        if (ms5) ms5[i] = ctx->prof_ms[i];
        ctx->prof_ms[i] = 0;
    }
    if (steps) *steps = ctx->prof_steps;
    ctx->prof_steps = 0;
    return TSAT_OK;
}

tsat_status tsat_kernels_per_step(tsat_ctx ctx, int32_t* n) {
    GUARD_CTX();
    if (!n) return TSAT_E_ARG;
    int k = 0;
    k += 1;                                                                     // clause (or accumulator reset)
    k += 1;                                                                     // gtable
    if (ctx->have_batch && ctx->cnf.n_hub_sc > 0) ++k;                         // hub
    if (ctx->have_cnf && ctx->cnf.V > 0) ++k;                                  // update (phase A when split)
    if (ctx->have_batch && ctx->use_seg && ctx->cnf.seg_C.size() == 8) {       // clause: short + long segment kernels
        const bool s = ctx->cnf.seg_C[1] + ctx->cnf.seg_C[2] + ctx->cnf.seg_C[3] > 0;
        const bool l = ctx->cnf.seg_C[4] + ctx->cnf.seg_C[5] + ctx->cnf.seg_C[6] + ctx->cnf.seg_C[7] > 0;
        if (s && l) ++k;
    }
    if (ctx->sharded) k += 5;   // pack/unpack max, update B, rows finish, step end (NCCL's own kernels not counted)
    else if (ctx->chunked) k += 3;   // update B, rows finish, step end (+ the J reset memset)
    *n = k;
    return TSAT_OK;
}

tsat_status tsat_update_geometry(tsat_ctx ctx, int32_t* out, int32_t n_out) {
    GUARD_CTX();
    if (!out || n_out < 8) return fail(ctx, TSAT_E_ARG, "update_geometry: out must hold 8 values");
    if (!ctx->have_batch) return fail(ctx, TSAT_E_STATE, "update_geometry: no batch");
    out[0] = ctx->upd_GT;
    out[1] = ctx->upd_NG;
    out[2] = ctx->upd_grid;
    out[3] = (int32_t)ctx->upd_smem;
    out[4] = ctx->upd_chunk;
    out[5] = ctx->upd_cl;
    out[6] = ctx->upd_RB;
    out[7] = ctx->use_seg ? 1 : 0;
    return TSAT_OK;
}

const char* tsat_error_string(tsat_ctx ctx) {
    if (!ctx) return "null context";
    return ctx->err.c_str();
}

void tsat_destroy(tsat_ctx ctx) {
    if (!ctx) return;
    DevGuard dev_guard_(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    drop_graphs(ctx);
    for (auto e : ctx->events) cudaEventDestroy(e);
    free_cnf(ctx);
    cudaFree(ctx->dP);
    cudaFree(ctx->dAL);
    cudaFree(ctx->blk_rows);
    free_fp64(ctx);
    comm_destroy(ctx->comm);
    peer_release(ctx);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->cap_side) cudaStreamDestroy(ctx->cap_side);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    cudaFreeHost(ctx->h_steptab);
    cudaFreeHost(ctx->h_scal);
    for (auto e : ctx->tab_ev)
        if (e) cudaEventDestroy(e);
    delete ctx;
}

}  // extern "C"

extern "C" tsat_status tsat_lr_at(const tsat_config* cfg, int64_t t, double* lr) {
    if (!cfg || !lr || t < 0 || cfg->decay_every < 1 || cfg->restart_every < 1) return TSAT_E_ARG;
    *lr = lr_at(*cfg, t);
    return TSAT_OK;
}
