// tsat_internal.h - shared between the host runtime (capi.cu, host_cnf.cpp)
// and the sm_100a kernels.  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace tsat {

// ---------------------------------------------------------------- limits
constexpr int kMaxK = 15;              // clause length supported by the kernels (K > 7: KB = 16)
constexpr int kMaxStepsPerCall = 4096;
constexpr int kTopkMax = 2048;         // export: k most confident variables per candidate
constexpr int kRecCap = 512;           // occurrence-record words a warp group stages per row (longer rows: hubs)
constexpr int kHubSlab = 1023;         // occurrences per hub super-chunk (11-bit signed counters)
#ifndef TSAT_HUB_SLAB_BATCHES
#define TSAT_HUB_SLAB_BATCHES 63      // c4: k_hub 1.53 -> 1.35 ms vs 127 (more, shorter warps; 255: 1.89, 31: 1.39, 15: 1.60)
#endif
constexpr int kHubSlabBatches = TSAT_HUB_SLAB_BATCHES;   // batched records: batches (<= 4 occurrences) per hub super-chunk (k_hub int10)
constexpr int kMaxPeers = 8;           // peer-exchange path: ranks (GPUs of one NVSwitch node)
constexpr int kExportCap = 1 << 16;    // export exchange: u64 words per rank and phase (M and M * k)

// Peer-exchange buffer of one rank (cudaMalloc'd, CUDA-IPC shared).
// Every rank writes its slot [src = its rank] of every rank's buffer:
//   S: [2][W] x {~best key, gmax bits, thmax bits, loss S 2^e} + flags [2][W]
//      (once per step, double-buffered by generation parity)
//   J, Q: [W][V] int64 row partials, each as two self-validating u64 words
//         (generation << 32 | 32-bit half)                                   (per row, per step)
// The generation is monotone per context and identical on every rank (the
// ranks run the same call sequence).
//   E: export all-gathers (tsat_export_best): flags [2][W] + [2 phases][W][kExportCap] u64
struct PeerLayout {
    size_t sx, sf, jx, qx, ef, ex, total;
};
inline PeerLayout peer_layout(int V, int W) {
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    PeerLayout L{};
    size_t o = 0;
    L.sx = o; o = al(o + (size_t)2 * W * 32);
    L.sf = o; o = al(o + (size_t)2 * W * 4);
    L.jx = o; o = al(o + (size_t)W * V * 16);
    L.qx = o; o = al(o + (size_t)W * V * 16);
    L.ef = o; o = al(o + (size_t)2 * W * 4);
    L.ex = o; o = al(o + (size_t)2 * W * kExportCap * 8);
    L.total = o;
    return L;
}
struct PeerArgs {
    char* xb[kMaxPeers];               // every rank's buffer in this process's address space
    int W, rank, V;
    int exchange_rows;                 // 0 with normalize = 2 (per shard): J, Q stay local
    PeerLayout L;
};

// ---------------------------------------------------------------- host CNF
// Literal code used on the device: (var << 1) | negated, var 0-based.
struct HostCnf {
    int32_t V = 0;
    int64_t C = 0;
    int64_t nnz = 0;
    int32_t K = 0;
    std::vector<uint32_t> clause_ptr;   // C+1
    std::vector<uint32_t> clause_lit;   // nnz codes
    // variable -> occurrence records (canonical clause-ascending order):
    //   rec[0] = (len << 1) | own_negated, rec[1..len-1] = the other literal codes
    std::vector<uint32_t> occ_ptr;      // V+1 (word offsets into occ_rec)
    std::vector<uint32_t> occ_rec;
    std::vector<uint32_t> occ_cnt;      // V: occurrences of the variable
    std::vector<int32_t> occ_pn;        // 2V: (positive, negative) occurrences
    // hub rows: a variable whose signed per-bin counts may leave int8, or whose
    // records exceed kRecCap, is counted by the k_hub pre-pass (int32).
    std::vector<int32_t> hub_of;        // V: hub index or -1
    std::vector<int32_t> hub_sc;        // 4 per super-chunk: hub, var, rec_begin, rec_end (word offsets
                                        // into occ_rec, or into bat_rec when batched)
    int32_t n_hubs = 0;
    int32_t n_hub_sc = 0;
    int64_t header_C = -1;
    int64_t n_warnings = 0, n_tautologies = 0, n_duplicates = 0;
    int32_t has_empty = 0;
    int32_t uniform_len = 0;            // every clause has exactly K literals
    int32_t max_rec_words = 0;          // max record words k_update stages, over non-hub rows
    // batched records (host_cnf.cpp build_batched), staged by k_update for
    // every instance except uniform 3-SAT
    int32_t batched = 0;
    std::vector<uint32_t> bat_ptr;      // V+1
    std::vector<uint32_t> bat_rec;
    // length segments (build_segments, K <= 7): clauses of length L at
    // seg_lit[seg_off[L] .. + seg_C[L] * L), L = 1..7 (empty clauses in L = 1)
    std::vector<int64_t> seg_C, seg_off;
    std::vector<uint32_t> seg_lit;
};

// Parse DIMACS.  Returns 0 on success, 2 (TSAT_E_PARSE) with msg.
int parse_dimacs(const char* text, size_t len, int32_t* V, std::vector<int64_t>* ptr,
                 std::vector<int32_t>* lits, int64_t* header_C, int64_t* n_warnings, std::string* msg);
// Build HostCnf from signed-literal clause arrays (dedup, tautology count,
// codes, occurrence records, hub tables).  Returns 0, or 1 (arg) / 3 (range).
int build_cnf(int32_t V, int64_t C, const int64_t* ptr, const int32_t* lits, HostCnf* out, std::string* msg);

// ---------------------------------------------------------------- device
// Per-iteration scalars, computed on the host (libm) and uploaded per call.
struct StepScalars {
    int64_t t;        // iteration index of the evaluated state
    double lr;
    float wdf;        // (float)(1 - lr*wd)
    float a1;         // (float)(1 - beta1)
    float b2f;        // (float)beta2
    float a2;         // (float)(1 - beta2)
    float nss;        // (float)(-(lr / (1 - beta1^(t+1))))
    float rbc2;       // (float)(1 / sqrt(1 - beta2^(t+1)))  (R6c)
    float epsf;       // (float)eps
    float nz;         // (float)(lr * noise_sigma)
    float mkeep;      // 0 at a moment reset (m *= 0; b2f = 0 zeroes v), else 1
    unsigned xgen;    // peer path: exchange generation of this iteration
    int pad;
    double tau;       // SmoothMin temperature of this iteration (R1; annealed: R29)
    double E[16];     // exp(-tau d), d = 0..15 (host libm, R11)
    // fp64 state (R30): the AdamW scalars unrounded
    double wdf64, a1_64, b2_64, a2_64, nss64, rbc2_64, eps64, nz64;
};

// Device-resident scalars (one struct in the workspace).
struct DevScalars {
    unsigned long long best_key;     // min over candidates of (unsat << 32 | global idx)
    unsigned long long gmax_bits;    // max |g| (non-negative double bits)
    unsigned int thmax_bits[2];      // max |theta| of theta_t, indexed by t & 1
    int row_counter;                 // k_update dynamic row scheduler
    int pad0;
    double loss;
    long long sol_step;              // first iteration with a 0-unsat candidate (-1)
    long long sol_idx;
    long long info_t;
    int info_best_unsat;
    int pad1;
    long long info_best_idx;
    double info_loss;
    long long loss_fx;               // sharded: this rank's sum of round(S_n 2^e) (exact int64, MethodConsts)
    unsigned int gt_done;            // k_gtable blocks finished (last block does the step bookkeeping)
    unsigned int xerr;               // peer path: an exchange timed out (step result invalid)
    unsigned long long thmax64_bits[2];   // fp64 state (R30): max |theta| as fp64 bits, by t & 1
};

// Histogram bins per candidate for an instance of max clause length K: R in
// 0..KB-1 (KB = 4: 2-bit R, K <= 3; 8: 3-bit, K <= 7; 16: 4-bit, K <= 15).
inline int bins_for_K(int K) { return K <= 3 ? 4 : (K <= 7 ? 8 : 16); }

// Method constants passed by value to kernels.
struct MethodConsts {
    double E[16];       // exp(-tau d), d = 0..15 (host libm)
    double tau;
    double eps_norm;
    int normalize;
    int K;              // instance max clause length
    long long Nnorm;    // candidates Eq. 5 averages over: N (normalize 0/1) or N/W (2, per shard)
    long long n0;       // first global candidate index of this rank
    unsigned long long seed;
    int noise;          // noise_sigma != 0
    double loss_scale;    // sharded / peer / chunked loss: sum_n round(S_n 2^e) in int64, 2^e with
    double loss_unscale;  // e = min(40, 61 - ceil(log2(N_global K))) so the sum cannot overflow; 2^-e
};

// Pointers and sizes one iteration's kernels need (built by capi.cu).
struct StepArgs {
    float *theta, *m, *v;
    uint32_t *A0, *A1;
    int *hist, *unsat;
    float* gtab;                     // [KB][N] fp32 derivative table (R26)
    double* S;
    double* lossp;                   // [ceil(N/256)] k_gtable per-block sums of S_n
    long long* rowQ;
    double *rowD, *rowRho;
    unsigned char *rowGuard, *sol;
    int* hubD;                       // [n_hubs][KB-1][N] int32 signed bin counts
    DevScalars* ds;
    const uint32_t *cptr, *clit, *occ_ptr, *occ_rec, *occ_cnt;
    const uint32_t *upd_ptr, *upd_rec;  // records k_update stages: occ_* (uniform 3-SAT) or batched
    const int2* occ_pn;
    const int* hub_of;
    const int4* hub_sc;
    int n_hubs, n_hub_sc;
    int V, N;
    long long C;
    int KB;
    int uniform_len;                 // every clause has exactly K literals
    int num_sms;
    int upd_mode;                    // 0 (persistent k_update; kept for the ABI's geometry report)
    int upd_chunk;                   // candidates per k_update work item (== N: fused; < N: split sequence)
    int upd_gs_global;               // g table read from global memory (chunked)
    int upd_GT, upd_NG, upd_grid;    // v2 launch geometry
    int upd_rec_cap;                 // record words a group stages per row (max over non-hub rows)
    int upd_recbufs;                 // record buffers per group (1 or 2, configure_update)
    int upd_RB;                      // rows per work item: 1, or 32 / (N/32) for small shards (k_update_blk)
    int upd_blk_cap;                 // record words a group stages per row block (max over blocks, non-hub rows)
    int upd_cw6;                     // K <= 3 fused W = 1: 6-plane counters (no row above 31 same-sign occurrences)
    int upd_cl;                      // > 1: cluster-split rows (k_update MODE 3), CTAs per cluster
    int upd_prefetch;                // k_update: L2 bulk prefetch of each row's streams (configure_update)
    const int* blk_rows;             // [V] rows in block order (grouped by gather length; k_update_blk)
    // clause length segments (k_clause_seg; HostCnf::seg_*): use_seg = 1 when
    // the instance is not uniform 3-SAT, K <= 7 and N >= 1024 per GPU
    int use_seg;
    const uint32_t* seg_lit;
    long long seg_C[8], seg_off[8];
    // dense tensor-core clause evaluation (k_dense.cu; config.clause_eval = 1)
    int dense;
    const uint8_t* dP;               // [dCp][dKp] uint8 0/1 problem matrix (K-major)
    uint8_t* dAL;                    // [ceil(N/256)*256][dKp] uint8 0/1 assignment matrix (K-major)
    int dKp, dCp;
    // fp64 state (config.state_fp64 = 1, k_fp64.cu, reading R30): library-owned buffers
    int fp64;
    double *th64, *m64, *v64, *G64, *gt64;   // [V][N] x 4, [KB][N]
    long long* J64;                  // [V] int64 J partials (exact sums)
    unsigned long long* Qp64;        // [V][nb][2] 128-bit row-sum partials per 256-candidate block
    uint32_t *Pw64, *Nw64;           // [V][N/32] sign words of the next state
    int pdl;                         // launch k_clause / k_gtable / k_update with programmatic
                                     // stream serialisation (PDL; fused W = 1 path without hubs)
    size_t upd_smem;
    // candidate-sharded path (world > 1, or a 1-rank communicator)
    int sharded;
    float* Gbuf;                     // [V][N] fp32 G of the evaluated state
    long long* Jbuf;                 // [V] int64 partial / global J (fixed point)
    long long* Qbuf;                 // [V+1] int64 partial / global Q, slot V = loss (fixed point)
    uint32_t *Pbuf, *Nbuf;           // [V][N/32] sign planes of the next state
    unsigned long long* maxbuf;      // [3] (~best key, gmax bits, thmax bits)
    // peer-exchange path (W GPUs, exchanges over NVLink peer memory inside the kernels)
    int peer;
    PeerArgs px;
    MethodConsts mc;
};

// Workspace layout (byte offsets), see capi.cu: make_layout().
struct Layout {
    size_t theta, m, v, A0, A1, hist, gtab, S, lossp, unsat, rowQ, rowD, rowRho, rowGuard, scal, steptab, sol, hubD;
    size_t Gbuf, Jbuf, Qbuf, Pbuf, Nbuf, maxbuf, total;
};

// ---------------------------------------------------------------- launchers
// Launch with programmatic stream serialisation when pdl: the kernel may be
// scheduled while its predecessor in the stream drains, and waits for it with
// griddepcontrol.wait (pdl_wait) before touching any of its outputs.
template <typename... Exp, typename... Act>
inline cudaError_t launch_maybe_pdl(bool pdl, void (*k)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                    Act&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Act>(args)...);
}
cudaError_t launch_init(float* theta, float* m, float* v, int V, int N, long long n0, unsigned long long seed,
                        cudaStream_t st);
cudaError_t launch_rowstats(const float* theta, int V, int N, const MethodConsts& mc, long long* rowQ, double* rowD,
                            double* rowRho, unsigned char* rowGuard, uint32_t* A, unsigned int* thmax_bits,
                            cudaStream_t st);
// Step kernels, in order: 0 clause, 1 gtable, 2 hub, 3 update, 4 step_end.
constexpr int kKernelsPerStep = 5;
cudaError_t launch_step_kernel(int which, const StepArgs& a, const StepScalars* sc_dev, long long t, cudaStream_t st);
// Choose the k_update geometry for (N, KB) and set kernel attributes.
cudaError_t configure_kernels(StepArgs* a);
// sharded path (k_shard.cu); phases of one iteration between the collectives
cudaError_t launch_shard_pack_max(const StepArgs& a, const StepScalars* sc, cudaStream_t st);
cudaError_t launch_shard_unpack_max(const StepArgs& a, const StepScalars* sc, cudaStream_t st, bool key_only);
cudaError_t launch_update_a(const StepArgs& a, const uint32_t* Acur, const StepScalars* sc, cudaStream_t st);
cudaError_t launch_update_b(const StepArgs& a, const uint32_t* Acur, const StepScalars* sc, cudaStream_t st);
cudaError_t launch_rows_partial(const StepArgs& a, const float* theta, unsigned int* thmax_bits, cudaStream_t st);
cudaError_t launch_rows_finish(const StepArgs& a, uint32_t* Anext, cudaStream_t st);
// row-block k_update (k_update_blk.cu): rows per work item for a shard of N candidates
// (1: the per-row kernel), and the block kernel's geometry
int update_block_rows(int N);
cudaError_t configure_update_blk(StepArgs* a);
cudaError_t launch_update_blk(const StepArgs& a, const uint32_t* Acur, uint32_t* Anext, const StepScalars* sc,
                              cudaStream_t st);
// fp64 state (k_fp64.cu)
cudaError_t launch_init64(const StepArgs& a, unsigned long long seed, cudaStream_t st);
cudaError_t launch_rowstats64(const StepArgs& a, long long t, cudaStream_t st);
cudaError_t launch_update64(const StepArgs& a, const uint32_t* Acur, uint32_t* Anext, const StepScalars* sc,
                            cudaStream_t st);
cudaError_t launch_absG64(const StepArgs& a, const int* cols_dev, int M, double* absG, cudaStream_t st);
int fp64_blocks_per_row(int N);
// dense clause evaluation (k_dense.cu)
cudaError_t configure_dense();
cudaError_t launch_dense_clause(const StepArgs& a, const uint32_t* Acur, const StepScalars* sc, cudaStream_t st);
int dense_tile_m();
int dense_tile_n();
// whether the fused k_update geometry fits (else: chunked split sequence)
bool update_fits_fused(int KB, int N, int rec_cap, int optin);
// MODE 3 cluster size for a W = 1 batch of N candidates (0: not used), k_update.cu
int update_cluster_size(int KB, int N, int rec_cap, int optin);
// peer path: exchange of Qbuf[0..V) row partials (init / set_state), gen = exchange generation
cudaError_t launch_peer_rows_exchange(const StepArgs& a, unsigned gen, cudaStream_t st);
cudaError_t launch_step_end_sharded(const StepArgs& a, const StepScalars* sc, cudaStream_t st);
// NCCL (comm.cpp); return 0 or 7 (TSAT_E_NCCL) with err
int comm_unique_id(void* out128, std::string* err);
int comm_init(void** comm, const void* uid128, int rank, int world, std::string* err);
void comm_destroy(void* comm);
int comm_allreduce_max_u64(void* comm, unsigned long long* buf, size_t n, cudaStream_t st, std::string* err);
int comm_allreduce_sum_i64(void* comm, long long* buf, size_t n, cudaStream_t st, std::string* err);
int comm_allgather_u64(void* comm, const unsigned long long* send, unsigned long long* recv, size_t n, cudaStream_t st,
                       std::string* err);
int comm_async_error(void* comm, std::string* err);

cudaError_t launch_export(const StepArgs& a, long long t_eval, const int* cols_dev, int M, int k, double* absG,
                          unsigned long long* keys, int n64, int* out_v, double* out_g, cudaStream_t st, int phase);
// export entries of the selected owned columns: (|G| fp32 bits << 32) | (v << 1) | b_vn (evaluated state)
cudaError_t launch_export_pack(const StepArgs& a, long long t_eval, const int* cols_dev, const int* pos_dev, int Mo,
                               int k, const int* out_v, const double* out_g, unsigned long long* entries,
                               cudaStream_t st);
// peer path: all-gather of n u64 words per rank (phase 0 / 1 regions of PeerLayout E)
cudaError_t launch_peer_allgather(const StepArgs& a, int phase, const unsigned long long* send, int n,
                                  unsigned long long* recv, unsigned gen, cudaStream_t st);

}  // namespace tsat
