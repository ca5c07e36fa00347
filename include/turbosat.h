/*
 * turbosat.h - C-ABI of libturbosat, a B200-native (sm_100a) implementation of
 * TurboSAT's batched differentiable SAT step (arXiv 2511.07737).
 *
 * One iteration ("step") over a batch of N candidate assignments does, in the
 * paper's order (Fig. 3, §3.2, §4.1):
 *   Eq. 5 per-variable normalisation -> Eq. 2 binarisation B = clip(sign,0,1)
 *   -> Eq. 1 R = P A (clause evaluation) -> §3.1.4 per-candidate unsat count
 *   -> Eq. 4 SmoothMin, Eq. 3 loss -> straight-through backward (P^T, l.226)
 *   -> Eq. 5 Jacobian -> AdamW with step decay / restarts (l.255-259)
 *   -> re-binarisation; best-candidate selection (§4.2 l.279-287).
 * Export (§4.2 l.279-281) hands the k most confident variables of the best
 * candidates to a CPU CDCL solver (outside this library).
 *
 * Conventions
 *  - Every call returns tsat_status; nothing throws or exits across the ABI.
 *  - A CUDA/NCCL failure poisons the context: every later call on it returns
 *    the same code.  tsat_error_string() describes the last error.
 *  - Variables are 1-based in DIMACS text and in exported literals, 0-based in
 *    arrays indexed by variable.  Candidate indices are global and 0-based.
 *  - Device work is enqueued on the caller's CUDA stream (tsat_create).  Calls
 *    that return host data synchronise that stream.
 *  - Host pointers are plain host memory owned by the caller.  The batch
 *    workspace is device memory owned by the caller (size from
 *    tsat_workspace_bytes), alive until tsat_destroy or the next
 *    tsat_init_batch.  The parsed CNF (host and device copies) is owned by the
 *    library.
 *  - Numerics are canonical: integer /
 *    fixed-point cross-candidate sums and fixed-order IEEE ops, so results are
 *    bit-identical for any launch configuration and GPU count.
 */
#ifndef TURBOSAT_H
#define TURBOSAT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSAT_ABI_VERSION 2    /* 2: explicit element counts on host-array calls; global export */

typedef struct tsat_ctx_s* tsat_ctx;

typedef enum {
    TSAT_OK = 0,
    TSAT_E_ARG = 1,          /* invalid argument (null pointer, bad size, N % 32 != 0, k < 1, ...) */
    TSAT_E_PARSE = 2,        /* malformed DIMACS (SPEC S:45 error list) */
    TSAT_E_RANGE = 3,        /* instance/batch outside the supported range (e.g. clause length > 15) */
    TSAT_E_STATE = 4,        /* call out of order (step before init, export before any step, ...) */
    TSAT_E_OOM = 5,          /* host or device allocation failed / workspace too small */
    TSAT_E_CUDA = 6,         /* CUDA error (context poisoned) */
    TSAT_E_NCCL = 7,         /* NCCL error (context poisoned) */
    TSAT_E_UNSUPPORTED = 8   /* feature not built in this library */
} tsat_status;

/* Optimiser / method configuration.  Defaults (tsat_config_default) are the
 * paper's: AdamW lr 1e-1 -> 1e-15, /10 every 30 its, restart every 360
 * (PAPER.md l.255-259); AdamW beta/eps/weight decay = PyTorch defaults
 * (reading R6); tau = 1 (R1); Eq. 5 normalisation on, over all N (R20). */
typedef struct {
    double  tau;             /* SmoothMin temperature, Eq. 4 (> 0) */
    int32_t normalize;       /* 1 = Eq. 5 over all N candidates; 0 = off; 2 = per shard: each GPU averages
                                over its own N/W candidates and keeps J local; 3 = Eq. 5 with the row's
                                mean MAGNITUDE mean_n |theta_vn| as denominator (reading R28; its
                                Jacobian term carries sign(theta_vn))  (variants) */
    double  beta1, beta2;    /* AdamW moments (0.9, 0.999) */
    double  eps;             /* AdamW eps (1e-8) */
    double  weight_decay;    /* AdamW decoupled weight decay (1e-2) */
    double  lr0;             /* initial learning rate (1e-1) */
    double  lr_min;          /* learning-rate floor (1e-15) */
    double  decay_factor;    /* lr divisor per decay period (10) */
    int32_t decay_every;     /* iterations per decay period (30) */
    int32_t restart_every;   /* iterations per LR restart (360) */
    double  noise_sigma;     /* optional Philox noise in the update (0 = paper-exact, R17) */
    double  eps_norm;        /* Eq. 5 guard: |mean| <= eps_norm -> divide by +-eps_norm (1e-8) */
    int32_t reset_moments_on_restart;  /* 1 = re-create AdamW at each LR restart (t > 0, t % restart_every
                                          == 0): m = v = 0 and the bias-correction step restarts at 1
                                          (variant; 0 = paper default, R8) */
    double  tau_final;       /* SmoothMin temperature annealing (variant f2, reading R29): > 0 -> within each LR
                                cycle tau_t = tau * (tau_final / tau)^((t mod restart_every) / (restart_every - 1)),
                                geometric from tau to tau_final; 0 = constant tau (paper default, R1) */
    int32_t clause_eval;     /* rows a4/a5 (R = P A, histogram): 0 = bit-sliced sparse gathers (default);
                                1 = dense tensor-core tiles (tcgen05 uint8 MMA over the C x 2V matrix P and
                                the 2V x N assignment matrix, SURVEY 8(f) f4 experiment; library-owned
                                buffers of ceil(C/128)*128 x 2V and ceil(N/256)*256 x 2V bytes, TSAT_E_RANGE
                                above 2^31 bytes each) */
    int32_t state_fp64;      /* 1 = theta, m, v in fp64 and every fp32 rounding of the step in fp64 (variant
                                f2, SPEC's choice; reading R30): library-owned state of 48 B per
                                (variable, candidate); one GPU only (TSAT_E_UNSUPPORTED with world > 1); the
                                state is read / written with tsat_get_state64 / tsat_set_state64 */
} tsat_config;

typedef struct {
    int32_t V;               /* variables */
    int64_t C;               /* clauses (as stored; empty clauses included) */
    int64_t nnz;             /* literal occurrences after de-duplication */
    int32_t K;               /* longest clause */
    int64_t header_C;        /* clause count declared by the DIMACS header (-1 for tsat_load_clauses) */
    int64_t n_warnings;      /* header/body clause-count mismatch, missing final 0, ... */
    int64_t n_tautologies;   /* clauses containing x and ~x (kept) */
    int64_t n_duplicates;    /* duplicate literals removed */
    int32_t has_empty;       /* an empty clause is present: the instance is UNSAT */
    int32_t n_hub_rows;      /* variables whose occurrences are counted by the hub pre-pass */
} tsat_cnf_info;

typedef struct {
    int64_t t;               /* iterations completed (state is theta_t) */
    int32_t best_unsat;      /* min over candidates of unsat count at the last evaluated state theta_{t-1} */
    int64_t best_idx;        /* its global candidate index (ties -> lower index) */
    int32_t solved;          /* some candidate reached 0 unsat at some evaluated state */
    int64_t solved_step;     /* iteration at which the first model was found (-1 if none) */
    int64_t solved_idx;      /* candidate index of that model (-1 if none) */
    double  loss;            /* Eq. 3 loss -sum_n S_n at the last evaluated state */
} tsat_step_info;

typedef struct {
    int64_t  candidate;      /* out: global candidate index */
    int32_t  unsat;          /* out: its unsat count at the last evaluated state */
    int32_t  k;              /* out: number of literals written */
    int32_t* lits;           /* caller-allocated [k_req]: signed 1-based DIMACS literals, most confident first */
    float*   abs_grad;       /* caller-allocated [k_req] or NULL: |G_vn| (pre-Jacobian, R14), ascending */
} tsat_partial;

/* Fill *out with the paper defaults above. */
tsat_status tsat_config_default(tsat_config* out);

/* Host-only DIMACS validation (no context, no GPU): parses text[0..len) with
 * the same rules as tsat_load_dimacs and fills *info.  SPEC S:41-49. */
tsat_status tsat_parse_dimacs(const char* text, size_t len, tsat_cnf_info* info);

/* Human-readable name of a status code (static string). */
const char* tsat_status_string(tsat_status s);

/* Create a context on CUDA device `cuda_device`, enqueueing on `cuda_stream`
 * (a cudaStream_t; NULL = legacy default stream).
 * Multi-GPU (candidate sharding): every rank calls
 * tsat_create concurrently with the same `nccl_unique_id` (128 bytes from
 * tsat_nccl_unique_id on one rank, broadcast by the caller), its `rank` and
 * `world`; rank r then holds candidates [r N/W, (r+1) N/W).  Per iteration
 * the ranks exchange, over NCCL on the caller's stream, only exact integer
 * quantities (Eq. 5 row sums and Jacobian sums, the best candidate and two
 * maxima), so results are bit-identical for every world size.
 * nccl_unique_id == NULL requires world == 1 (single-GPU fused path); a
 * non-NULL id with world == 1 runs the sharded kernels on a 1-rank
 * communicator.  Errors: TSAT_E_ARG, TSAT_E_NCCL (libnccl.so.2 missing or
 * communicator init failed), TSAT_E_CUDA. */
tsat_status tsat_create(tsat_ctx* out, int cuda_device, void* cuda_stream,
                        const void* nccl_unique_id, int rank, int world);

/* Write a fresh NCCL unique id (NCCL_UNIQUE_ID_BYTES = 128) to out[0..bytes).
 * Host only; opens libnccl.so.2 at run time.  TSAT_E_NCCL if unavailable. */
/* Peer-exchange multi-GPU path: one process (or context) per
 * GPU of one NVLink/NVSwitch node, world <= 8.  The per-iteration exchanges
 * (per-row J and Q partials, the best key / maxima / loss) run inside the
 * step kernels as system-scope stores into every rank's exchange buffer,
 * mapped by CUDA IPC: no NCCL call and no extra kernel on the step path.
 * Sequence on every rank: tsat_create_peer -> tsat_load_* (allocates the
 * exchange buffer, sized by V) -> tsat_peer_handle -> all-gather the handles
 * (any host transport, e.g. torch.distributed) -> tsat_peer_open(all W handles
 * in rank order) -> tsat_init_batch / tsat_step as usual.  Every rank must make
 * the same sequence of init / set_state / step calls (they are collective).
 * world = 1 runs the same kernels exchanging with itself.  A peer that stops
 * responding makes the waiting kernels give up after 20 s: the step returns
 * TSAT_E_NCCL and the context is poisoned. */
#define TSAT_PEER_HANDLE_BYTES 64
tsat_status tsat_create_peer(tsat_ctx* out, int cuda_device, void* cuda_stream, int rank, int world);
/* This rank's exchange-buffer handle (TSAT_PEER_HANDLE_BYTES bytes into out). */
tsat_status tsat_peer_handle(tsat_ctx ctx, void* out, size_t bytes);
/* Map every rank's buffer: handles = world * TSAT_PEER_HANDLE_BYTES bytes, rank order. */
tsat_status tsat_peer_open(tsat_ctx ctx, const void* handles, size_t bytes);

tsat_status tsat_nccl_unique_id(void* out, size_t bytes);

/* Load a CNF from DIMACS text: comments 'c', header
 * 'p cnf V C', clauses as signed integers terminated by 0.  Duplicate
 * literals are removed, tautologies kept, empty clauses preserved.
 * Errors: malformed header, '-0', variable > V, non-integer token
 * -> TSAT_E_PARSE; clause length > 15 -> TSAT_E_RANGE.  Replaces any
 * previously loaded CNF and invalidates the batch. */
tsat_status tsat_load_dimacs(tsat_ctx ctx, const char* text, size_t len, tsat_cnf_info* info);

/* Load a CNF from arrays: clause c is dimacs_lits[clause_ptr[c] .. clause_ptr[c+1])
 * (signed 1-based literals, no terminators); clause_ptr has C+1 entries. */
tsat_status tsat_load_clauses(tsat_ctx ctx, int32_t V, int64_t C, const int64_t* clause_ptr,
                              const int32_t* dimacs_lits, tsat_cnf_info* info);

/* Device workspace bytes for a batch of N_global candidates (this rank holds
 * N_global / world of them).  N_global must be a multiple of 32 * world. */
tsat_status tsat_workspace_bytes(tsat_ctx ctx, int64_t N_global, size_t* bytes);

/* (a1) Initialise the batch (§4.1 l.250-252): theta_vn ~ N(0,1) from
 * Philox4x32-10 keyed by `seed` at counter (n>>2, v, 0, 0) over the GLOBAL
 * candidate index (shard-invariant), m = v = 0, t = 0.  `cfg` may be NULL
 * (defaults).  dev_workspace: caller-owned device memory of >= bytes. */
tsat_status tsat_init_batch(tsat_ctx ctx, int64_t N_global, uint64_t seed, const tsat_config* cfg,
                            void* dev_workspace, size_t bytes);

/* Run k >= 1 iterations (rows a2-a10).  The k-iteration sequence is captured
 * once as a CUDA graph and replayed; blocks only for the small *out readback
 * (out may be NULL, then it does not block). */
tsat_status tsat_step(tsat_ctx ctx, int32_t k, tsat_step_info* out);

/* Last step's info without stepping (blocks). */
tsat_status tsat_get_info(tsat_ctx ctx, tsat_step_info* out);

/* Per-candidate unsat counts of the last evaluated state for this rank's
 * N_local candidates (§3.1.4 l.169-177); *first_global_idx = index of
 * host_out[0].  n = elements of host_out, must equal N_local (TSAT_E_ARG). */
tsat_status tsat_query_unsat(tsat_ctx ctx, int32_t* host_out, size_t n, int64_t* first_global_idx);

/* Asynchronous variants (§3.1.4 l.169-177, same data).  tsat_query_unsat_async
 * enqueues the device->host copy of the N_local counts on the context's
 * stream and returns at once: host_out must be PINNED host memory
 * (cudaMallocHost / torch pin_memory) owned by the caller, and is valid only
 * after a later blocking call (tsat_sync, tsat_get_info, tsat_step with a
 * non-NULL out, or a synchronisation of the stream).  With tsat_step(ctx, k,
 * NULL) this lets a caller read every step's result while the next step
 * runs.  tsat_sync blocks until all work queued by this context is done. */
tsat_status tsat_query_unsat_async(tsat_ctx ctx, int32_t* host_out, size_t n, int64_t* first_global_idx);
tsat_status tsat_sync(tsat_ctx ctx);

/* (a10/a11) Export: the M best candidates by (unsat asc, index asc) over ALL
 * ranks, each with its k most confident variables = smallest
 * |G_vn| (ties -> lower v), paired with the candidate's value, all at the last
 * evaluated state (l.279-281; R14, R23).  k <= 0 selects the paper's rule
 * k = min(V, max(ceil(V/10^4), 20)).  host_out: M caller-owned entries whose
 * lits/abs_grad arrays hold at least k entries; 1 <= M <= N_global.
 * world > 1: a COLLECTIVE call (every rank calls it with the same M, k).  The
 * ranks all-gather their first M (unsat, index) keys (NCCL, or the peer
 * buffers), every rank merges them identically, each rank computes the
 * entries of the selected candidates it owns (only those candidates' bits
 * are read), and a second all-gather gives every rank the full list.
 * Multi-GPU limits: M <= 65536 and M * k <= 65536 (TSAT_E_RANGE). */
tsat_status tsat_export_best(tsat_ctx ctx, int32_t M, int32_t k, tsat_partial* host_out);

/* The number of literals tsat_export_best writes per candidate for a request
 * k_req (k_req <= 0: the paper's rule k = min(V, max(ceil(V/10^4), 20)),
 * l.279; else min(k_req, V)), so callers can size the lits / abs_grad arrays. */
tsat_status tsat_export_k(tsat_ctx ctx, int32_t k_req, int32_t* k_out);

/* Host-only selection step of the export (no context, no GPU): the M smallest
 * of n candidate keys (unsat << 32 | global index; unused slots ~0), ascending,
 * into out[0..M).  Keys hold the candidate index, so they are unique and the
 * order is the paper's (satisfied clauses desc, l.287; ties -> lower index).
 * tsat_export_best applies it to the all-gathered per-rank lists. */
tsat_status tsat_merge_keys(const uint64_t* keys, size_t n, int32_t M, uint64_t* out);

/* Binary values (0/1, V bytes) of candidate global_idx at the last evaluated state. */
tsat_status tsat_export_model(tsat_ctx ctx, int64_t global_idx, uint8_t* host_values);

/* The first model found (V bytes); TSAT_E_STATE if no candidate has reached 0
 * unsat.  world > 1: *idx and *step are global; the bits are written only on
 * the rank that owns candidate *idx (other ranks leave host_values untouched). */
tsat_status tsat_get_solution(tsat_ctx ctx, uint8_t* host_values, int64_t* idx, int64_t* step);

/* Checkpoint / resume: theta, m, v as [V][N_local] fp32 host arrays (any may be
 * NULL in get_state) and the iteration counter t. */
/* elems = elements of each non-NULL array; must equal V * N_local (TSAT_E_ARG
 * otherwise, e.g. a checkpoint of another world size or batch). */
tsat_status tsat_get_state(tsat_ctx ctx, float* theta, float* m, float* v, size_t elems, int64_t* t);
/* The same for a batch initialised with config.state_fp64 = 1 (fp64 arrays, V * N_local elements each);
 * the fp32 calls return TSAT_E_STATE on such a batch and these on an fp32 one. */
tsat_status tsat_get_state64(tsat_ctx ctx, double* theta, double* m, double* v, size_t elems, int64_t* t);
tsat_status tsat_set_state64(tsat_ctx ctx, const double* theta, const double* m, const double* v, size_t elems,
                             int64_t t);
tsat_status tsat_set_state(tsat_ctx ctx, const float* theta, const float* m, const float* v, size_t elems, int64_t t);

/* Rows rows[0..nrows) (0-based variables) of theta, m, v into host arrays of
 * [nrows][N_local] fp32 (any may be NULL): sampled checks at full size.
 * row_elems must equal N_local. */
tsat_status tsat_get_rows(tsat_ctx ctx, const int32_t* rows, int32_t nrows, float* theta, float* m, float* v,
                          size_t row_elems);

/* Copy an internal buffer to host (tests / diagnostics):
 *   which 0: histogram h [N_local][KB] int32 of the last evaluated state (KB = 4 if K <= 3 else 8)
 *         1: derivative table g [KB][N_local] fp32 (bin-major, R26);   2: S [N_local] fp64
 *         3: bits of the last evaluated state [V][N_local/32] uint32 (bit j of word w = candidate 32w+j)
 *         4: row statistics Q [V] int64 of the CURRENT state theta_t
 * bytes must equal the buffer size. */
tsat_status tsat_debug_copy(tsat_ctx ctx, int32_t which, void* host_dst, size_t bytes);

/* Kernel timing: when enabled, CUDA events bracket every kernel of every step
 * (also inside the graph).  tsat_kernel_times fills ms5 with the accumulated
 * milliseconds per segment [clause, gtable, hub, update, end] (sharded: the
 * segments also hold the collectives and small bookkeeping kernels) and
 * *steps with the number of steps timed, then resets the accumulators. */
tsat_status tsat_set_profiling(tsat_ctx ctx, int32_t enable);
tsat_status tsat_kernel_times(tsat_ctx ctx, double* ms5, int64_t* steps);

/* Number of CUDA kernels one iteration launches (for launch accounting; the
 * hub pre-pass only runs when the instance has hub variables). */
tsat_status tsat_kernels_per_step(tsat_ctx ctx, int32_t* n);

/* Launch geometry of the initialised batch (diagnostics, tests): out[0..7] =
 * {warp-group threads GT, warp groups per CTA, k_update grid (CTAs), k_update
 * dynamic shared memory (bytes), candidates per CTA slice or work item,
 * cluster size (> 1: rows split over a thread-block cluster),
 * rows per work item (> 1: row-block kernel), length-segmented clause
 * evaluation (1 / 0)}.  n_out must be >= 8.  TSAT_E_STATE before init. */
tsat_status tsat_update_geometry(tsat_ctx ctx, int32_t* out, int32_t n_out);

/* Learning rate of iteration t under cfg (readings R7/R9), host only
 * (for traces: iteration, lr, loss, best fraction, SPEC's --trace columns). */
tsat_status tsat_lr_at(const tsat_config* cfg, int64_t t, double* lr);

/* Last error message on ctx (static storage owned by ctx, valid until the next call). */
const char* tsat_error_string(tsat_ctx ctx);

/* Release the context and everything the library owns (not the caller's workspace). */
void tsat_destroy(tsat_ctx ctx);

/* ---------------------------------------------------------------- instances (host only)
 * Native generators of the benchmark instance families, deterministic per
 * seed (SplitMix64 stream; not bit-compatible with the Python tsat_synth
 * generators the parity tests use).  Arrays are caller-owned, clause_ptr has
 * C + 1 int64 offsets, literals are signed 1-based DIMACS, sigma is the
 * planted model (V bytes, 0/1).  TSAT_E_ARG on invalid sizes. */

/* Planted random k-SAT (k <= 15): k distinct variables per clause, the
 * clause's truth pattern under sigma uniform over the 2^k - 1 patterns that
 * satisfy it (hidden = 1) or over 1 .. 2^k - 2 so that the complement of sigma
 * satisfies it too (hidden = 2).  dimacs_lits holds C * k entries. */
tsat_status tsat_gen_planted(int32_t V, int64_t C, int32_t k, uint64_t seed, int32_t hidden,
                             int64_t* clause_ptr, int32_t* dimacs_lits, uint8_t* sigma);

/* Industrial-shaped CNF: clause lengths i.i.d. from len_probs[0..kmax]
 * (len_probs[0] must be 0; normalised), variables drawn with probability
 * proportional to rank^-alpha under a random id permutation, signs planted
 * (hidden = 1).  lits_capacity >= C * kmax. */
tsat_status tsat_gen_industrial(int32_t V, int64_t C, uint64_t seed, double alpha, int32_t kmax,
                                const double* len_probs, int64_t* clause_ptr, int32_t* dimacs_lits,
                                int64_t lits_capacity, uint8_t* sigma);

/* DIMACS text ("c planted ..." comment when sigma != NULL and V <= 64, the
 * header, one clause per line).  out == NULL: *length = bytes needed;
 * otherwise writes *length bytes (no terminator; TSAT_E_RANGE if capacity
 * is too small). */
tsat_status tsat_write_dimacs(int32_t V, int64_t C, const int64_t* clause_ptr, const int32_t* dimacs_lits,
                              const uint8_t* sigma, char* out, size_t capacity, size_t* length);

/* Number of clauses the 0/1 assignment model (V bytes) leaves unsatisfied
 * (0: model is a satisfying assignment; an empty clause is never satisfied). */
tsat_status tsat_verify_model(int32_t V, int64_t C, const int64_t* clause_ptr, const int32_t* dimacs_lits,
                              const uint8_t* model, int64_t* n_unsat);

/* ---------------------------------------------------------------- CPU hand-off
 * PAPER.md §4.2 l.277-287: once the best candidate satisfies > 99 % of the
 * clauses, the k most confident literals of each exported candidate
 * (tsat_export_best) initialise one CDCL instance per CPU thread; more
 * candidates than threads: the ones with more satisfied clauses first.
 * Host-only (no context, no GPU); the confident literals are assumed as the
 * first decisions, so a seed that excludes every model ends with status 21
 * (unsatisfiable under its assumptions) and the thread takes the next seed. */
typedef struct {
    int32_t status;          /* 10 = SAT (model written), 20 = UNSAT (the formula), 21 = UNSAT under the
                                assumptions (tsat_cdcl_solve), 0 = unknown (limit reached) */
    int32_t winner;          /* portfolio: index of the seed whose instance finished, -1 = the unseeded
                                instance, -2 = none */
    double  seconds;         /* wall time until the result (portfolio: since the call) */
    int64_t conflicts, decisions, propagations;   /* of the finishing instance */
    int32_t failed_seeds;    /* portfolio: seeded instances that were UNSAT under their assumptions */
    int32_t threads;         /* portfolio: threads used */
} tsat_cdcl_result;

/* One CDCL run on a CNF (clause_ptr[C+1] int64 offsets into dimacs_lits, signed
 * 1-based literals) under n_assumptions assumed literals.  conflict_limit <= 0:
 * none.  seed 0: deterministic default heuristics; otherwise randomised initial
 * activities and phases.  model_out (V bytes, 0/1, caller-owned, may be NULL)
 * is written on SAT.  TSAT_E_ARG on malformed arrays (non-monotone offsets,
 * literal 0 or |lit| > V); TSAT_E_OOM on allocation failure. */
tsat_status tsat_cdcl_solve(int32_t V, int64_t C, const int64_t* clause_ptr, const int32_t* dimacs_lits,
                            int32_t n_assumptions, const int32_t* assumptions, int64_t conflict_limit,
                            uint64_t seed, uint8_t* model_out, tsat_cdcl_result* out);

/* Portfolio of seeded CDCL instances on `threads` host threads: seeds is M x k
 * signed DIMACS literals (the lits arrays of tsat_export_best, best candidate
 * first; 0 entries are ignored), unseeded != 0 adds one instance without
 * assumptions (started first).  Stops at the first SAT (model_out, V bytes)
 * or UNSAT verdict, or after time_limit_s seconds (status 0). */
tsat_status tsat_cdcl_portfolio(int32_t V, int64_t C, const int64_t* clause_ptr, const int32_t* dimacs_lits,
                                int32_t M, int32_t k, const int32_t* seeds, int32_t threads, int32_t unseeded,
                                double time_limit_s, uint8_t* model_out, tsat_cdcl_result* out);

#ifdef __cplusplus
}
#endif
#endif /* TURBOSAT_H */
