/* mist.h -- C ABI of libmist, the B200 (sm_100a) implementation of the
 * intra-stage tuning sweep of Mist (arXiv 2503.19050).
 *
 * The sweep (Sec. 5.3, Eq. 4-6): for every candidate
 * stage context -- gradient-accumulation steps G, first/last stage flags,
 * in-flight microbatches w, layer count l and submesh (n, m) -- enumerate every
 * configuration (TP/DP split, ZeRO level z, checkpointed layers c, offload
 * ratios WO, GO, OO, AO), evaluate the overlap-aware stable time t and
 * first/last-microbatch delta d (Eq. 5-6, Alg. 1 interference model, lines
 * 563-605) and the peak memory max(Mem_fwd, Mem_bwd) (Eq. 4), drop configs over
 * Mem_Budget, and return per-group Pareto frontiers that the inter-stage MILP
 * samples (Eq. 3: IntraStagePareto(i, l_i, (n_i, m_i))[f_i]).
 *
 * Readings of the paper (O1-O12, L1-L34) are listed in DESIGN.md.
 *
 * Conventions (all functions):
 *  - Return mist_status_t; MIST_OK == 0.  mist_status_string() names it.
 *  - Callers own every buffer.  The library owns only what a mist_ctx_t
 *    allocates (device scratch, cached results, NCCL communicator), released
 *    by mist_ctx_destroy().
 *  - Structs and small inputs are host pointers.  Bulk outputs are documented
 *    per function as "device" (must be device memory, e.g. a torch CUDA
 *    tensor's data_ptr()) or "any" (host or device; copied with
 *    cudaMemcpyDefault).
 *  - Calls are synchronous: when a call returns, results are in caller memory.
 *  - One ctx per device per host thread.  A CUDA/NCCL failure returns
 *    MIST_ERR_CUDA/MIST_ERR_NCCL; the ctx stays destroyable.
 *  - There is no CPU fallback: without a CUDA device mist_ctx_create fails.
 */
#ifndef MIST_H
#define MIST_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MIST_MAX_SPLITS 8
#define MIST_NCCL_ID_BYTES 128

typedef enum {
    MIST_OK = 0,
    MIST_ERR_INVALID_ARG = 1,      /* bad shape/option, see each function   */
    MIST_ERR_EMPTY_SPACE = 2,      /* no group has a valid (DP, TP) split    */
    MIST_ERR_BUFFER_TOO_SMALL = 3, /* *n_out holds the needed size           */
    MIST_ERR_CUDA = 4,
    MIST_ERR_NCCL = 5,
    MIST_ERR_OOM = 6
} mist_status_t;

/* Model shape (Table 4; Fig. 8 symbols lines 517-531). */
typedef struct {
    int32_t num_layers;          /* L */
    int32_t hidden;              /* h */
    int32_t heads;               /* a */
    int32_t kv_heads;            /* k; kv dim = k*h/a must be an integer */
    int32_t ffn;                 /* f */
    int32_t vocab;               /* V */
    int32_t seq;                 /* s */
    int32_t elem_bytes;          /* e = 2 (FP16 mixed precision, line 489) */
    int32_t gated_mlp;           /* g in {0,1} */
    int32_t parallel_attn;       /* p in {0,1}: one TP all-reduce per layer (line 751) */
    int32_t flash_attn;          /* fl in {0,1}: no s^2 scores saved */
    int32_t norm_vecs_per_layer; /* nrm */
} mist_model_t;

/* Device mesh (N, M) and memory budget (line 625; Eq. 4). */
typedef struct {
    int32_t nodes;               /* N */
    int32_t gpus_per_node;       /* M */
    int64_t mem_budget_bytes;    /* Mem_Budget per GPU, bytes, 1 <= budget < 2^46 */
} mist_mesh_t;

/* Search-space options. */
typedef struct {
    int32_t offload_steps;       /* Q >= 1: ratios k/Q, k = 0..Q (Table 2 "Float [0,1]", L19) */
    int32_t zero_mask;           /* bit z set => ZeRO level z enumerated (default 0xF) */
    int32_t max_stages;          /* 0 => min(L, N*M) pipeline stages */
    int32_t n_grad_accum;        /* 0 => G over all divisors of B */
    const int32_t* grad_accum;   /* host, n_grad_accum entries */
    /* Search-space presets (fig:search-space P:364-370,
     * fig:eval-3-ablation P:810-822).  Zero = the full space.  A configuration
     * outside the preset keeps its index (O3) but is never feasible, never
     * fingerprinted and never on a frontier. */
    int32_t ckpt_ends_only;      /* 1 => CKPT c in {0, l} only (no / full recomputation, Megatron-style) */
    int32_t offload_off;         /* bit 0 WO, 1 GO, 2 OO, 3 AO: that ratio is fixed at 0 */
} mist_space_t;

/* Profiled coefficients: stand-in for the operator database (line 541) and
 * the communication model (bytes / bandwidth + latency).  Time tables are
 * row-major [n_b][n_tp], seconds, host pointers. */
typedef struct {
    int32_t n_b;  const int32_t* b_values;    /* microbatch sizes present in the tables */
    int32_t n_tp; const int32_t* tp_values;   /* TP sizes present in the tables */
    const double* t_layer_fwd;   /* Tf  per transformer layer */
    const double* t_layer_bwd;   /* Tb */
    const double* t_emb_fwd;     /* Tef embedding block (first stage) */
    const double* t_emb_bwd;     /* Teb */
    const double* t_head_fwd;    /* Thf LM-head block (last stage) */
    const double* t_head_bwd;    /* Thb */
    double bw[4][2];             /* [AR, AG, RS, P2P][intra, inter] bytes/s */
    double lat[4][2];            /* seconds */
    double bw_h2d, bw_d2h;       /* PCIe bytes/s (no latency, L23) */
    double intf[16][4];          /* Alg. 1 slowdown factors F[mask][channel] >= 1;
                                    channel bits C=1, NCCL=2, H2D=4, D2H=8 (L6);
                                    rows with < 2 bits are ignored */
} mist_coeffs_t;

/* One group = one IntraStagePareto key (G, first, last, w, l, n, m) (O2, L33). */
typedef struct {
    int32_t G, first, last, w, layers, n, m, n_splits;
    int32_t tp[MIST_MAX_SPLITS], dp[MIST_MAX_SPLITS], b[MIST_MAX_SPLITS];  /* ascending TP */
    uint64_t tuple_offset;       /* first global tuple id of the group */
    uint64_t config_offset;      /* first global config index of the group */
    uint64_t count;              /* n_splits * |zero levels| * (l+1) * (Q+1)^4 */
} mist_group_t;

/* One frontier point.  idx = global config index (O3):
 * idx = T*(Q+1)^4 + ((kW*(Q+1) + kG)*(Q+1) + kO)*(Q+1) + kA, T = global tuple id,
 * tuples ordered (group, split, z, c). */
typedef struct {
    uint64_t idx;
    double t;                    /* stable microbatch time, s (Eq. 5) */
    double y;                    /* d (Eq. 6) for MIST_Y_DELTA, mem for MIST_Y_MEM */
    double mem;                  /* max(Mem_fwd, Mem_bwd), bytes (Eq. 4) */
} mist_point_t;

typedef enum { MIST_Y_DELTA = 0, MIST_Y_MEM = 1 } mist_ykey_t;   /* ledger L1 */

typedef struct mist_ctx mist_ctx_t;

/* Per-call statistics of the last mist_pareto_frontier / mist_eval_* call. */
typedef struct {
    uint64_t configs_evaluated;  /* configs whose t, d, mem were computed */
    uint64_t candidates;         /* records emitted by the eval kernel (after prefilters) */
    uint64_t frontier_points;    /* local (pre-merge) frontier size */
    int64_t kernel_launches;     /* kernels launched by the call */
    double eval_ms;              /* sum of eval-kernel durations (CUDA events, ctx stream) */
    double precompute_ms;        /* tuple precompute kernels */
    double reduce_ms;            /* sort + scan + compaction kernels */
    double merge_ms;             /* NCCL all-gather + final frontier pass */
    double total_ms;             /* whole call, CUDA events on the ctx stream */
    int64_t chunks;              /* tuple chunks processed */
    int64_t reductions;          /* sort+scan passes run */
    uint64_t sort_keys;          /* keys pushed through the radix sort */
    int32_t sort_passes;         /* digit passes actually run (after skipping) */
    int32_t unit_factors;        /* 1 if the unit-factor (max) specialisation ran */
    uint64_t h2d_bytes;          /* host->device input bytes copied by the call */
    uint64_t d2h_bytes;          /* device->host result bytes copied by the call */
    double pilot_ms;             /* pilot sub-grid sweeps that seed the staircase filter */
    uint64_t pilot_configs;      /* configs evaluated by the pilot (extra work, not in configs_evaluated) */
    int64_t rollbacks;           /* optimistic chunks re-run after a candidate-buffer overflow */
    uint64_t phases_evaluated;   /* Alg. 1 phase rows (PredINTF calls) the main eval kernel ran */
    uint64_t bound_rows;         /* R5 lower-bound rows (DESIGN R5/R7) the main eval kernel ran */
} mist_stats_t;
/* total_ms spans the device work of the call from the moment its inputs are
 * resident in HBM to the last kernel (results still on the device). */

/* ---- context ------------------------------------------------------------ */
/* device: CUDA ordinal.  Fails with MIST_ERR_CUDA when no device is usable. */
mist_status_t mist_ctx_create(int device, mist_ctx_t** out);
void mist_ctx_destroy(mist_ctx_t* ctx);
const char* mist_status_string(mist_status_t st);
/* Text of the last error seen by this ctx (never NULL). */
const char* mist_ctx_last_error(const mist_ctx_t* ctx);
mist_status_t mist_ctx_stats(const mist_ctx_t* ctx, mist_stats_t* out);
/* Enable per-kernel CUDA-event timing (stats *_ms fields); default on. */
mist_status_t mist_ctx_set_timing(mist_ctx_t* ctx, int enabled);

/* Multi-GPU: rank 0 calls mist_nccl_unique_id, the id is
 * broadcast by the caller (e.g. torch.distributed), then every rank calls
 * mist_ctx_init_comm.  With a comm, mist_pareto_frontier all-gathers local
 * frontiers over NVLink (ncclAllGather) and returns the merged global
 * frontier on every rank. */
mist_status_t mist_nccl_unique_id(uint8_t id[MIST_NCCL_ID_BYTES]);
/* Host-only: the tuple ranges that `rank` of `world` evaluates when
 * mist_pareto_frontier is called with t_end == 0 and a communicator.
 * Block-cyclic (SURVEY 8(e) "weight ranges if the measured imbalance exceeds a
 * few percent"): [0, n_tuples) is cut into nb = world*K blocks at
 * floor(n_tuples*i/nb), K = clamp(n_tuples/(world*2048), 1, 512), and rank r
 * owns blocks i = r (mod world); adjacent owned blocks are coalesced.  Every
 * tuple holds (Q+1)^4 configs, so shares are equal in configs to within one
 * tuple per block, and the per-tuple cost, which varies by orders of
 * magnitude along the group order, is sampled evenly by every rank.
 * Two-call pattern: begins/ends == NULL (or cap too small) => *n_ranges is
 * set (MIST_ERR_BUFFER_TOO_SMALL when the buffers are too small).
 * INVALID_ARG if rank/world are out of range. */
mist_status_t mist_shard_ranges(uint64_t n_tuples, int rank, int world, uint64_t* begins,
                                uint64_t* ends, int64_t cap, int64_t* n_ranges);
mist_status_t mist_ctx_init_comm(mist_ctx_t* ctx, const uint8_t id[MIST_NCCL_ID_BYTES],
                                 int rank, int world);

/* ---- a1: enumerate_space (O2-O3) ---------------------
 * Host-only, integer.  groups == NULL => size query: writes *n_groups and
 * *n_configs.  Groups are in canonical order (lexicographic on
 * (G, first, last, w, l, n, m)).  Only groups realizable by a complete plan are
 * kept (L34).
 * Errors: INVALID_ARG (L, h, a, k < 1; a does not divide k*h; B < 1; Q < 1;
 * budget <= 0; zero_mask == 0; a needed (b, TP) missing from coeffs -- coeffs
 * may be NULL for a pure size query, then this check is skipped);
 * EMPTY_SPACE (no group has a valid split); BUFFER_TOO_SMALL
 * (groups_cap < *n_groups). */
mist_status_t mist_enumerate_space(const mist_model_t* model, int64_t global_batch,
                                   const mist_mesh_t* mesh, const mist_space_t* space,
                                   const mist_coeffs_t* coeffs_or_null,
                                   mist_group_t* groups, int64_t groups_cap,
                                   int64_t* n_groups, uint64_t* n_configs);

/* ---- a2-a7 dense evaluation (parity / debug path) ------------------------
 * Evaluates global config indices [begin, end) and writes, at position
 * idx - begin: t (s), d (s), mem (bytes) and feasible (1 iff mem <= budget).
 * Outputs: device pointers, any may be NULL.  groups/n_groups come from
 * mist_enumerate_space with the same inputs.
 * Errors: INVALID_ARG (end > total configs, begin > end, inconsistent groups). */
mist_status_t mist_eval_stage_costs(mist_ctx_t* ctx, const mist_model_t* model, int64_t B,
                                    const mist_mesh_t* mesh, const mist_space_t* space,
                                    const mist_coeffs_t* coeffs, const mist_group_t* groups,
                                    int64_t n_groups, uint64_t begin, uint64_t end, double* t,
                                    double* d, double* mem, uint8_t* feasible);

/* Test hook: same as above for an arbitrary list idx[0..n) (device pointer).
 * Every index is checked on the device: one >= the space's total config count
 * is never decoded, its outputs are left untouched, and the call returns
 * INVALID_ARG after the kernel (the other positions are written). */
mist_status_t mist_eval_stage_costs_at(mist_ctx_t* ctx, const mist_model_t* model, int64_t B,
                                       const mist_mesh_t* mesh, const mist_space_t* space,
                                       const mist_coeffs_t* coeffs, const mist_group_t* groups,
                                       int64_t n_groups, const uint64_t* idx, int64_t n,
                                       double* t, double* d, double* mem, uint8_t* feasible);

/* ---- a2-a11: the sweep ---------------------------------------------------
 * Evaluates the global tuple range [t_begin, t_end) (t_end == 0 => all
 * tuples; with a comm and t_end == 0, this rank's mist_shard_ranges share), keeps
 * feasible configs, and returns the exact per-group frontier over
 * (x, y) = (t, d) or (t, mem) (O10): point p beats q iff x_p <= x_q,
 * y_p <= y_q and (x_p < x_q or y_p < y_q or idx_p < idx_q); the frontier is
 * the set of feasible configs beaten by none.  Output is grouped by group in
 * canonical order, each group sorted by t ascending (y strictly descending);
 * group g occupies out[group_offsets[g] .. group_offsets[g+1]).  A group with no
 * feasible config has an empty range (not an error).
 * out: any memory, out_cap points; group_offsets: any memory, n_groups+1.
 * fp_count / fp_hash (any memory, n_groups each, may be NULL): feasible-set
 * fingerprint per group over the evaluated range: count and
 * sum of splitmix64(idx) mod 2^64 (merged across ranks with a comm).
 * If out_cap < needed: returns BUFFER_TOO_SMALL with *n_out = needed and
 * keeps the result cached in ctx; an immediate retry with the same
 * arguments and a larger buffer only copies. */
mist_status_t mist_pareto_frontier(mist_ctx_t* ctx, const mist_model_t* model, int64_t B,
                                   const mist_mesh_t* mesh, const mist_space_t* space,
                                   const mist_coeffs_t* coeffs, const mist_group_t* groups,
                                   int64_t n_groups, uint64_t t_begin, uint64_t t_end,
                                   mist_ykey_t ykey, mist_point_t* out, int64_t out_cap,
                                   int64_t* n_out, int64_t* group_offsets, uint64_t* fp_count,
                                   uint64_t* fp_hash);

/* ---- a9 + a10 on an explicit point set ------------------------------------
 * Exact per-group frontier (O10 on (x, y) = (t, y), idx tie-break) of the
 * points points[0..n), point i belonging to group groups[i] (0 <= g < n_groups).
 * This is the O12 merge step (frontier(A u B) = frontier(frontier(A) u
 * frontier(B))): e.g. frontiers gathered by other means can be merged here.
 * points, groups: any memory.  out: any memory, out_cap points, grouped and
 * t-sorted as in mist_pareto_frontier; group_offsets: any memory, n_groups+1.
 * Every t must be >= 0 and finite (t orders as its bit pattern).
 * Errors: INVALID_ARG (n < 0, n_groups < 1 or >= 2^24, group out of range,
 * negative or non-finite t); BUFFER_TOO_SMALL (*n_out = needed). */
mist_status_t mist_frontier_points(mist_ctx_t* ctx, const mist_point_t* points, const int32_t* groups,
                                   int64_t n, int64_t n_groups, mist_point_t* out, int64_t out_cap,
                                   int64_t* n_out, int64_t* group_offsets);

/* ---- a12: sample_frontier (O11) ----------------------------------
 * Host pointers.  For alpha_j = j/(K-1), j = 0..K-1, picks per group the
 * argmin over the group's frontier of alpha*G*t + (1-alpha)*y (ties: smaller
 * t, then smaller idx); distinct picks in order of first appearance.
 * picked: frontier positions (0-based into `frontier`), picked_cap entries;
 * picked_offsets: n_groups+1 entries.  Errors: INVALID_ARG if K < 2;
 * BUFFER_TOO_SMALL (with *n_picked = needed). */
mist_status_t mist_sample_frontier(const mist_point_t* frontier, const int64_t* group_offsets,
                                   int64_t n_groups, const mist_group_t* groups, int32_t K,
                                   int64_t* picked, int64_t picked_cap, int64_t* n_picked,
                                   int64_t* picked_offsets);

/* ---- a12 on the device -------------------------------
 * Same operation as mist_sample_frontier (O11: alpha_j = j/(K-1), argmin over the
 * group's frontier of alpha*G*t + (1-alpha)*y evaluated as ((alpha*G)*t) +
 * ((1-alpha)*y) without contraction, ties to the smaller t then the smaller idx,
 * distinct picks in order of first appearance), computed by one warp
 * per group on the ctx device.
 * frontier [n_points], group_offsets [n_groups+1] (group_offsets[0] = 0,
 * group_offsets[n_groups] = n_points, non-decreasing): host or device memory,
 * e.g. the outputs of mist_pareto_frontier with ykey = MIST_Y_DELTA.
 * groups: host, n_groups entries (for G).  Outputs, host or device memory:
 * picked[n_groups*K] = positions into `frontier` of group g's picks at
 * picked[g*K .. g*K + n_picked[g]), -1 after them; n_picked[n_groups].
 * INVALID_ARG for K < 2 or inconsistent offsets.  Synchronous. */
mist_status_t mist_sample_frontier_gpu(mist_ctx_t* ctx, const mist_point_t* frontier, int64_t n_points,
                                       const int64_t* group_offsets, int64_t n_groups,
                                       const mist_group_t* groups, int32_t K, int64_t* picked,
                                       int32_t* n_picked);
/* Sweep + a12 in one call, for an MILP-only consumer: the
 * (t, d) frontier is computed exactly as by mist_pareto_frontier(ykey =
 * MIST_Y_DELTA) and sampled on the device; only the samples leave the GPU.
 * out[n_groups*K]: group g's picks at out[g*K .. g*K + n_picked[g]) in pick
 * order, padded with {idx = UINT64_MAX, t = y = mem = 0}; n_picked[n_groups].
 * Host or device memory.  Multi-GPU as mist_pareto_frontier. */
mist_status_t mist_pareto_sample(mist_ctx_t* ctx, const mist_model_t* model, int64_t global_batch,
                                 const mist_mesh_t* mesh, const mist_space_t* space,
                                 const mist_coeffs_t* coeffs, const mist_group_t* groups,
                                 int64_t n_groups, uint64_t t_begin, uint64_t t_end, int32_t K,
                                 mist_point_t* out, int32_t* n_picked);

/* ---- inter-stage consumer (Eq. 2-3)
 * Host-only.  Chooses G, the number of stages S and, per stage i = 1..S, a group
 * (the IntraStagePareto key (G, [i=1], [i=S], min(G, S-i+1), l_i, n_i, m_i), O2) and
 * one of its candidate points, with sum l_i = num_layers and sum n_i*m_i =
 * n_devices, minimising Eq. 2:
 *     (G-1) max_i t_i + sum_i t_i + max_i (d_i - sum_{j<i} t_j)   (reading L4).
 * Exact over the given candidates (label-setting DP); the objective
 * is non-decreasing in every t_i and d_i, so passing each group's (t, d) frontier
 * (mist_pareto_frontier with MIST_Y_DELTA) gives the optimum over the whole
 * configuration space, and passing the alpha-samples (mist_sample_frontier /
 * mist_pareto_sample) gives the paper's sampled formulation (Eq. 3).
 * groups[n_groups]: the enumeration's group table; points + group_offsets
 * [n_groups+1]: group g's candidates at points[group_offsets[g] ..
 * group_offsets[g+1]), y = d.  All host memory.  n_threads <= 0: one per core
 * (the G values are independent).
 * plan: stage i's group index plan->group[i-1] and candidate position (into
 * points) plan->point[i-1]; objective and its three terms recomputed from
 * the chosen points in Eq. 2's order.  Ties: the first G (ascending), then the
 * fewest stages.
 * Errors: INVALID_ARG (null pointers, n_groups < 1, num_layers < 1, n_devices < 1,
 * non-monotone offsets, a key field out of range); EMPTY_SPACE (no complete plan
 * has a candidate at every stage); BUFFER_TOO_SMALL (S > MIST_MAX_STAGES). */
#define MIST_MAX_STAGES 128
typedef struct {
    int32_t G, S;
    double objective;            /* Eq. 2, s */
    double t_max, t_sum, d_term; /* max_i t_i, sum_i t_i, max_i (d_i - sum_{j<i} t_j) */
    int64_t labels;              /* DP labels kept, summed over G (diagnostic) */
    int32_t group[MIST_MAX_STAGES];
    int64_t point[MIST_MAX_STAGES];
} mist_plan_t;
mist_status_t mist_solve_inter(const mist_group_t* groups, int64_t n_groups, const mist_point_t* points,
                               const int64_t* group_offsets, int32_t num_layers, int32_t n_devices,
                               int32_t n_threads, mist_plan_t* plan);

/* ---- interference model over observation tables -----
 * Alg. 1 "Batched Interference Estimation" and the
 * fitting of its slowdown factors, which the paper describes only as
 * "data-driven ... the resulting runtime data is used to train the slowdown
 * factors" (line 561).  Readings F1-F3.
 * X: device memory, n rows of 4 doubles [C, NCCL, H2D, D2H] (the channel order
 * of mist_coeffs_t.intf; Alg. 1's G2G = NCCL, C2G = H2D, G2C = D2H, L6),
 * 32-byte aligned, every entry >= 0 and finite.  intf / init / out: the 16x4
 * pattern-indexed factor table of mist_coeffs_t.intf (rows with < 2 bits
 * ignored; member factors >= 1).
 * mist_pred_intf: T[n] (device) = PredINTF of every row.
 * mist_fit_intf: T_obs[n] (device, > 0) observed totals.  F1 loss = mean of
 * ((PredINTF(X_i) - T_obs_i) / T_obs_i)^2; F2 coordinate descent over the 28
 * member factors (pattern ascending, channel ascending), `iters` sweeps; F3 per
 * coordinate 3 nested grids of 31 points over [1, fmax], each centred on the
 * best value so far with half-width one previous step (lower end clamped at 1);
 * a value replaces the current one only when its loss is strictly lower, so
 * *loss never exceeds the loss of `init`.  out: fitted table (host), *loss:
 * its loss.  Each grid level is ONE pass over the observations that evaluates
 * all 32 candidates (one per lane).
 * Errors: INVALID_ARG (null pointers, n < 1 for the fit, a member factor < 1,
 * fmax <= 1, an invalid row or observation -- counted on the device, text in
 * mist_ctx_last_error); CUDA.  Synchronous. */
mist_status_t mist_pred_intf(mist_ctx_t* ctx, const double* X, int64_t n, const double intf[16][4], double* T);
mist_status_t mist_fit_intf(mist_ctx_t* ctx, const double* X, const double* T_obs, int64_t n,
                            const double init[16][4], int32_t iters, double fmax, double out[16][4],
                            double* loss);

/* ---- search-space size (fig:search-space) ----
 * Host-only.  *n_in_space = number of configurations of the space that the
 * preset fields of `space` admit: sum over groups of n_splits * |ZeRO levels|
 * * |CKPT choices| * prod over the four ratios of (1 if disabled else Q+1);
 * |CKPT choices| = l+1, or 2 with ckpt_ends_only (l >= 1, so 0 != l).  *n_configs = the full index space (as mist_enumerate_space).
 * Errors as mist_enumerate_space. */
mist_status_t mist_count_space(const mist_model_t* model, int64_t global_batch, const mist_mesh_t* mesh,
                               const mist_space_t* space, uint64_t* n_in_space, uint64_t* n_configs);

#ifdef __cplusplus
}
#endif
#endif /* MIST_H */
