/* mist_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for Mist's intra-stage tuning
 * sweep (arXiv 2503.19050, Sec. 5.3, Eq. 4-6, Alg. 1).  It shares no
 * code, header, table or helper with the CUDA product under
 * paper_2503_19050_b200/ and include/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, O-, L- and P-numbers = the
 * readings in SURVEY.md Sec. 8(c), restated in DESIGN.md.
 */
#ifndef MIST_ORACLE_H
#define MIST_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_SPLITS 8

typedef struct {
    int32_t L, h, a, k, f, V, s, e, g, p, fl, nrm;   /* O1, Table 4 / Fig. 8 symbols */
} orc_model_t;

typedef struct {
    orc_model_t model;
    int64_t B;                 /* global batch */
    int32_t N, M;              /* device mesh (N, M) */
    int64_t mem_budget;        /* Mem_Budget, bytes (Eq. 4) */
    int32_t Q;                 /* ratio grid k/Q (L19) */
    int32_t zero_mask;         /* allowed ZeRO levels, bit z */
    int32_t max_stages;        /* 0 => min(L, N*M) */
    int32_t n_grad_accum;      /* 0 => all divisors of B */
    const int32_t* grad_accum;
    /* profiled coefficients, tables [n_b][n_tp] row-major */
    int32_t n_b; const int32_t* b_values;
    int32_t n_tp; const int32_t* tp_values;
    const double *Tf, *Tb, *Tef, *Teb, *Thf, *Thb;
    double bw[4][2], lat[4][2];   /* [AR,AG,RS,P2P][intra,inter] */
    double bw_h2d, bw_d2h;
    double intf[16][4];           /* F[mask][channel], channels C,NCCL,H2D,D2H */
    /* search-space preset: 0 = the full space */
    int32_t ckpt_ends_only;       /* CKPT c in {0, l} only */
    int32_t offload_off;          /* bit 0 WO, 1 GO, 2 OO, 3 AO fixed at ratio 0 */
} orc_problem_t;

typedef struct {
    int32_t G, first, last, w, l, n, m, n_splits;
    int32_t tp[ORC_MAX_SPLITS], dp[ORC_MAX_SPLITS], b[ORC_MAX_SPLITS];
    uint64_t tuple_offset, config_offset, count;
} orc_group_t;

/* every intermediate of one configuration, for the worked-example pins */
typedef struct {
    /* O4 sizes */
    double P_layer, P_st, A_full, A_bnd, A_H, X;
    /* phase channel vectors [block][phase][channel]:
       block 0 = layer (not ckpt), 1 = layer (ckpt), 2 = embedding, 3 = head
       phase 0 = F, 1 = B, 2 = F', 3 = B' */
    double ch[4][4][4];
    double T[4][4];            /* PredINTF of each vector */
    double p2p;
    /* O9 memory, each term multiplied by D = Q*TP*DP (exact integers) */
    double D, Ms, Mwb, Mgb, Mob, Ma, Afull_D, mem_fwd_D, mem_bwd_D;
    double t, d, mem;
    int32_t feasible;
} orc_detail_t;

typedef struct {
    uint64_t idx; double t, y, mem; int64_t group;
} orc_point_t;

/* Alg. 1 PredINTF, literal. */
double orc_pred_intf(const double X[4], const double F[16][4]);
void orc_pred_intf_batch(const double* X, int64_t n, const double F[16][4], double* T);
double orc_intf_loss(const double* X, const double* Tobs, int64_t n, const double F[16][4]);
/* O5 collective time: kind 0=AR,1=AG,2=RS,3=P2P */
double orc_coll(const orc_problem_t* pb, int kind, double bytes, int gsz, int inter);

/* O2-O3 enumeration.  groups==NULL => size query. Returns 0 ok, <0 error. */
uint64_t orc_count_space(const orc_problem_t* pb, const orc_group_t* groups, int64_t n_groups);
int orc_enumerate(const orc_problem_t* pb, orc_group_t* groups, int64_t cap,
                  int64_t* n_groups, uint64_t* n_configs);

/* O4-O9 on one explicit configuration. */
int orc_eval_detail(const orc_problem_t* pb, const orc_group_t* grp, int split, int z,
                    int c, int kW, int kG, int kO, int kA, orc_detail_t* out);

/* O3 decode + O4-O9 for a list of global config indices. */
int orc_eval_indices(const orc_problem_t* pb, const orc_group_t* groups, int64_t n_groups,
                     const uint64_t* idx, int64_t n, double* t, double* d, double* mem,
                     uint8_t* feasible);
/* same for a contiguous range [begin, end) */
int orc_eval_range(const orc_problem_t* pb, const orc_group_t* groups, int64_t n_groups,
                   uint64_t begin, uint64_t end, double* t, double* d, double* mem,
                   uint8_t* feasible);

/* O10 frontier of an explicit point set (x = t, y, idx); method 0 auto,
   1 pairwise O(k^2) (the definition), 2 sort + scan. Output sorted by x. */
int64_t orc_frontier_points(const orc_point_t* pts, int64_t n, int method, orc_point_t* out);

/* Per-group sweep: evaluate every config of group g, keep feasible ones,
   return its frontier (ykey 0 = d, 1 = mem) and the feasible fingerprint
   (count, sum of splitmix64(idx) mod 2^64).  out==NULL => count only. */
int orc_group_frontier(const orc_problem_t* pb, const orc_group_t* groups, int64_t n_groups,
                       int64_t g, int ykey, int method, orc_point_t* out, int64_t cap,
                       int64_t* n_out, uint64_t* fp_count, uint64_t* fp_hash);

/* Whole sweep over groups [g_begin, g_end) (OpenMP over groups when
   threads > 1). out sized by caller (cap); group_offsets has g_end-g_begin+1. */
int orc_sweep(const orc_problem_t* pb, const orc_group_t* groups, int64_t n_groups,
              int64_t g_begin, int64_t g_end, int ykey, int threads,
              orc_point_t* out, int64_t cap, int64_t* n_out, int64_t* group_offsets,
              uint64_t* fp_count, uint64_t* fp_hash);

/* O11 alpha sampling over a frontier (points sorted by t within each group). */
int orc_sample(const orc_point_t* frontier, const int64_t* group_offsets, int64_t n_groups,
               const orc_group_t* groups, int32_t K, int64_t* picked, int64_t cap,
               int64_t* n_picked, int64_t* picked_offsets);

uint64_t orc_splitmix64(uint64_t x);

#ifdef __cplusplus
}
#endif
#endif
