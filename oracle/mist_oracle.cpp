/* mist_oracle.cpp -- TEST INFRASTRUCTURE ONLY (see mist_oracle.h).
 *
 * A plain CPU implementation of Mist's intra-stage tuning sweep written from
 * the paper, step by step, for checking the CUDA product.  Build flags:
 * -O2 -ffp-contract=off (no fast-math, no FMA contraction; ledger L32).
 *
 *   O2/O3  enumeration of groups, tuples and configs ......... orc_enumerate
 *   O4     sizes (params, weights, grads, optimizer, activations)
 *   O5     communication model ("dividing bytes by the bandwidth")
 *   O6     phase channel vectors of the overlap schedule
 *   O7     Alg. 1 PredINTF .......................... orc_pred_intf
 *   O8     stage time t and delta d (Eq. 5-6)
 *   O9     peak memory and feasibility (Eq. 4), exact rational
 *   O10    Pareto frontier (Eq. 3) ....................... orc_frontier_points
 *   O11    alpha sampling ............................... orc_sample
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions without a pin would say
 * "parity unpinned" here; every function below is pinned.
 */
#include "mist_oracle.h"

#include <algorithm>
#include <cmath>
#include <limits>
#include <set>
#include <tuple>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __int128 i128;

/* ------------------------------------------------------------------------ */
/* O7 -- Alg. 1 "Batched Interference Estimation", one row.      */
/* X = [C, G2G, C2G, G2C] = [C, NCCL, H2D, D2H] (ledger L6).          */
/* ------------------------------------------------------------------------ */

/* Update: ids = {j | (X_j != 0) matches mask}.  "matches" is read
 * as exact equality of the row's nonzero pattern with the mask (ledger L9). */
static void alg1_update(double X[4], double* T, int mask, const double factors[4]) {
    int pattern = 0;
    for (int j = 0; j < 4; ++j)
        if (X[j] != 0.0) pattern |= 1 << j;
    if (pattern != mask) return;                       /* ids = empty -> return */
    double scaled[4];
    double overlap = std::numeric_limits<double>::infinity();
    for (int j = 0; j < 4; ++j)
        if (mask >> j & 1) {
            scaled[j] = X[j] * factors[j];             /* scaled <- X[ids] x factors */
            overlap = std::min(overlap, scaled[j]);    /* overlap <- min(scaled) */
        }
    for (int j = 0; j < 4; ++j)
        if (mask >> j & 1) X[j] = (scaled[j] - overlap) / factors[j];
    *T += overlap;                                     /* T[ids] += overlap */
}

extern "C" double orc_pred_intf(const double Xin[4], const double F[16][4]) {
    double X[4] = {Xin[0], Xin[1], Xin[2], Xin[3]};
    double T = 0.0;
    for (int n = 4; n >= 2; --n) {                     /* n = 4 downto 2 */
        /* all C(4, n) combinations, lexicographic order */
        for (int a = 0; a < 4; ++a)
            for (int b = a + 1; b < 4; ++b) {
                if (n == 2) { int mask = (1 << a) | (1 << b); alg1_update(X, &T, mask, F[mask]); continue; }
                for (int c = b + 1; c < 4; ++c) {
                    if (n == 3) { int mask = (1 << a) | (1 << b) | (1 << c); alg1_update(X, &T, mask, F[mask]); continue; }
                    for (int d = c + 1; d < 4; ++d) {
                        int mask = (1 << a) | (1 << b) | (1 << c) | (1 << d);
                        alg1_update(X, &T, mask, F[mask]);
                    }
                }
            }
    }
    T += ((X[0] + X[1]) + X[2]) + X[3];                /* T += sum(X, axis=-1) */
    return T;
}

/* Alg. 1 over a batch of rows ("Batched Interference Estimation"):
 * X[n][4] row-major, T[n] out.  Row by row, the literal routine above. */
extern "C" void orc_pred_intf_batch(const double* X, int64_t n, const double F[16][4], double* T) {
    for (int64_t i = 0; i < n; ++i) T[i] = orc_pred_intf(X + 4 * i, F);
}

/* Fitting loss ("the resulting runtime data is used to
 * train the slowdown factors"; reading F1 in DESIGN.md 9): mean over the
 * observations of the squared relative error ((PredINTF(X_i) - T_i) / T_i)^2,
 * summed in row order. */
extern "C" double orc_intf_loss(const double* X, const double* Tobs, int64_t n, const double F[16][4]) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double r = (orc_pred_intf(X + 4 * i, F) - Tobs[i]) / Tobs[i];
        s += r * r;
    }
    return s / (double)n;
}

/* ------------------------------------------------------------------------ */
/* O5 -- communication model (ring coefficients S:152, ledger L23).   */
/* ------------------------------------------------------------------------ */
enum { AR = 0, AG = 1, RS = 2, P2P = 3 };

extern "C" double orc_coll(const orc_problem_t* pb, int kind, double bytes, int gsz, int inter) {
    if (kind == P2P) return bytes / pb->bw[P2P][inter] + pb->lat[P2P][inter];
    if (gsz == 1) return 0.0;
    double coef = (kind == AR) ? 2.0 * (gsz - 1) / gsz : (double)(gsz - 1) / gsz;
    return coef * bytes / pb->bw[kind][inter] + pb->lat[kind][inter];
}

static double h2d(const orc_problem_t* pb, double bytes) { return bytes / pb->bw_h2d; }
static double d2h(const orc_problem_t* pb, double bytes) { return bytes / pb->bw_d2h; }

/* ------------------------------------------------------------------------ */
/* O2/O3 -- enumeration                                                      */
/* ------------------------------------------------------------------------ */
static std::vector<int> grad_accum_list(const orc_problem_t* pb) {
    std::vector<int> out;
    if (pb->n_grad_accum > 0 && pb->grad_accum) {
        for (int i = 0; i < pb->n_grad_accum; ++i) out.push_back(pb->grad_accum[i]);
        std::sort(out.begin(), out.end());
        out.erase(std::unique(out.begin(), out.end()), out.end());
    } else {
        for (int64_t G = 1; G <= pb->B; ++G)
            if (pb->B % G == 0) out.push_back((int)G);     /* all divisors of B */
    }
    return out;
}

/* Alpa-style submeshes: {(1,m): m = 2^j <= M, m | M} u {(n,M): 2 <= n <= N} */
static std::vector<std::pair<int, int>> submeshes(const orc_problem_t* pb) {
    std::vector<std::pair<int, int>> out;
    for (int m = 1; m <= pb->M; m *= 2)
        if (pb->M % m == 0) out.push_back({1, m});
    for (int n = 2; n <= pb->N; ++n) out.push_back({n, pb->M});
    return out;
}

static int num_zero_levels(const orc_problem_t* pb) {
    int nz = 0;
    for (int z = 0; z < 4; ++z) nz += (pb->zero_mask >> z) & 1;
    return nz;
}

static int zero_level(const orc_problem_t* pb, int zi) {
    for (int z = 0; z < 4; ++z)
        if ((pb->zero_mask >> z) & 1) { if (zi == 0) return z; --zi; }
    return -1;
}

static int table_index(const orc_problem_t* pb, int b, int tp) {
    int ib = -1, it = -1;
    for (int i = 0; i < pb->n_b; ++i) if (pb->b_values[i] == b) ib = i;
    for (int i = 0; i < pb->n_tp; ++i) if (pb->tp_values[i] == tp) it = i;
    if (ib < 0 || it < 0) return -1;
    return ib * pb->n_tp + it;
}

extern "C" int orc_enumerate(const orc_problem_t* pb, orc_group_t* groups, int64_t cap,
                             int64_t* n_groups, uint64_t* n_configs) {
    const orc_model_t& md = pb->model;
    if (pb->B < 1 || pb->Q < 1 || pb->N < 1 || pb->M < 1 || md.L < 1 || md.a < 1 ||
        md.k < 1 || (md.k * (int64_t)md.h) % md.a != 0 || pb->mem_budget <= 0 ||
        (pb->zero_mask & 0xF) == 0)
        return -1;
    const int devices = pb->N * pb->M;
    int Smax = std::min(md.L, devices);
    if (pb->max_stages > 0) Smax = std::min(Smax, pb->max_stages);
    auto meshes = submeshes(pb);
    std::vector<int> sizes;
    for (auto& nm : meshes) sizes.push_back(nm.first * nm.second);
    /* can[k][r]: r devices split into exactly k submesh sizes (subset-sum DP, L34) */
    std::vector<std::vector<char>> can(Smax + 1, std::vector<char>(devices + 1, 0));
    can[0][0] = 1;
    for (int k = 1; k <= Smax; ++k)
        for (int r = 0; r <= devices; ++r)
            for (int sz : sizes)
                if (sz <= r && can[k - 1][r - sz]) { can[k][r] = 1; break; }

    /* O2 keys (G, first, last, w, l, n, m), deduplicated, lexicographic order */
    std::set<std::tuple<int, int, int, int, int, int, int>> keys;
    for (int G : grad_accum_list(pb))
        for (int S = 1; S <= Smax; ++S)
            for (int i = 1; i <= S; ++i) {
                int first = (i == 1), last = (i == S), w = std::min(G, S - i + 1);
                for (int l = 1; l <= md.L - S + 1; ++l)
                    for (auto& nm : meshes) {
                        int rest = devices - nm.first * nm.second;
                        if (rest < 0) continue;
                        if (S == 1 && (l != md.L || rest != 0)) continue;
                        if (!can[S - 1][rest]) continue;
                        keys.insert(std::make_tuple(G, first, last, w, l, nm.first, nm.second));
                    }
            }

    const int nz = num_zero_levels(pb);
    const uint64_t R = (uint64_t)(pb->Q + 1) * (pb->Q + 1) * (pb->Q + 1) * (pb->Q + 1);
    int64_t ng = 0;
    uint64_t tuples = 0, configs = 0;
    for (auto& key : keys) {
        orc_group_t gr = {};
        std::tie(gr.G, gr.first, gr.last, gr.w, gr.l, gr.n, gr.m) = key;
        /* O3 splits, ascending TP: TP = 2^j <= m, TP | n*m, TP | a, TP | k;
           DP = n*m/TP; valid iff G*DP | B; b = B/(G*DP) (L18) */
        for (int tp = 1; tp <= gr.m; tp *= 2) {
            if ((gr.n * gr.m) % tp || md.a % tp || md.k % tp) continue;
            int dp = gr.n * gr.m / tp;
            if (pb->B % ((int64_t)gr.G * dp)) continue;
            int b = (int)(pb->B / ((int64_t)gr.G * dp));
            if (table_index(pb, b, tp) < 0) return -2;     /* coefficient table lacks (b, TP) */
            if (gr.n_splits >= ORC_MAX_SPLITS) return -3;
            gr.tp[gr.n_splits] = tp; gr.dp[gr.n_splits] = dp; gr.b[gr.n_splits] = b;
            gr.n_splits++;
        }
        if (gr.n_splits == 0) continue;                    /* keys with zero splits dropped */
        uint64_t nt = (uint64_t)gr.n_splits * nz * (gr.l + 1);
        gr.tuple_offset = tuples;
        gr.config_offset = configs;
        gr.count = nt * R;                                 /* n_splits * |z| * (l+1) * (Q+1)^4 */
        if (groups) {
            if (ng >= cap) return -4;
            groups[ng] = gr;
        }
        ng++;
        tuples += nt;
        configs += gr.count;
    }
    *n_groups = ng;
    *n_configs = configs;
    return ng == 0 ? -5 : 0;
}

/* ------------------------------------------------------------------------ */
/* O4-O9 -- one configuration                                                */
/* ------------------------------------------------------------------------ */
struct Block {              /* one repeated block of the stage (layer, embedding or head) */
    double W, Gr, O;        /* bytes per GPU of weights, grads, optimizer states (O4) */
    double A[2];            /* saved activation bytes, A_r for r = 0 (full) / 1 (ckpt boundary) */
    double Tf, Tb;          /* profiled fwd / bwd compute */
    int nf, nb;             /* TP all-reduces per direction (O5) */
};

/* O6 phase channels [C, NCCL, H2D, D2H] for one block. */
static void phase_vectors(const orc_problem_t* pb, const Block& blk, int r, int z, int TP, int DP,
                          int dp_inter, double X, double WO, double GO, double OO, double AO,
                          double out[4][4]) {
    const double sw = (z == 3) ? 1.0 / DP : 1.0;   /* sigma_w */
    const double sg = (z >= 2) ? 1.0 / DP : 1.0;   /* sigma_g */
    const double so = (z >= 1) ? 1.0 / DP : 1.0;   /* sigma_o */
    const double ARtp_f = blk.nf * orc_coll(pb, AR, X, TP, 0);
    const double ARtp_b = blk.nb * orc_coll(pb, AR, X, TP, 0);
    const double AGw = orc_coll(pb, AG, blk.W, DP, dp_inter);
    const double RSg = orc_coll(pb, RS, blk.Gr, DP, dp_inter);
    const double ARg = orc_coll(pb, AR, blk.Gr, DP, dp_inter);
    const double Ar = blk.A[r];
    double* F = out[0]; double* B = out[1]; double* Fp = out[2]; double* Bp = out[3];
    /* F: stable forward */
    F[0] = blk.Tf + ARtp_f;
    F[1] = (z == 3) ? AGw : 0.0;
    F[2] = h2d(pb, WO * sw * blk.W);
    F[3] = d2h(pb, AO * Ar);
    /* B: stable backward; a checkpointed layer recomputes its forward (L17) */
    B[0] = blk.Tb + ARtp_b + r * (blk.Tf + ARtp_f);
    B[1] = ((z == 3) ? AGw : 0.0) + ((z >= 2) ? RSg : 0.0);
    B[2] = h2d(pb, WO * sw * blk.W + GO * sg * blk.Gr + AO * Ar);
    B[3] = d2h(pb, GO * sg * blk.Gr);
    /* F': first-microbatch forward with the repositioned optimizer step */
    Fp[0] = F[0];
    Fp[1] = F[1] + ((z == 1 || z == 2) ? AGw : 0.0);
    Fp[2] = F[2] + h2d(pb, OO * so * blk.O + GO * sg * blk.Gr);
    Fp[3] = F[3] + d2h(pb, OO * so * blk.O + WO * sw * blk.W);
    /* B': last-microbatch backward, gradient synchronisation */
    Bp[0] = B[0];
    Bp[1] = B[1] + ((z == 0) ? ARg : 0.0) + ((z == 1) ? RSg : 0.0);
    Bp[2] = B[2];
    Bp[3] = B[3];
}

struct CfgId {
    const orc_group_t* g;
    int split, z, c, kW, kG, kO, kA;
};

/* Search-space presets (fig:search-space P:364-370,
 * fig:eval-3-ablation P:810-822): a configuration is in the preset unless it
 * checkpoints a strict subset of the layers under ckpt_ends_only, or uses a
 * nonzero ratio of a disabled offload type. */
static bool in_preset(const orc_problem_t* pb, const CfgId& cf) {
    if (pb->ckpt_ends_only && cf.c != 0 && cf.c != cf.g->l) return false;
    const int k[4] = {cf.kW, cf.kG, cf.kO, cf.kA};
    for (int r = 0; r < 4; ++r)
        if ((pb->offload_off >> r & 1) && k[r] != 0) return false;
    return true;
}

static int eval_config(const orc_problem_t* pb, const CfgId& cf, orc_detail_t* o) {
    const orc_model_t& md = pb->model;
    const orc_group_t& gr = *cf.g;
    const int TP = gr.tp[cf.split], DP = gr.dp[cf.split], b = gr.b[cf.split];
    const int z = cf.z, c = cf.c, l = gr.l, Q = pb->Q;
    const int ti = table_index(pb, b, TP);
    if (ti < 0 || c < 0 || c > l || z < 0 || z > 3) return -1;
    /* L19: ratios k/Q by IEEE division */
    const double WO = (double)cf.kW / Q, GO = (double)cf.kG / Q, OO = (double)cf.kO / Q,
                 AO = (double)cf.kA / Q;
    const double e = md.e, s = md.s, h = md.h, a = md.a, f = md.f, V = md.V;
    const double bb = b;

    /* ---- O4 sizes ---- */
    const double kvd = (double)(md.k * (int64_t)md.h / md.a);
    const double P_layer = 2 * h * h + 2 * h * kvd + (2 + md.g) * h * f + md.nrm * h;
    const double P_E = V * h, P_H = V * h;                       /* untied (L21, L30) */
    const double X = e * s * bb * h;
    const double A_full = e * s * bb * (4 * h + (2 * h + 2 * kvd + (2 + 2 * md.g) * f +
                                                 (1 - md.fl) * a * s) / TP);
    const double A_bnd = e * s * bb * h;
    const double A_H = e * s * bb * h + 4 * s * bb * V / TP;
    o->P_layer = P_layer;
    o->P_st = l * P_layer / TP + gr.first * P_E / TP + gr.last * P_H / TP;
    o->A_full = A_full; o->A_bnd = A_bnd; o->A_H = A_H; o->X = X;

    Block layer = {e * P_layer / TP, e * P_layer / TP, 12 * P_layer / TP, {A_full, A_bnd},
                   pb->Tf[ti], pb->Tb[ti], 2 - md.p, 2 - md.p};
    Block emb = {e * P_E / TP, e * P_E / TP, 12 * P_E / TP, {0.0, 0.0},
                 pb->Tef[ti], pb->Teb[ti], 1, 0};
    Block head = {e * P_H / TP, e * P_H / TP, 12 * P_H / TP, {A_H, A_H},
                  pb->Thf[ti], pb->Thb[ti], 0, 1};
    const int dp_inter = gr.n > 1;                              /* DP group spans nodes iff n > 1 */

    /* ---- O6 + O7 ---- */
    for (int blk = 0; blk < 4; ++blk)
        for (int ph = 0; ph < 4; ++ph) {
            for (int j = 0; j < 4; ++j) o->ch[blk][ph][j] = 0.0;
            o->T[blk][ph] = 0.0;
        }
    phase_vectors(pb, layer, 0, z, TP, DP, dp_inter, X, WO, GO, OO, AO, o->ch[0]);
    phase_vectors(pb, layer, 1, z, TP, DP, dp_inter, X, WO, GO, OO, AO, o->ch[1]);
    if (gr.first) phase_vectors(pb, emb, 0, z, TP, DP, dp_inter, X, WO, GO, OO, AO, o->ch[2]);
    if (gr.last) phase_vectors(pb, head, 0, z, TP, DP, dp_inter, X, WO, GO, OO, AO, o->ch[3]);
    for (int blk = 0; blk < 4; ++blk) {
        if (blk == 2 && !gr.first) continue;
        if (blk == 3 && !gr.last) continue;
        for (int ph = 0; ph < 4; ++ph) o->T[blk][ph] = orc_pred_intf(o->ch[blk][ph], pb->intf);
    }

    /* ---- O8: Eq. 5-6 assembled per phase (L2, L7, L25) ---- */
    const double (*T)[4] = o->T;
    const int p2p_inter = pb->N > 1;
    o->p2p = orc_coll(pb, P2P, X, 1, p2p_inter);
    double t = (l - c) * (T[0][0] + T[0][1]) + c * (T[1][0] + T[1][1]);
    double d = (l - c) * ((T[0][2] - T[0][0]) + (T[0][3] - T[0][1])) +
               c * ((T[1][2] - T[1][0]) + (T[1][3] - T[1][1]));
    if (gr.first) {
        t += T[2][0] + T[2][1];
        d += (T[2][2] - T[2][0]) + (T[2][3] - T[2][1]);
    }
    if (gr.last) {
        t += T[3][0] + T[3][1];
        d += (T[3][2] - T[3][0]) + (T[3][3] - T[3][1]);
    }
    if (!gr.last) t += o->p2p;      /* send activations to the next stage */
    if (!gr.first) t += o->p2p;     /* send gradients to the previous stage */
    o->t = t;
    o->d = std::max(0.0, d);

    /* ---- O9: peak memory, every term multiplied by D = Q*TP*DP (exact) ---- */
    const i128 D = (i128)Q * TP * DP;
    const i128 iPl = (i128)2 * md.h * md.h + (i128)2 * md.h * (md.k * (int64_t)md.h / md.a) +
                     (i128)(2 + md.g) * md.h * md.f + (i128)md.nrm * md.h;       /* P_layer */
    const i128 iVh = (i128)md.V * md.h;
    const i128 P_raw = (i128)l * iPl + gr.first * iVh + gr.last * iVh;           /* TP * P_st */
    const i128 sw_ = (z == 3) ? 1 : DP, sg_ = (z >= 2) ? 1 : DP, so_ = (z >= 1) ? 1 : DP; /* DP*sigma */
    const int m2 = std::min(l, 2);
    const i128 ikvd = md.k * (int64_t)md.h / md.a;
    /* TP * A_full, TP * A_bnd, TP * A_H (integers) */
    const i128 TA_full = (i128)md.e * md.s * b *
                         ((i128)4 * md.h * TP + 2 * md.h + 2 * ikvd + (i128)(2 + 2 * md.g) * md.f +
                          (i128)(1 - md.fl) * md.a * md.s);
    const i128 TA_bnd = (i128)TP * md.e * md.s * b * md.h;
    const i128 TA_H = (i128)TP * md.e * md.s * b * md.h + (i128)4 * md.s * b * md.V;
    /* M_s = P_st [2(1-WO) sw + 2(1-GO) sg + 12(1-OO) so] */
    const i128 Ms = P_raw * (2 * (Q - cf.kW) * sw_ + 2 * (Q - cf.kG) * sg_ + 12 * (Q - cf.kO) * so_);
    /* M_wb = m2 W_L ([z=3] + [z<3] WO), W_L = e P_layer / TP */
    const i128 Mwb = (i128)m2 * md.e * iPl * DP * ((z == 3) ? Q : cf.kW);
    /* M_gb = m2 Gr_L ([z>=2] + [z<2] GO) */
    const i128 Mgb = (i128)m2 * md.e * iPl * DP * ((z >= 2) ? Q : cf.kG);
    /* M_ob = m2 O_L sigma_o OO, O_L = 12 P_layer / TP */
    const i128 Mob = (i128)m2 * 12 * iPl * so_ * cf.kO;
    /* M_a = w (1-AO) [c A_bnd + (l-c) A_full + last A_H] */
    const i128 Ma = (i128)gr.w * (Q - cf.kA) * DP * ((i128)c * TA_bnd + (i128)(l - c) * TA_full +
                                                      gr.last * TA_H);
    const i128 DAf = (i128)Q * DP * TA_full;                                    /* D * A_full */
    const i128 fwd = Ms + Mwb + Mob + Ma + DAf;                 /* Mem_fwd */
    const i128 bwd = Ms + Mwb + Mgb + Ma + (c > 0 ? DAf : 0) + DAf;   /* Mem_bwd */
    const i128 Dmem = std::max(fwd, bwd);
    o->D = (double)D; o->Ms = (double)Ms; o->Mwb = (double)Mwb; o->Mgb = (double)Mgb;
    o->Mob = (double)Mob; o->Ma = (double)Ma; o->Afull_D = (double)DAf;
    o->mem_fwd_D = (double)fwd; o->mem_bwd_D = (double)bwd;
    o->mem = (double)Dmem / (double)D;
    o->feasible = Dmem <= (i128)pb->mem_budget * D;      /* max(Mem_fwd, Mem_bwd) <= Mem_Budget */
    if (!in_preset(pb, cf)) o->feasible = 0;             /* outside the search-space preset */
    return 0;
}

/* Number of configurations a preset admits: counted one by one over every
 * (group, split, z, c, kW, kG, kO, kA) -- small spaces only. */
extern "C" uint64_t orc_count_space(const orc_problem_t* pb, const orc_group_t* groups, int64_t n_groups) {
    const int nzl = num_zero_levels(pb);
    uint64_t n = 0;
    for (int64_t g = 0; g < n_groups; ++g)
        for (int sp = 0; sp < groups[g].n_splits; ++sp)
            for (int zi = 0; zi < nzl; ++zi)
                for (int c = 0; c <= groups[g].l; ++c)
                    for (int kW = 0; kW <= pb->Q; ++kW)
                        for (int kG = 0; kG <= pb->Q; ++kG)
                            for (int kO = 0; kO <= pb->Q; ++kO)
                                for (int kA = 0; kA <= pb->Q; ++kA) {
                                    CfgId cf = {&groups[g], sp, zero_level(pb, zi), c, kW, kG, kO, kA};
                                    n += in_preset(pb, cf) ? 1 : 0;
                                }
    return n;
}

extern "C" int orc_eval_detail(const orc_problem_t* pb, const orc_group_t* grp, int split, int z,
                               int c, int kW, int kG, int kO, int kA, orc_detail_t* out) {
    if (split < 0 || split >= grp->n_splits) return -1;
    CfgId cf = {grp, split, z, c, kW, kG, kO, kA};
    return eval_config(pb, cf, out);
}

/* O3 decode of a global config index. */
static int decode(const orc_problem_t* pb, const orc_group_t* groups, int64_t n_groups,
                  uint64_t idx, CfgId* cf, int64_t* gi) {
    int64_t lo = 0, hi = n_groups - 1;
    if (n_groups <= 0) return -1;
    if (idx >= groups[hi].config_offset + groups[hi].count) return -1;
    while (lo < hi) {                                  /* last group with config_offset <= idx */
        int64_t mid = (lo + hi + 1) / 2;
        if (groups[mid].config_offset <= idx) lo = mid; else hi = mid - 1;
    }
    const orc_group_t& g = groups[lo];
    const uint64_t Q1 = pb->Q + 1, R = Q1 * Q1 * Q1 * Q1;
    uint64_t local = idx - g.config_offset;
    uint64_t tup = local / R, r = local % R;
    const int nz = num_zero_levels(pb);
    cf->g = &g;
    cf->split = (int)(tup / ((uint64_t)nz * (g.l + 1)));
    uint64_t rem = tup % ((uint64_t)nz * (g.l + 1));
    cf->z = zero_level(pb, (int)(rem / (g.l + 1)));
    cf->c = (int)(rem % (g.l + 1));
    cf->kA = (int)(r % Q1); r /= Q1;                   /* AO fastest */
    cf->kO = (int)(r % Q1); r /= Q1;
    cf->kG = (int)(r % Q1); r /= Q1;
    cf->kW = (int)r;
    *gi = lo;
    return 0;
}

extern "C" int orc_eval_indices(const orc_problem_t* pb, const orc_group_t* groups,
                                int64_t n_groups, const uint64_t* idx, int64_t n, double* t,
                                double* d, double* mem, uint8_t* feasible) {
    int rc = 0;
#pragma omp parallel for schedule(static) reduction(min : rc)
    for (int64_t i = 0; i < n; ++i) {
        CfgId cf; int64_t gi; orc_detail_t o;
        if (decode(pb, groups, n_groups, idx[i], &cf, &gi)) { rc = -1; continue; }
        if (eval_config(pb, cf, &o)) { rc = -2; continue; }
        if (t) t[i] = o.t;
        if (d) d[i] = o.d;
        if (mem) mem[i] = o.mem;
        if (feasible) feasible[i] = (uint8_t)o.feasible;
    }
    return rc;
}

extern "C" int orc_eval_range(const orc_problem_t* pb, const orc_group_t* groups, int64_t n_groups,
                              uint64_t begin, uint64_t end, double* t, double* d, double* mem,
                              uint8_t* feasible) {
    int rc = 0;
    const int64_t n = (int64_t)(end - begin);
#pragma omp parallel for schedule(static) reduction(min : rc)
    for (int64_t k = 0; k < n; ++k) {
        CfgId cf; int64_t gi; orc_detail_t o;
        if (decode(pb, groups, n_groups, begin + (uint64_t)k, &cf, &gi)) { rc = -1; continue; }
        if (eval_config(pb, cf, &o)) { rc = -2; continue; }
        if (t) t[k] = o.t;
        if (d) d[k] = o.d;
        if (mem) mem[k] = o.mem;
        if (feasible) feasible[k] = (uint8_t)o.feasible;
    }
    return rc;
}

/* ------------------------------------------------------------------------ */
/* O10 -- Pareto frontier (Eq. 3-4; ledger L1, L26)                   */
/* p beats q iff x_p <= x_q, y_p <= y_q and (x_p < x_q or y_p < y_q or       */
/* idx_p < idx_q).  The frontier is the set of points beaten by none.        */
/* ------------------------------------------------------------------------ */
static bool beats(const orc_point_t& p, const orc_point_t& q) {
    return p.t <= q.t && p.y <= q.y && (p.t < q.t || p.y < q.y || p.idx < q.idx);
}

static bool by_x_y_idx(const orc_point_t& a, const orc_point_t& b) {
    if (a.t != b.t) return a.t < b.t;
    if (a.y != b.y) return a.y < b.y;
    return a.idx < b.idx;
}

extern "C" int64_t orc_frontier_points(const orc_point_t* pts, int64_t n, int method,
                                       orc_point_t* out) {
    std::vector<orc_point_t> keep;
    if (method == 1 || (method == 0 && n <= 10000)) {
        /* the definition: O(k^2) pairwise filter */
        for (int64_t q = 0; q < n; ++q) {
            bool beaten = false;
            for (int64_t p = 0; p < n && !beaten; ++p)
                if (p != q && beats(pts[p], pts[q])) beaten = true;
            if (!beaten) keep.push_back(pts[q]);
        }
        std::sort(keep.begin(), keep.end(), by_x_y_idx);
    } else {
        /* sort by (x, y, idx); a point survives iff it is the first of its
           equal-x run and its y is below every y of the earlier runs */
        std::vector<orc_point_t> v(pts, pts + n);
        std::sort(v.begin(), v.end(), by_x_y_idx);
        double best_y = std::numeric_limits<double>::infinity();
        for (int64_t i = 0; i < n; ++i) {
            bool run_head = (i == 0) || (v[i].t != v[i - 1].t);
            if (!run_head) continue;
            if (v[i].y < best_y) keep.push_back(v[i]);
            best_y = std::min(best_y, v[i].y);
        }
    }
    for (size_t i = 0; i < keep.size(); ++i) out[i] = keep[i];
    return (int64_t)keep.size();
}

extern "C" uint64_t orc_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static int group_points(const orc_problem_t* pb, const orc_group_t* groups, int64_t n_groups,
                        int64_t g, int ykey, std::vector<orc_point_t>* pts, uint64_t* fp_count,
                        uint64_t* fp_hash) {
    const orc_group_t& gr = groups[g];
    uint64_t cnt = 0, hsum = 0;
    for (uint64_t i = gr.config_offset; i < gr.config_offset + gr.count; ++i) {
        CfgId cf; int64_t gi; orc_detail_t o;
        if (decode(pb, groups, n_groups, i, &cf, &gi)) return -1;
        if (eval_config(pb, cf, &o)) return -2;
        if (!o.feasible) continue;                       /* Eq. 4 constraint */
        cnt++;
        hsum += orc_splitmix64(i);
        orc_point_t p = {i, o.t, ykey ? o.mem : o.d, o.mem, g};
        pts->push_back(p);
    }
    if (fp_count) *fp_count = cnt;
    if (fp_hash) *fp_hash = hsum;
    return 0;
}

extern "C" int orc_group_frontier(const orc_problem_t* pb, const orc_group_t* groups,
                                  int64_t n_groups, int64_t g, int ykey, int method,
                                  orc_point_t* out, int64_t cap, int64_t* n_out,
                                  uint64_t* fp_count, uint64_t* fp_hash) {
    if (g < 0 || g >= n_groups) return -1;
    std::vector<orc_point_t> pts;
    int rc = group_points(pb, groups, n_groups, g, ykey, &pts, fp_count, fp_hash);
    if (rc) return rc;
    std::vector<orc_point_t> fr(pts.size() + 1);
    int64_t k = orc_frontier_points(pts.data(), (int64_t)pts.size(), method, fr.data());
    *n_out = k;
    if (out) {
        if (k > cap) return -3;
        for (int64_t i = 0; i < k; ++i) out[i] = fr[i];
    }
    return 0;
}

extern "C" int orc_sweep(const orc_problem_t* pb, const orc_group_t* groups, int64_t n_groups,
                         int64_t g_begin, int64_t g_end, int ykey, int threads,
                         orc_point_t* out, int64_t cap, int64_t* n_out, int64_t* group_offsets,
                         uint64_t* fp_count, uint64_t* fp_hash) {
    if (g_begin < 0 || g_end > n_groups || g_begin > g_end) return -1;
    const int64_t ng = g_end - g_begin;
    std::vector<std::vector<orc_point_t>> fr(ng);
    std::vector<int> rcs(ng, 0);
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
#endif
    for (int64_t i = 0; i < ng; ++i) {
        std::vector<orc_point_t> pts;
        uint64_t c = 0, h = 0;
        rcs[i] = group_points(pb, groups, n_groups, g_begin + i, ykey, &pts, &c, &h);
        if (fp_count) fp_count[i] = c;
        if (fp_hash) fp_hash[i] = h;
        fr[i].resize(pts.size() + 1);
        int64_t k = orc_frontier_points(pts.data(), (int64_t)pts.size(), 0, fr[i].data());
        fr[i].resize(k);
    }
    int64_t total = 0;
    for (int64_t i = 0; i < ng; ++i) {
        if (rcs[i]) return rcs[i];
        if (group_offsets) group_offsets[i] = total;
        for (auto& p : fr[i]) {
            if (out) {
                if (total >= cap) return -3;
                out[total] = p;
            }
            total++;
        }
    }
    if (group_offsets) group_offsets[ng] = total;
    *n_out = total;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* O11 -- alpha sampling ("a series of alpha in [0,1] sampled          */
/* uniformly"; Eq. 4 objective alpha*G*t + (1-alpha)*d; ledger L29)          */
/* ------------------------------------------------------------------------ */
extern "C" int orc_sample(const orc_point_t* frontier, const int64_t* group_offsets,
                          int64_t n_groups, const orc_group_t* groups, int32_t K,
                          int64_t* picked, int64_t cap, int64_t* n_picked,
                          int64_t* picked_offsets) {
    if (K < 2) return -1;
    int64_t np = 0;
    for (int64_t g = 0; g < n_groups; ++g) {
        if (picked_offsets) picked_offsets[g] = np;
        std::vector<int64_t> mine;
        for (int j = 0; j < K; ++j) {
            const double alpha = (double)j / (K - 1);
            int64_t best = -1;
            double best_score = 0.0;
            for (int64_t i = group_offsets[g]; i < group_offsets[g + 1]; ++i) {
                const orc_point_t& p = frontier[i];
                double score = alpha * groups[g].G * p.t + (1.0 - alpha) * p.y;
                if (best < 0 || score < best_score ||
                    (score == best_score && (p.t < frontier[best].t ||
                                             (p.t == frontier[best].t && p.idx < frontier[best].idx)))) {
                    best = i;
                    best_score = score;
                }
            }
            if (best >= 0 && std::find(mine.begin(), mine.end(), best) == mine.end())
                mine.push_back(best);
        }
        for (int64_t v : mine) {
            if (picked) {
                if (np >= cap) return -3;
                picked[np] = v;
            }
            np++;
        }
    }
    if (picked_offsets) picked_offsets[n_groups] = np;
    *n_picked = np;
    return 0;
}
