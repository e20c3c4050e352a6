// mist_eval.cu -- a2..a8: tuple precompute, per-config evaluation, feasibility
// filter and warp-ballot compaction (sm_100a, FP64 CUDA cores; no tensor
// cores: nothing here is a dense contraction).
//
// Paper: Eq. 4-6 over the overlap schedule template
// (lines 476-492) with the interference model of Alg. 1 (lines 563-605);
// memory per Eq. 4's constraint (line 683).  Readings O4-O9 in DESIGN.md.
//
// Work decomposition: unit = (tuple, kW, kA) -> OO-run = unit + kG -> config =
// run + kO.  t never reads OO (P13), so the F phases are evaluated once per unit,
// B and B' once per run, and only the first-microbatch forward F' and the memory
// per config.  Memory is evaluated as exact integers scaled by D = Q*TP*DP (O9),
// so feasibility is bit-exact.  The frontier sweep (k_eval_q, CTA run queue):
// each CTA takes a window of 512 units, two per thread for the per-unit setup
// (L20 twins and the tuple-level R7 cut first, then the F rows, the first
// feasible run in closed form and the unit-level R7 cut, R7-R9); the
// surviving runs of the window are numbered by a block prefix sum and dealt to
// warps in batches of 32 from a shared counter.  The pilot
// sub-grid sweep runs on the same kernel (MODE 2); k_eval is the lockstep
// variant used for the dense outputs (and the round-1 pilot, A/B knob).
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <atomic>

#include <cstdlib>
#include <cstring>

#include "mist_internal.h"

namespace mist {

typedef unsigned long long u64;

// ---------------------------------------------------------------------------
// a2: tuple precompute
// ---------------------------------------------------------------------------
__device__ __forceinline__ double coll_time(const DevProblem& P, int kind, double bytes, int gsz,
                                            int inter) {
    if (gsz == 1) return 0.0;   // O5: a group of one does not communicate
    const double c = (kind == kAR) ? 2.0 * (gsz - 1) / gsz : (double)(gsz - 1) / gsz;
    return c * bytes / P.bw[kind][inter] + P.lat[kind][inter];
}

__device__ void block_const(const DevProblem& P, BlockConst& bc, int z, int DP, int dp_inter,
                            double ARtp, double W, double Gr, double O, double A0, double A1,
                            double Tf, double Tb, int nf, int nb) {
    const double sw = (z == 3) ? 1.0 / DP : 1.0;   // sigma_w, sigma_g, sigma_o
    const double sg = (z >= 2) ? 1.0 / DP : 1.0;
    const double so = (z >= 1) ? 1.0 / DP : 1.0;
    const double ARf = nf * ARtp, ARb = nb * ARtp;
    const double AGw = coll_time(P, kAG, W, DP, dp_inter);
    const double RSg = coll_time(P, kRS, Gr, DP, dp_inter);
    const double ARg = coll_time(P, kAR, Gr, DP, dp_inter);
    bc.C_F = Tf + ARf;
    bc.C_B = Tb + ARb;
    bc.C_B1 = Tb + ARb + (Tf + ARf);                       // recompute (L17)
    bc.N_F = (z == 3) ? AGw : 0.0;
    bc.N_B = ((z == 3) ? AGw : 0.0) + ((z >= 2) ? RSg : 0.0);
    bc.N_Fp = bc.N_F + ((z == 1 || z == 2) ? AGw : 0.0);   // post-update gather (L12)
    bc.N_Bp = bc.N_B + ((z == 0) ? ARg : 0.0) + ((z == 1) ? RSg : 0.0);
    const double qh = P.Q * P.bw_h2d, qd = P.Q * P.bw_d2h;
    bc.sWh = sw * W / qh; bc.sGh = sg * Gr / qh; bc.sOh = so * O / qh;
    bc.sWd = sw * W / qd; bc.sGd = sg * Gr / qd; bc.sOd = so * O / qd;
    bc.sAh = A0 / qh; bc.sAd = A0 / qd;
    bc.sAh1 = A1 / qh; bc.sAd1 = A1 / qd;
}

__device__ int find_group_by_tuple(const DevGroup* groups, int ng, u64 T) {
    int lo = 0, hi = ng - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (groups[mid].tuple_offset <= T) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ void make_tuple(const DevProblem& P, const DevGroup* groups, int ng,
                           const double* __restrict__ coef, u64 T, TupleConst& o) {
    const int gi = find_group_by_tuple(groups, ng, T);
    const DevGroup& G = groups[gi];
    const u64 local = T - G.tuple_offset;
    const u64 per_split = (u64)P.nz * (G.l + 1);
    const int split = (int)(local / per_split);
    const int rem = (int)(local - (u64)split * per_split);
    const int zi = rem / (G.l + 1);
    const int z = P.zlev[zi];
    const int c = rem % (G.l + 1);
    const int TP = G.tp[split], DP = G.dp[split], b = G.b[split], ti = G.ti[split];
    const int rows = P.n_b * P.n_tp;
    const double Tf = coef[0 * rows + ti], Tb = coef[1 * rows + ti];
    const double Tef = coef[2 * rows + ti], Teb = coef[3 * rows + ti];
    const double Thf = coef[4 * rows + ti], Thb = coef[5 * rows + ti];
    const int l = G.l, Q = P.Q;
    const long long kvd = (long long)P.k * P.h / P.a;
    const double e = P.e, s = P.s, h = P.h, bb = b;
    const double Pl = (double)(2LL * P.h * P.h + 2LL * P.h * kvd + (long long)(2 + P.g) * P.h * P.f +
                               (long long)P.nrm * P.h);            // P_layer (O4)
    const double Vh = (double)P.V * P.h;                            // P_E = P_H (untied)
    const double X = e * s * bb * h;                                // boundary activation bytes
    // TP * A_full, TP * A_bnd, TP * A_H (integers; O4 with dropout-free layers)
    const double TA_full = e * s * bb * (4.0 * h * TP + 2.0 * h + 2.0 * (double)kvd +
                                         (2.0 + 2.0 * P.g) * P.f + (1.0 - P.fl) * (double)P.a * s);
    const double TA_bnd = (double)TP * e * s * bb * h;
    const double TA_H = (double)TP * e * s * bb * h + 4.0 * s * bb * P.V;
    const double A_full = TA_full / TP, A_bnd = TA_bnd / TP, A_H = TA_H / TP;
    const int dp_inter = G.n > 1;
    const double ARtp = coll_time(P, kAR, X, TP, 0);               // TP groups intra-node

    o.idx_base = T * (u64)P.Q1 * P.Q1 * P.Q1 * P.Q1;
    o.group = gi; o.first = G.first; o.last = G.last; o.c = c;
    o.nl0 = (double)(l - c); o.nl1 = (double)c;
    const int p2p_inter = P.N > 1;
    const double p2p = X / P.bw[kP2P][p2p_inter] + P.lat[kP2P][p2p_inter];
    o.t_p2p = (G.last ? 0.0 : p2p) + (G.first ? 0.0 : p2p);
    const int nl = 2 - P.p;                                          // TP all-reduces per layer
    block_const(P, o.L, z, DP, dp_inter, ARtp, e * Pl / TP, e * Pl / TP, 12.0 * Pl / TP, A_full,
                A_bnd, Tf, Tb, nl, nl);
    if (G.first)
        block_const(P, o.E, z, DP, dp_inter, ARtp, e * Vh / TP, e * Vh / TP, 12.0 * Vh / TP, 0.0, 0.0,
                    Tef, Teb, 1, 0);
    if (G.last)
        block_const(P, o.H, z, DP, dp_inter, ARtp, e * Vh / TP, e * Vh / TP, 12.0 * Vh / TP, A_H, A_H,
                    Thf, Thb, 0, 1);

    // O9, scaled by D = Q*TP*DP.  All non-negative integers; exact below 2^53.
    const double sw_ = (z == 3) ? 1.0 : DP, sg_ = (z >= 2) ? 1.0 : DP, so_ = (z >= 1) ? 1.0 : DP;
    const double Praw = (double)l * Pl + (G.first ? Vh : 0.0) + (G.last ? Vh : 0.0);  // TP * P_st
    const double m2 = (double)min(l, 2);
    o.mW = 2.0 * Praw * sw_;
    o.mG = 2.0 * Praw * sg_;
    o.mO = 12.0 * Praw * so_;
    const double lay = m2 * e * Pl * DP;
    o.wb_c = (z == 3) ? lay * Q : 0.0;  o.wb_k = (z == 3) ? 0.0 : lay;
    o.gb_c = (z >= 2) ? lay * Q : 0.0;  o.gb_k = (z >= 2) ? 0.0 : lay;
    o.ob_k = m2 * 12.0 * Pl * so_;
    o.ma_k = (double)G.w * DP * ((double)c * TA_bnd + (double)(l - c) * TA_full +
                                 (G.last ? TA_H : 0.0));
    o.DA = (double)Q * DP * TA_full;
    o.DAx = c > 0 ? o.DA : 0.0;
    o.D = (double)Q * TP * DP;
    o.DMB = (double)P.mem_budget * o.D;
    // preset: CKPT c in {0, l} only -- a tuple outside it is
    // never feasible (every D*mem >= 0 > -1)
    if (P.ckpt_ends && c != 0 && c != l) o.DMB = -1.0;
    o.twin_T = (DP == 1 && zi > 0) ? T - (u64)zi * (u64)(l + 1) : ~0ull;
    o.pad_ = 0;
}

// a2 over a rank's block-cyclic share: seg[2*s] = first tuple of segment s,
// seg[2*s+1] = its first position in `out` (prefix of the segment lengths,
// seg[2*nseg+1] = total); one launch for all segments.
// Table position of the logical tuple j when `halves` is set: the even logical
// positions fill the first half of the table, the odd ones the second, so a sweep of
// the first half refines the staircase of every group before the second half runs.
__device__ __forceinline__ u64 half_order(u64 i, u64 nT, bool halves) {
    if (!halves) return i;
    const u64 h = (nT + 1) / 2;
    return i < h ? 2 * i : 2 * (i - h) + 1;
}

// Both precompute kernels run kPreThreads threads per CTA: every thread builds its
// tuple into shared memory and the CTA then writes its tuples out as one contiguous,
// coalesced stream (a per-thread struct store would touch 72 separate 576-B-strided
// words per warp instruction).
constexpr int kPreThreads = 64;

__device__ __forceinline__ void store_tuples(TupleConst* sT, u64 o0, u64 nT, TupleConst* __restrict__ out) {
    __syncthreads();
    const int nt = (int)min((u64)kPreThreads, nT - o0);
    const double2* src = reinterpret_cast<const double2*>(sT);
    double2* dst = reinterpret_cast<double2*>(out + o0);
    const int nw = nt * (int)(sizeof(TupleConst) / 16);
    for (int i = threadIdx.x; i < nw; i += kPreThreads) dst[i] = src[i];
    __syncthreads();
}

__global__ void __launch_bounds__(kPreThreads)
k_tuple_precompute_segs(DevProblem P, const DevGroup* __restrict__ groups, int ng,
                        const double* __restrict__ coef, const u64* __restrict__ seg, int nseg,
                        u64 nT, TupleConst* __restrict__ out, bool halves) {
    __shared__ __align__(16) TupleConst sT[kPreThreads];
    for (u64 o0 = (u64)blockIdx.x * kPreThreads; o0 < nT; o0 += (u64)gridDim.x * kPreThreads) {
        const u64 o = o0 + threadIdx.x;
        if (o < nT) {
            const u64 i = half_order(o, nT, halves);
            int lo = 0, hi = nseg - 1;              // last segment whose first position <= i
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (seg[2 * mid + 1] <= i) lo = mid; else hi = mid - 1;
            }
            make_tuple(P, groups, ng, coef, seg[2 * lo] + (i - seg[2 * lo + 1]), sT[threadIdx.x]);
        }
        store_tuples(sT, o0, nT, out);
    }
}

__global__ void __launch_bounds__(kPreThreads)
k_tuple_precompute(DevProblem P, const DevGroup* __restrict__ groups, int ng,
                   const double* __restrict__ coef, u64 T0, u64 nT,
                   TupleConst* __restrict__ out, bool halves) {
    __shared__ __align__(16) TupleConst sT[kPreThreads];
    for (u64 o0 = (u64)blockIdx.x * kPreThreads; o0 < nT; o0 += (u64)gridDim.x * kPreThreads) {
        const u64 o = o0 + threadIdx.x;
        if (o < nT) make_tuple(P, groups, ng, coef, T0 + half_order(o, nT, halves), sT[threadIdx.x]);
        store_tuples(sT, o0, nT, out);
    }
}

// ---------------------------------------------------------------------------
// a5: Alg. 1 PredINTF.  At each round at most one subset matches
// the row's nonzero pattern, so the literal algorithm is "look up
// the factor row of the current pattern, scale, take the min, update".  The
// shared-memory table holds {f, g} per (pattern, channel): f = F, g = 1/F for
// member channels and f = 1, g = 0 for the others, so that non-member
// channels stay (+-)0 through the update without selects; the min over the
// members is a predicated compare-and-select chain (DSETP + 2 FSEL each).
// Channels: x0 = C, x1 = NCCL (G2G), x2 = H2D (C2G), x3 = D2H (G2C).
// ---------------------------------------------------------------------------
typedef double2 FGRow[4];

// min/max without fmin/fmax's NaN handling (no NaN can occur here): DSETP + 2 selects
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }

// Code-size knobs for A/B builds (-DMIST_NI_*): one shared, called copy instead
// of an inlined copy per call site (the eval kernel's SASS is ~127 KB against a
// 32 KB L1.5 instruction cache).
#ifdef MIST_NI_PRED
#define MIST_PRED_ATTR __noinline__
#else
#define MIST_PRED_ATTR __forceinline__
#endif
#ifdef MIST_NI_DLB
#define MIST_DLB_ATTR __noinline__
#else
#define MIST_DLB_ATTR __forceinline__
#endif
#ifdef MIST_NI_CUT
#define MIST_CUT_ATTR __noinline__
#else
#define MIST_CUT_ATTR
#endif

__device__ MIST_PRED_ATTR double pred_intf_gen(double x0, double x1, double x2, double x3,
                                               const FGRow* __restrict__ FG) {
    double T = 0.0;
#pragma unroll
    for (int round = 0; round < 3; ++round) {
        const bool q0 = x0 != 0.0, q1 = x1 != 0.0, q2 = x2 != 0.0, q3 = x3 != 0.0;
        const int pat = (int)q0 | ((int)q1 << 1) | ((int)q2 << 2) | ((int)q3 << 3);
        if (__popc(pat) < 2) break;
        const double2 a0 = FG[pat][0], a1 = FG[pat][1], a2 = FG[pat][2], a3 = FG[pat][3];
        const double s0 = x0 * a0.x, s1 = x1 * a1.x, s2 = x2 * a2.x, s3 = x3 * a3.x;
        // min over the member channels: predicated compare-and-select chain
        double ov = q0 ? s0 : CUDART_INF;
        ov = (q1 && s1 < ov) ? s1 : ov;
        ov = (q2 && s2 < ov) ? s2 : ov;
        ov = (q3 && s3 < ov) ? s3 : ov;
        x0 = (s0 - ov) * a0.y;     // argmin -> exactly 0; non-members -> -0 (g = 0)
        x1 = (s1 - ov) * a1.y;
        x2 = (s2 - ov) * a2.y;
        x3 = (s3 - ov) * a3.y;
        T += ov;
    }
    return T + (((x0 + x1) + x2) + x3);
}

template <bool UNIT>
__device__ __forceinline__ double pred_intf(double x0, double x1, double x2, double x3,
                                            const FGRow* __restrict__ FG) {
    if (UNIT) return dmax(dmax(x0, x1), dmax(x2, x3));   // unit factors: perfect overlap = max
    return pred_intf_gen(x0, x1, x2, x3, FG);
}

// Loop nest of one thread: unit (kW, kA) -> run kG -> config kO.
// F phases read only (kW, kA) (O6: F = [C, NCCL, kW sWh, kA sAd]), so they are
// evaluated once per unit; B, B' and t once per run (t never reads OO, P13);
// F' and the memory once per config.

// Per-unit state: the F phase of every block.
struct UnitState {
    double TF_L0, TF_L1, TF_E, TF_H;            // T(F) of each block (0 when absent)
    double FH_L, FH_E, FH_H;                    // F H2D = kW sWh
    double FD_L0, FD_L1, FD_E, FD_H;            // F D2H = kA sAd (r = 0 / 1 for layers)
};

// Per-run state: everything that does not depend on kO.
struct RunState {
    double t, dbase;
    double dsc;                     // deferred B' (DEFER): rounding scale of the lower-bound dbase
    bool dexact;                    // dbase is exact (else a lower bound from R5 rows of B')
    double FpH_L, FpD_L0, FpD_L1;   // F' layer H2D / D2H at kO = 0
    double FpH_E, FpD_E, FpH_H, FpD_H;
    double Kf, Kb;                  // D*Mem_fwd / D*Mem_bwd without the (Q-kO), kO terms
};

// O9 (exact integers): the kO-independent part of D*Mem_fwd and D*Mem_bwd.
__device__ __forceinline__ void run_memory(const TupleConst& tc, double kW, double kG, double kA, double Q,
                                           RunState& rs) {
    const double common = tc.mW * (Q - kW) + tc.mG * (Q - kG) + (tc.wb_c + tc.wb_k * kW) +
                          tc.ma_k * (Q - kA) + tc.DA;
    rs.Kf = common;
    rs.Kb = common + (tc.gb_c + tc.gb_k * kG) + tc.DAx;
}

// D*max(Mem_fwd, Mem_bwd) of config kO of the run (Eq. 4)
__device__ __forceinline__ double mem_kO(const TupleConst& tc, const RunState& rs, double kO, double Q) {
    const double qo = Q - kO;
    const double fwd = rs.Kf + tc.mO * qo + tc.ob_k * kO;   // Mem_fwd: + M_ob
    const double bwd = rs.Kb + tc.mO * qo;                  // Mem_bwd: + M_gb, recompute buffer
    return dmax(fwd, bwd);
}

// Smallest feasible kO of a run whose kO = Q config is feasible (R2).  D*Mem_fwd
// and D*Mem_bwd are affine in kO with slopes -(mO - ob_k) <= 0 and -mO <= 0, so
// the boundary is max over the two of ceil((D*Mem_X(0) - D*MB) / slope); a
// float reciprocal gives an under-estimate (error << 1 step) and the exact
// integer memory test walks it up to the boundary (feasibility is monotone in kO).
__device__ __forceinline__ unsigned first_feasible_kO(const TupleConst& tc, const RunState& rs, double Q) {
    if (mem_kO(tc, rs, 0.0, Q) <= tc.DMB) return 0u;
    const double rb = rs.Kb + tc.mO * Q - tc.DMB;          // bwd(k) <= DMB  <=>  mO k >= rb
    const double sf = tc.mO - tc.ob_k;
    const double rf = rs.Kf + tc.mO * Q - tc.DMB;          // fwd(k) <= DMB  <=>  sf k >= rf
    double g = 0.0;
    if (rb > 0.0) g = tc.mO > 0.0 ? rb * (double)__frcp_rn((float)tc.mO) : Q;
    if (rf > 0.0) g = dmax(g, sf > 0.0 ? rf * (double)__frcp_rn((float)sf) : Q);
    g = g * (1.0 - 1e-5) - 1e-5;                           // under-estimate (float reciprocal: 2^-23 relative)
    int k = g > 1.0 ? (int)ceil(g < Q ? g : Q) : 1;
    const int iQ = (int)Q;
    while (k < iQ && !(mem_kO(tc, rs, (double)k, Q) <= tc.DMB)) ++k;
    return (unsigned)k;
}

// First run (kG) of a unit whose kO = kOend config fits the budget, in closed form
// (R2' applied to kG, like R2" to kO): under the kG-suffix property (mG >= gb_k),
// D*Mem_fwd and D*Mem_bwd at kO = kOend are affine in kG with slopes -mG and
// -(mG - gb_k), so the boundary is the max of two ceilings; a float reciprocal
// under-estimates it and the exact integer test walks up to it.  Returns gend when
// no run of the unit is feasible.
__device__ __forceinline__ unsigned first_feasible_kG(const TupleConst& tc, double kW, double kA, unsigned gend,
                                                      double kOend, double Q) {
    RunState r0;
    run_memory(tc, kW, 0.0, kA, Q, r0);
    const double f0 = r0.Kf + tc.mO * (Q - kOend) + tc.ob_k * kOend;
    const double b0 = r0.Kb + tc.mO * (Q - kOend);
    if (dmax(f0, b0) <= tc.DMB) return 0u;
    const double sb = tc.mG - tc.gb_k;
    double g = 0.0;
    if (f0 > tc.DMB) g = tc.mG > 0.0 ? (f0 - tc.DMB) * (double)__frcp_rn((float)tc.mG) : 1e30;
    if (b0 > tc.DMB) g = dmax(g, sb > 0.0 ? (b0 - tc.DMB) * (double)__frcp_rn((float)sb) : 1e30);
    g = g * (1.0 - 1e-5) - 1e-5;                           // under-estimate (float reciprocal: 2^-23 relative)
    unsigned k = g > 1.0 ? (unsigned)ceil(g < (double)gend ? g : (double)gend) : 1u;
    RunState rm;
    while (k < gend) {
        run_memory(tc, kW, (double)k, kA, Q, rm);
        if (mem_kO(tc, rm, kOend, Q) <= tc.DMB) break;
        ++k;
    }
    return k;
}

// F phases of the unit
template <bool UNIT>
__device__ __forceinline__ void unit_forward(const TupleConst& tc, double kW, double kA, const FGRow* FG,
                                             UnitState& us) {
    us.FH_L = kW * tc.L.sWh;
    us.FD_L0 = kA * tc.L.sAd;
    us.FD_L1 = kA * tc.L.sAd1;
    us.TF_L0 = us.TF_L1 = us.TF_E = us.TF_H = 0.0;
    if (tc.nl0 > 0.0) us.TF_L0 = pred_intf<UNIT>(tc.L.C_F, tc.L.N_F, us.FH_L, us.FD_L0, FG);
    if (tc.nl1 > 0.0) us.TF_L1 = pred_intf<UNIT>(tc.L.C_F, tc.L.N_F, us.FH_L, us.FD_L1, FG);
    if (tc.first) {
        us.FH_E = kW * tc.E.sWh;
        us.FD_E = kA * tc.E.sAd;
        us.TF_E = pred_intf<UNIT>(tc.E.C_F, tc.E.N_F, us.FH_E, us.FD_E, FG);
    }
    if (tc.last) {
        us.FH_H = kW * tc.H.sWh;
        us.FD_H = kA * tc.H.sAd;
        us.TF_H = pred_intf<UNIT>(tc.H.C_F, tc.H.N_F, us.FH_H, us.FD_H, FG);
    }
}

// sum over blocks of count * T(F) (Eq. 5's forward part)
__device__ __forceinline__ double unit_tf(const TupleConst& tc, const UnitState& us) {
    double tf = 0.0;
    if (tc.nl0 > 0.0) tf += tc.nl0 * us.TF_L0;
    if (tc.nl1 > 0.0) tf += tc.nl1 * us.TF_L1;
    if (tc.first) tf += us.TF_E;
    if (tc.last) tf += us.TF_H;
    return tf;
}

// B and B' of one block; returns T(B), writes T(B') - T(B).
// Not inlined: it runs once per run and block, and one shared copy instead of four
// inlined ones shrinks the eval loop's instruction footprint (same-box A/B: cfg2
// 77.5 -> 74.5 ms, profiles/r1/ab_ni_summary.txt).
template <bool UNIT>
__device__ __noinline__ double block_backward(const BlockConst& b, bool r1, double FH, double kG, double kA,
                                                 const FGRow* FG, double& dBp) {
    const double sAh = r1 ? b.sAh1 : b.sAh;
    const double CB = r1 ? b.C_B1 : b.C_B;                   // a checkpointed layer recomputes (L17)
    const double BH = FH + kG * b.sGh + kA * sAh, BD = kG * b.sGd;
    const double TB = pred_intf<UNIT>(CB, b.N_B, BH, BD, FG);
    dBp = (b.N_Bp == b.N_B) ? 0.0 : pred_intf<UNIT>(CB, b.N_Bp, BH, BD, FG) - TB;
    return TB;
}

// Deferred B' (DEFER): B's exact row and, when B' differs (z < 2 at DP > 1), only
// the R5 bound of B' -- d's backward part T(B') - T(B) >= lb(B') - T(B).  The bound
// test of the first configs runs on that lower bound; a run that survives it gets
// the exact B' rows (run_dbase_exact) before any d is evaluated, so every cut is
// exact and every d is the same as without deferral.
template <bool UNIT, bool NI>
__device__ __forceinline__ double lb_row(double x0, double x1, double x2, double x3, const FGRow* FG);

template <bool UNIT>
__device__ __noinline__ double block_backward_lb(const BlockConst& b, bool r1, double FH, double kG, double kA,
                                                 const FGRow* FG, double& dBp_lb) {
    const double sAh = r1 ? b.sAh1 : b.sAh;
    const double CB = r1 ? b.C_B1 : b.C_B;
    const double BH = FH + kG * b.sGh + kA * sAh, BD = kG * b.sGd;
    const double TB = pred_intf<UNIT>(CB, b.N_B, BH, BD, FG);
    dBp_lb = (b.N_Bp == b.N_B) ? 0.0 : lb_row<UNIT, false>(CB, b.N_Bp, BH, BD, FG) - TB;
    return TB;
}

// exact sum count (T(B') - T(B)), the same operations in the same order as run_backward
template <bool UNIT>
__device__ __noinline__ double run_dbase_exact(const TupleConst& tc, const UnitState& us, double kG, double kA,
                                               const FGRow* FG) {
    double db = 0.0, dBp;
    if (tc.nl0 > 0.0) { block_backward<UNIT>(tc.L, false, us.FH_L, kG, kA, FG, dBp); db += tc.nl0 * dBp; }
    if (tc.nl1 > 0.0) { block_backward<UNIT>(tc.L, true, us.FH_L, kG, kA, FG, dBp); db += tc.nl1 * dBp; }
    if (tc.first) { block_backward<UNIT>(tc.E, false, us.FH_E, kG, kA, FG, dBp); db += dBp; }
    if (tc.last) { block_backward<UNIT>(tc.H, false, us.FH_H, kG, kA, FG, dBp); db += dBp; }
    return db;
}

// Stable phases of the run: t (Eq. 5) and the kO-independent part of d (Eq. 6).
template <bool UNIT, bool DEFER = false>
__device__ __forceinline__ void run_backward(const TupleConst& tc, const UnitState& us, double kW, double kG,
                                             double kA, const FGRow* FG, RunState& rs) {
    double tb = 0.0, db = 0.0, dBp, dsc = 0.0;
    bool exact = true;
    auto bb = [&](const BlockConst& b, bool r1, double FH) -> double {
        if (!DEFER) return block_backward<UNIT>(b, r1, FH, kG, kA, FG, dBp);
        const double TB = block_backward_lb<UNIT>(b, r1, FH, kG, kA, FG, dBp);
        if (b.N_Bp != b.N_B) { exact = false; dsc += fabs(dBp) + 2.0 * TB; }
        return TB;
    };
    rs.FpH_L = us.FH_L + kG * tc.L.sGh;
    rs.FpD_L0 = us.FD_L0 + kW * tc.L.sWd;
    rs.FpD_L1 = us.FD_L1 + kW * tc.L.sWd;
    if (tc.nl0 > 0.0) {
        tb += tc.nl0 * bb(tc.L, false, us.FH_L);
        db += tc.nl0 * dBp;
    }
    if (tc.nl1 > 0.0) {
        tb += tc.nl1 * bb(tc.L, true, us.FH_L);
        db += tc.nl1 * dBp;
    }
    if (tc.first) {
        tb += bb(tc.E, false, us.FH_E);
        db += dBp;
        rs.FpH_E = us.FH_E + kG * tc.E.sGh;
        rs.FpD_E = us.FD_E + kW * tc.E.sWd;
    }
    if (tc.last) {
        tb += bb(tc.H, false, us.FH_H);
        db += dBp;
        rs.FpH_H = us.FH_H + kG * tc.H.sGh;
        rs.FpD_H = us.FD_H + kW * tc.H.sWd;
    }
    rs.t = (unit_tf(tc, us) + tb) + tc.t_p2p;
    rs.dbase = db;                   // d = db + sum count * (T(F') - T(F)), block by block (Eq. 6)
    rs.dexact = exact;
    rs.dsc = dsc * (tc.nl0 + tc.nl1 + 2.0);   // counts multiply the per-block terms
}

// d of config kO of the run: first-microbatch forward F' of every block (Eq. 6).
template <bool UNIT>
__device__ __forceinline__ double d_kO(const TupleConst& tc, const UnitState& us, const RunState& rs, double kO,
                                       const FGRow* FG) {
    // per-block differences T(F') - T(F): exactly 0 for a block whose F' equals its F
    double ds = rs.dbase;
    const double H = rs.FpH_L + kO * tc.L.sOh;
    if (tc.nl0 > 0.0)
        ds += tc.nl0 * (pred_intf<UNIT>(tc.L.C_F, tc.L.N_Fp, H, rs.FpD_L0 + kO * tc.L.sOd, FG) - us.TF_L0);
    if (tc.nl1 > 0.0)
        ds += tc.nl1 * (pred_intf<UNIT>(tc.L.C_F, tc.L.N_Fp, H, rs.FpD_L1 + kO * tc.L.sOd, FG) - us.TF_L1);
    if (tc.first)
        ds += pred_intf<UNIT>(tc.E.C_F, tc.E.N_Fp, rs.FpH_E + kO * tc.E.sOh, rs.FpD_E + kO * tc.E.sOd, FG) - us.TF_E;
    if (tc.last)
        ds += pred_intf<UNIT>(tc.H.C_F, tc.H.N_Fp, rs.FpH_H + kO * tc.H.sOh, rs.FpD_H + kO * tc.H.sOd, FG) - us.TF_H;
    return ds > 0.0 ? ds : 0.0;                             // L25: clamp at 0
}

// Lower bound of one Alg. 1 row (R4, R5).  With every factor >= 1 each channel's
// isolated time is consumed at rate 1/f <= 1 per unit of elapsed time, so
// T >= max_j x_j (R4).  Tighter (R5): the first round lasts ov = min_j x_j F_j
// over the nonzero pattern S and leaves channel m with x_m - ov/F_m, which takes
// at least that long again, so T >= x_m + ov (1 - 1/F_m) for every m in S (and
// T >= ov for the zero channels, which have g = 0 in the table).  Unit factors
// make Alg. 1 the max itself, so only R4 is used there.
__device__ __forceinline__ double lb_row_gen(double x0, double x1, double x2, double x3, const FGRow* FG);

// NI: one shared, called copy of the bound row instead of an inlined copy per call
// site.  The eval kernel's SASS (~127 KB) is far above the 32 KB L1.5 instruction
// cache; the called copy pays where the kO loops are short (Q = 10: cfg2 25.0 ->
// 22.7 ms) and costs where they are long (Q = 50: cfg5 windows +1.5-3%), so the
// launcher picks it by Q (eval_ni).
__device__ __noinline__ double lb_row_ni(double x0, double x1, double x2, double x3, const FGRow* FG) {
    return lb_row_gen(x0, x1, x2, x3, FG);
}

template <bool UNIT, bool NI = false>
__device__ __forceinline__ double lb_row(double x0, double x1, double x2, double x3, const FGRow* FG) {
    if (UNIT) return dmax(dmax(x0, x1), dmax(x2, x3));
    if (NI) return lb_row_ni(x0, x1, x2, x3, FG);
    return lb_row_gen(x0, x1, x2, x3, FG);
}

__device__ __forceinline__ double lb_row_gen(double x0, double x1, double x2, double x3, const FGRow* FG) {
    const double mx = dmax(dmax(x0, x1), dmax(x2, x3));
    const unsigned pat = (unsigned)(x0 != 0.0) | ((unsigned)(x1 != 0.0) << 1) | ((unsigned)(x2 != 0.0) << 2) |
                         ((unsigned)(x3 != 0.0) << 3);
    if (__popc(pat) < 2) return mx;
    const double2 r0 = FG[pat][0], r1 = FG[pat][1], r2 = FG[pat][2], r3 = FG[pat][3];
    const double s0 = x0 * r0.x, s1 = x1 * r1.x, s2 = x2 * r2.x, s3 = x3 * r3.x;
    double ov = (pat & 1u) ? s0 : CUDART_INF;
    ov = ((pat & 2u) && s1 < ov) ? s1 : ov;
    ov = ((pat & 4u) && s2 < ov) ? s2 : ov;
    ov = ((pat & 8u) && s3 < ov) ? s3 : ov;
    const double b0 = fma(ov, 1.0 - r0.y, x0), b1 = fma(ov, 1.0 - r1.y, x1);
    const double b2 = fma(ov, 1.0 - r2.y, x2), b3 = fma(ov, 1.0 - r3.y, x3);
    return dmax(dmax(b0, b1), dmax(b2, b3));
}

// True when every F' row has nonzero H2D and D2H at kO = 0, i.e. the nonzero
// pattern of the rows is the same for every kO of the run.
__device__ __forceinline__ bool fp_pattern_fixed(const TupleConst& tc, const RunState& rs) {
    bool ok = true;
    if (tc.nl0 > 0.0) ok = ok && rs.FpH_L != 0.0 && rs.FpD_L0 != 0.0;
    if (tc.nl1 > 0.0) ok = ok && rs.FpH_L != 0.0 && rs.FpD_L1 != 0.0;
    if (tc.first) ok = ok && rs.FpH_E != 0.0 && rs.FpD_E != 0.0;
    if (tc.last) ok = ok && rs.FpH_H != 0.0 && rs.FpD_H != 0.0;
    return ok;
}

// Lower bound of d at config kO: rs.dbase + sum count * (lb_row(F') - T(F)) over the blocks.
// `scale` bounds the magnitudes summed, for a rounding margin.
template <bool UNIT, bool NI>
__device__ MIST_DLB_ATTR double d_lower_bound(const TupleConst& tc, const UnitState& us, const RunState& rs,
                                                double kO, const FGRow* FG, double& scale) {
    double lb = rs.dbase, sc = fabs(rs.dbase);
    const double H = rs.FpH_L + kO * tc.L.sOh;
    if (tc.nl0 > 0.0) {
        const double m = lb_row<UNIT, NI>(tc.L.C_F, tc.L.N_Fp, H, rs.FpD_L0 + kO * tc.L.sOd, FG);
        lb += tc.nl0 * (m - us.TF_L0); sc += tc.nl0 * (m + us.TF_L0);
    }
    if (tc.nl1 > 0.0) {
        const double m = lb_row<UNIT, NI>(tc.L.C_F, tc.L.N_Fp, H, rs.FpD_L1 + kO * tc.L.sOd, FG);
        lb += tc.nl1 * (m - us.TF_L1); sc += tc.nl1 * (m + us.TF_L1);
    }
    if (tc.first) {
        const double m = lb_row<UNIT, NI>(tc.E.C_F, tc.E.N_Fp, rs.FpH_E + kO * tc.E.sOh, rs.FpD_E + kO * tc.E.sOd, FG);
        lb += m - us.TF_E; sc += m + us.TF_E;
    }
    if (tc.last) {
        const double m = lb_row<UNIT, NI>(tc.H.C_F, tc.H.N_Fp, rs.FpH_H + kO * tc.H.sOh, rs.FpD_H + kO * tc.H.sOd, FG);
        lb += m - us.TF_H; sc += m + us.TF_H;
    }
    scale = sc;
    return lb;
}

// R7 (run cut before the backward rows).  t of run kG is (sum count T(F)) + sum count
// T(B(kG)) + p2p, with T(F) exact per unit and T(B) bounded below by R4/R5.  The
// bound is non-decreasing in kG: the B channels H2D = FH + kG sGh + kA sAh and
// D2H = kG sGd grow with kG, R5 is monotone in the channels while the nonzero
// pattern is fixed (every kG >= 1), and R4 (the max, used at kG = 0) lies below R5
// at kG = 1.  So the runs whose bound clears the staircase are a suffix in kG.
template <bool UNIT, bool NI>
__device__ __forceinline__ double lb_backward(const BlockConst& b, bool r1, double FH, double kG, double kA,
                                              const FGRow* FG) {
    const double CB = r1 ? b.C_B1 : b.C_B;
    const double BH = FH + kG * b.sGh + kA * (r1 ? b.sAh1 : b.sAh), BD = kG * b.sGd;
    if (kG == 0.0) return dmax(dmax(CB, b.N_B), dmax(BH, BD));
    return lb_row<UNIT, NI>(CB, b.N_B, BH, BD, FG);
}

template <bool UNIT, bool NI>
__device__ __forceinline__ double run_t_lb(const TupleConst& tc, const UnitState& us, double kG, double kA,
                                           const FGRow* FG) {
    double tb = 0.0;
    if (tc.nl0 > 0.0) tb += tc.nl0 * lb_backward<UNIT, NI>(tc.L, false, us.FH_L, kG, kA, FG);
    if (tc.nl1 > 0.0) tb += tc.nl1 * lb_backward<UNIT, NI>(tc.L, true, us.FH_L, kG, kA, FG);
    if (tc.first) tb += lb_backward<UNIT, NI>(tc.E, false, us.FH_E, kG, kA, FG);
    if (tc.last) tb += lb_backward<UNIT, NI>(tc.H, false, us.FH_H, kG, kA, FG);
    return (unit_tf(tc, us) + tb) + tc.t_p2p;
}

// R7 for a whole tuple (ykey = d): every channel is non-decreasing in the ratio
// indices (O6), so every config of the tuple has t >= sum count (R4(F at kW = kA =
// 0) + R4(B at kG = kW = kA = 0)) + p2p = sum count (max(C_F, N_F) + max(C_B, N_B))
// + p2p.  When the group's y = 0 staircase point lies strictly left of that, every
// unit of the tuple is beaten (same argument as run_cut) and none is set up.
__device__ __forceinline__ bool tuple_cut(const TupleConst& tc, const double* ft, const double* fy, long long lo,
                                          long long hi) {
    if (lo >= hi || !(fy[hi - 1] <= 0.0)) return false;
    double tb = 0.0;
    if (tc.nl0 > 0.0) tb += tc.nl0 * (dmax(tc.L.C_F, tc.L.N_F) + dmax(tc.L.C_B, tc.L.N_B));
    if (tc.nl1 > 0.0) tb += tc.nl1 * (dmax(tc.L.C_F, tc.L.N_F) + dmax(tc.L.C_B1, tc.L.N_B));
    if (tc.first) tb += dmax(tc.E.C_F, tc.E.N_F) + dmax(tc.E.C_B, tc.E.N_B);
    if (tc.last) tb += dmax(tc.H.C_F, tc.H.N_F) + dmax(tc.H.C_B, tc.H.N_B);
    return ft[hi - 1] < (tb + tc.t_p2p) * (1.0 - 1e-12);
}

// End of the runs of a unit that the pilot staircase cannot rule out: runs
// [g0, result) stay, runs [result, gend) are beaten.  A staircase point p with
// t_p < lb_t(kG) and y_p <= every y of the unit beats every config of runs >= kG
// (O10: strictly smaller t).  y lower bound: d >= 0 (L25), so for ykey = d only a
// y = 0 staircase point (the group's last, y falls along t) can cut; for ykey =
// mem the unit's smallest mem is its (kG, kO) = (kmax, kmax) config exactly (O9
// is non-increasing in kG and kO under the kG-suffix property, R2').  The t bound
// carries a 1e-12 relative margin for the rounding of R4/R5 against Alg. 1.
template <bool UNIT, bool NI = false>
__device__ MIST_CUT_ATTR unsigned run_cut(const DevProblem& P, const TupleConst& tc, const UnitState& us, unsigned kW, unsigned kA,
                            unsigned g0, unsigned gend, const FGRow* FG, const double* ft, const double* fy,
                            long long lo, long long hi, unsigned& nlb, const unsigned* vals = nullptr) {
    // vals (pilot sub-grid): runs are indices into vals[] (ascending kG values)
    if (lo >= hi) return gend;
    const double dkA = kA;
    double ymin = 0.0;                         // ykey = d: y >= 0
    if (P.ykey) {
        if (vals || !(tc.mG >= tc.gb_k)) return gend;   // mem not monotone in kG / sub-grid: no cut
        RunState rm;
        run_memory(tc, (double)kW, (double)(gend - 1), dkA, (double)P.Q, rm);
        ymin = mem_kO(tc, rm, (double)P.kmax[2], (double)P.Q) / tc.D;
    } else if (!(fy[hi - 1] <= 0.0)) {
        return gend;                           // no y = 0 point: nothing below every d
    }
    const unsigned nrows = (unsigned)(tc.nl0 > 0.0) + (unsigned)(tc.nl1 > 0.0) + (unsigned)(tc.first != 0) +
                           (unsigned)(tc.last != 0);
    auto cut = [&](unsigned g) -> bool {
        const unsigned kG = vals ? vals[g] : g;
        if (kG != 0u) nlb += nrows;            // R5 rows (kG = 0 takes the R4 max)
        const double lb = run_t_lb<UNIT, NI>(tc, us, (double)kG, dkA, FG) * (1.0 - 1e-12);
        if (!P.ykey) return ft[hi - 1] < lb;
        long long a = lo, b = hi;              // points with t < lb: [lo, a)
        while (a < b) {
            const long long m = (a + b) >> 1;
            if (ft[m] < lb) a = m + 1; else b = m;
        }
        return a > lo && fy[a - 1] <= ymin;    // the smallest y among them
    };
    if (cut(g0)) return g0;
    if (!cut(gend - 1)) return gend;
    unsigned a = g0, b = gend - 1;             // cut(a) false, cut(b) true
    while (b - a > 1) {
        const unsigned m = (a + b) >> 1;
        if (cut(m)) b = m; else a = m;
    }
    return b;
}

// Quick form of R7's unit cut before the unit's F rows exist: every config of the
// unit's runs kG >= g0 has t >= sum count (R4(F at kW, kA) + lb(B at g0)) + p2p, with
// R4(F) = the max of F's channels <= T(F) (factors >= 1).  True when the group's y = 0
// staircase point lies strictly left of that bound (then every run of the unit is
// beaten, O10); the exact cut with T(F) follows otherwise.
template <bool UNIT, bool NI>
__device__ __forceinline__ bool unit_quick_cut(const TupleConst& tc, double kW, double kA, double kG0,
                                               const FGRow* FG, const double* ft, const double* fy, long long lo,
                                               long long hi, unsigned& nlb) {
    if (lo >= hi || !(fy[hi - 1] <= 0.0)) return false;
    const double FHL = kW * tc.L.sWh;
    double lb = 0.0;
    unsigned rows = 0;
    if (tc.nl0 > 0.0) {
        lb += tc.nl0 * (dmax(dmax(tc.L.C_F, tc.L.N_F), dmax(FHL, kA * tc.L.sAd)) +
                        lb_backward<UNIT, NI>(tc.L, false, FHL, kG0, kA, FG));
        ++rows;
    }
    if (tc.nl1 > 0.0) {
        lb += tc.nl1 * (dmax(dmax(tc.L.C_F, tc.L.N_F), dmax(FHL, kA * tc.L.sAd1)) +
                        lb_backward<UNIT, NI>(tc.L, true, FHL, kG0, kA, FG));
        ++rows;
    }
    if (tc.first) {
        const double FHE = kW * tc.E.sWh;
        lb += dmax(dmax(tc.E.C_F, tc.E.N_F), dmax(FHE, kA * tc.E.sAd)) +
              lb_backward<UNIT, NI>(tc.E, false, FHE, kG0, kA, FG);
        ++rows;
    }
    if (tc.last) {
        const double FHH = kW * tc.H.sWh;
        lb += dmax(dmax(tc.H.C_F, tc.H.N_F), dmax(FHH, kA * tc.H.sAd)) +
              lb_backward<UNIT, NI>(tc.H, false, FHH, kG0, kA, FG);
        ++rows;
    }
    if (kG0 != 0.0) nlb += rows;
    return ft[hi - 1] < (lb + tc.t_p2p) * (1.0 - 1e-12);
}

// fill the {f, g} factor table (non-members: f = 1, g = 0)
__device__ __forceinline__ void load_fg(const DevProblem& P, FGRow* FG, int tid) {
    if (tid < 64) {
        const int pat = tid >> 2, j = tid & 3;
        const bool member = __popc(pat) >= 2 && ((pat >> j) & 1);
        FG[pat][j] = member ? make_double2(P.F[pat][j], P.IF[pat][j]) : make_double2(1.0, 0.0);
    }
}

__device__ __forceinline__ u64 splitmix64(u64 x) {
    u64 z = x + 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------
// a3-a8: eval kernel.  MODE 0 = frontier candidates, MODE 1 = dense outputs.
// ---------------------------------------------------------------------------

constexpr int kEvalThreads = 256;

// Instrumented build (-DMIST_COUNTERS): per-thread event counters of the frontier
// sweep, flushed to A.phases[1..5]: runs through run_backward, runs dropped at
// their first config by the bound, configs whose d was evaluated, k0 scan steps,
// runs cut before their backward rows (R7).
#ifdef MIST_COUNTERS
#define MIST_CTR(i, v) (ctr[i] += (v))
#else
#define MIST_CTR(i, v) ((void)0)
#endif

__device__ __forceinline__ void flush_ctr(const EvalArgs& A, const unsigned* ctr, unsigned lane) {
#ifdef MIST_COUNTERS
    if (!A.phases) return;
    for (int i = 0; i < 5; ++i) {
        unsigned v = ctr[i];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && v) atomicAdd(A.phases + 1 + i, (u64)v);
    }
#endif
}

// O10 "p beats q" on (x, y, idx)
__device__ __forceinline__ bool beats(double tp, double yp, u64 ip, double tq, double yq, u64 iq) {
    return tp <= tq && yp <= yq && (tp < tq || yp < yq || ip < iq);
}

// a8: warp-ballot stream compaction, one atomic per warp, coalesced SoA stores
__device__ __forceinline__ void warp_emit(bool emit, double t, double y, double mem, u64 idx, unsigned grp,
                                          const EvalArgs& A, unsigned lane) {
    const unsigned ball = __ballot_sync(0xffffffffu, emit);
    if (!ball) return;
    u64 wbase = 0;
    if (lane == 0) wbase = atomicAdd(A.cand_count, (u64)__popc(ball));
    wbase = __shfl_sync(0xffffffffu, wbase, 0);
    if (emit) {
        const u64 pos = wbase + __popc(ball & ((1u << lane) - 1));
        if ((long long)pos < A.cand.cap) {
            A.cand.t[pos] = t;
            A.cand.y[pos] = y;
            A.cand.mem[pos] = mem;
            A.cand.idx[pos] = idx;
            A.cand.group[pos] = grp;
        }
    }
}

// Frontier-mode evaluation of one OO-run (tuple, kW, kG, kA): returns the run's
// candidate = min (d or mem, idx) over its feasible configs, or none.  The
// staircase filter (pilot frontier) is applied; (cv, ct, cy) is the caller's
// cached candidate, a known feasible point of the same group.
struct RunCand {
    bool has;
    double t, y, m;
    u64 idx;
};

// The pilot staircase as seen by one CTA: global arrays, or a shared-memory copy
// of the CTA's groups addressed with the global positions (pointers shifted).
struct FiltView {
    const double* t;
    const double* y;
    const u64* idx;
    const int64_t* off;     // null: no filter
};

template <bool UNIT, int MODE, bool NI = false>
__device__ __forceinline__ RunCand frontier_run(const DevProblem& P, const EvalArgs& A, const TupleConst& tc,
                                                const UnitState& us, unsigned kW, unsigned kG, unsigned kA,
                                                unsigned radix, double Q, int Q1, unsigned grp, const FGRow* FG,
                                                bool cv, double ct, double cy, unsigned nrows, unsigned brows,
                                                unsigned& nph, unsigned& nlb, u64& fcnt, u64& fhash,
                                                const FiltView& fv,
                                                unsigned* ctr) {
    // the staircase filter runs in the frontier sweep and in the pilot (both exact, O10)
    constexpr bool FILT = MODE == 0 || MODE == 2;
    const double dkW = kW, dkG = kG, dkA = kA;
    RunState rs;
    run_memory(tc, dkW, dkG, dkA, Q, rs);
    rs.t = 0.0;
    const long long f_lo = (FILT && fv.off) ? fv.off[grp] : 0;
    long long f_at = f_lo - 1;              // staircase point used by the filter (none if < f_lo)
    const u64 idx0 = tc.idx_base + ((u64)(kW * Q1 + kG) * Q1) * Q1 + kA;
    bool has = false;
    double best_y = CUDART_INF, best_m = 0.0;
    u64 best_i = 0;
    // preset: kO ranges over [0, kmax[2]] (pilot: the sub-grid values within it)
    const unsigned kend = (MODE == 2) ? (P.kmax[2] == P.Q ? radix : 1u) : (unsigned)P.kmax[2] + 1u;
    const double kOend = (MODE == 2) ? (double)A.vals[kend - 1] : (double)(kend - 1);
    if (mem_kO(tc, rs, kOend, Q) <= tc.DMB) {
        // D*mem is non-increasing in kO (O9: P_raw >= min(l,2) P_layer), so the
        // feasible configs of a run are a suffix in kO and a run whose kO = Q
        // config is over budget has none: its t and d are never needed (R2).
#ifdef MIST_DEFER_BP
        run_backward<UNIT, true>(tc, us, dkW, dkG, dkA, FG, rs);
        nph += nrows;
        if (!rs.dexact) nlb += brows - nrows;
#else
        run_backward<UNIT>(tc, us, dkW, dkG, dkA, FG, rs);
        nph += brows;
#endif
        MIST_CTR(0, 1);
        // Bound-and-skip (ykey = d): a config whose lower bound of d exceeds the
        // best d the run already has, or the y of a known feasible point with
        // t <= the run's t (pilot staircase / cached candidate, both with a
        // smaller-or-unrelated idx, so equal y is not needed), cannot be the run's
        // frontier candidate.  The bound is non-decreasing in kO (R4).
        // the staircase point with the largest t <= the run's t (one binary search, reused below)
        if (FILT && fv.off) {
            long long lo = f_lo, hi = fv.off[grp + 1];
            while (lo < hi) {                       // first position with f_t > t
                const long long mid = (lo + hi) >> 1;
                if (fv.t[mid] <= rs.t) lo = mid + 1; else hi = mid;
            }
            f_at = lo - 1;
        }
        double y_thr = CUDART_INF;
        if (FILT && !P.ykey) {
            if (cv && ct <= rs.t) y_thr = cy;
            if (f_at >= f_lo) {
                const double yf = fv.y[f_at];
                y_thr = yf < y_thr ? yf : y_thr;
            }
        }
        // First feasible config of the run: the feasible configs are a suffix in kO
        // (R2).  Starting every lane's evaluation loop there keeps the warp's F'
        // evaluations of kO_min in lockstep instead of serialising them.
        unsigned k0 = 0;
        if (MODE == 2) {
            while (k0 + 1 < kend && !(mem_kO(tc, rs, (double)A.vals[k0], Q) <= tc.DMB)) {
                ++k0;
                MIST_CTR(3, 1);
            }
        } else {
            k0 = first_feasible_kO(tc, rs, Q);
        }
        if (MODE == 0 && A.fp)
            for (unsigned k = k0; k < kend; ++k) {
                const u64 idx = idx0 + (u64)k * Q1;
                if (mem_kO(tc, rs, (double)k, Q) <= tc.DMB) { fcnt++; fhash += splitmix64(idx); }
            }
        for (unsigned k = k0; k < kend; ++k) {
            const unsigned ko = (MODE == 2) ? A.vals[k] : k;
            const double kO = ko;
            const double memD = mem_kO(tc, rs, kO, Q);
            if (!(memD <= tc.DMB)) continue;                 // Eq. 4 constraint, exact
            const u64 idx = idx0 + (u64)ko * Q1;
            if (FILT && !P.ykey) {
                double scale;
                double lb = d_lower_bound<UNIT, NI>(tc, us, rs, kO, FG, scale);
                nlb += nrows;
                const double thr = best_y < y_thr ? best_y : y_thr;
                bool over = lb - 1e-12 * (scale + rs.dsc) > thr;
                if (!over && !rs.dexact) {
                    // the lower-bound dbase did not cut: the exact B' rows, then the same test
                    rs.dbase = run_dbase_exact<UNIT>(tc, us, dkG, dkA, FG);
                    rs.dexact = true;
                    rs.dsc = 0.0;
                    nph += brows;
                    lb = d_lower_bound<UNIT, NI>(tc, us, rs, kO, FG, scale);
                    nlb += nrows;
                    over = lb - 1e-12 * scale > thr;
                }
                if (over) {
                    if (A.fp) continue;                       // keep counting feasible configs
                    // the bound is non-decreasing in kO while the F' nonzero pattern is fixed,
                    // which holds for kO >= 1 (H2D and D2H grow with kO); at kO = 0 a zero
                    // H2D or D2H channel switches the R5 factor row, so only skip that config
                    if (!UNIT && ko == 0 && !fp_pattern_fixed(tc, rs)) continue;
                    MIST_CTR(1, k == k0 ? 1u : 0u);
                    break;
                }
            }
            // P13: the whole run shares t; keep its min (y, idx)
            if (!P.ykey) nph += nrows;
            MIST_CTR(2, 1);
            const double y = P.ykey ? memD / tc.D : d_kO<UNIT>(tc, us, rs, kO, FG);
            if (y < best_y) { best_y = y; best_i = idx; best_m = memD; has = true; }
        }
    }
    if (FILT && has && f_at >= f_lo) {
        // staircase filter: the pilot frontier point with the largest t <= rt has the
        // smallest y among all pilot points with t <= rt; if it beats the run's best,
        // drop it (exact: it is a real feasible config of the same group, O10)
        if (beats(fv.t[f_at], fv.y[f_at], fv.idx[f_at], rs.t, best_y, best_i)) has = false;
    }
    RunCand r;
    r.has = has; r.t = rs.t; r.y = best_y; r.m = best_m; r.idx = best_i;
    return r;
}

// One thread per unit = (tuple, kW, kA); it loops over kG (runs) and kO
// (configs).  Units of one tuple are padded to a multiple of 32 when there are
// >= 64 of them, so that a warp never straddles two tuples (the phase
// structure -- c, z, first/last -- is then warp-uniform).  The thread keeps one
// cached candidate and emits it only when a later run's candidate is
// incomparable with it; a point beaten by another feasible config of the same
// group is dropped, which is exact (O10).  MODE 2 (pilot) walks the sub-grid
// vals[0..nv) on every ratio axis.
template <bool UNIT, int MODE, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB)
k_eval(DevProblem P, EvalArgs A) {
    extern __shared__ double smem[];
    FGRow* FG = reinterpret_cast<FGRow*>(smem);                    // 16 x 4 x {f, g}
    TupleConst* sT = reinterpret_cast<TupleConst*>(smem + 128);
    const int tid = threadIdx.x;
    load_fg(P, FG, tid);
    const double Q = P.Q;
    const int Q1 = P.Q1;
    const unsigned lane = tid & 31;
    const unsigned radix = (MODE == 2) ? A.nv : (unsigned)Q1;
    const unsigned upt = A.upt;                       // units per tuple (>= radix^2)
    const u64 n_units = A.n_units;
    for (u64 base = (u64)blockIdx.x * NT; base < n_units;
         base += (u64)gridDim.x * NT) {
        const u64 last_unit = min(base + NT, n_units) - 1;
        const u64 tb0 = base / upt, tb1 = last_unit / upt;
        const int ntl = (int)(tb1 - tb0 + 1);
        __syncthreads();   // previous iteration done with sT
        {
            const double* src = reinterpret_cast<const double*>(A.tuples + tb0);
            double* dst = reinterpret_cast<double*>(sT);
            const int nw = ntl * (int)(sizeof(TupleConst) / 8);
            for (int i = tid; i < nw; i += NT) dst[i] = __ldg(src + i);
        }
        __syncthreads();
        const u64 u = base + tid;
        const unsigned tk = u < n_units ? (unsigned)(u / upt - tb0) : 0u;
        const unsigned jj = (unsigned)(u - (tb0 + tk) * (u64)upt);
        const bool unit_ok = u < n_units && jj < radix * radix;
        const unsigned iW = jj / radix, iA = jj - iW * radix;
        const unsigned kW = (MODE == 2) ? A.vals[unit_ok ? iW : 0] : iW;
        const unsigned kA = (MODE == 2) ? A.vals[unit_ok ? iA : 0] : iA;
        // preset: a unit with kW or kA beyond its ratio's range has no configuration in
        // the space (the dense mode still writes t, d, mem for it, with feasible = 0)
        const bool in_unit = kW <= (unsigned)P.kmax[0] && kA <= (unsigned)P.kmax[3];
        const bool twin = MODE != 1 && unit_ok && sT[tk].twin_T != ~0ull && sT[tk].twin_T >= A.twin_floor;
        const bool in_pass = MODE != 0 || !A.unit_pass || ((A.unit_pass == 1) == (!(kW & 1u) && !(kA & 1u)));
        // tuple-level R7 (ykey = d) in the frontier and pilot modes
        const bool tcut = MODE != 1 && unit_ok && !P.ykey && A.f_off && !A.fp && !(A.no_r7 & 3) &&
                          tuple_cut(sT[tk], A.f_t, A.f_y, A.f_off[sT[tk].group], A.f_off[sT[tk].group + 1]);
        const bool active = unit_ok && (MODE == 1 || in_unit) && !twin && in_pass && !tcut;
        const double dkW = kW, dkA = kA;
        const TupleConst& tc = sT[tk];
        const unsigned grp = tc.group;
        UnitState us;
        if (active) unit_forward<UNIT>(tc, dkW, dkA, FG, us);
        // R7 (frontier and pilot modes): runs ig >= icut are beaten by the staircase on t alone
        unsigned icut = radix;
        unsigned nlb = 0;                      // R5 bound rows evaluated (roofline count)
        if (MODE != 1 && active && A.f_off && !A.fp && !(A.no_r7 & 1))
            icut = run_cut<UNIT>(P, tc, us, kW, kA, 0u, radix, FG, A.f_t, A.f_y, A.f_off[grp], A.f_off[grp + 1],
                                 nlb, MODE == 2 ? A.vals : nullptr);
        // phase rows evaluated by this thread (PredINTF calls), for the roofline's algorithmic count
        const unsigned nrows = (unsigned)(tc.nl0 > 0.0) + (unsigned)(tc.nl1 > 0.0) + (unsigned)(tc.first != 0) +
                               (unsigned)(tc.last != 0);
        const unsigned brows = nrows * (tc.L.N_Bp != tc.L.N_B ? 2u : 1u);
        unsigned nph = active ? nrows : 0u;
        unsigned ctr[5] = {0u, 0u, 0u, 0u, 0u};
        bool cv = false;                       // cached candidate
        double ct = 0.0, cy = 0.0, cm = 0.0;
        u64 ci = 0;
        u64 fcnt = 0, fhash = 0;
        for (unsigned ig = 0; ig < radix; ++ig) {
            bool emit = false;
            double et = 0.0, ey = 0.0, em = 0.0;
            u64 ei = 0;
            const unsigned kG = (MODE == 2) ? A.vals[ig] : ig;
            if (active && ig < icut && (MODE == 1 || kG <= (unsigned)P.kmax[1])) {
                const double dkG = kG;
                RunState rs;
                run_memory(tc, dkW, dkG, dkA, Q, rs);
                const u64 idx0 = tc.idx_base + ((u64)(kW * Q1 + kG) * Q1) * Q1 + kA;
                bool has = false;
                double best_y = CUDART_INF, best_m = 0.0;
                u64 best_i = 0;
                if (MODE == 1) {
                    run_backward<UNIT>(tc, us, dkW, dkG, dkA, FG, rs);
                    double kO = 0.0;
                    for (int k = 0; k < Q1; ++k, kO += 1.0) {
                        const u64 idx = idx0 + (u64)k * Q1;
                        if (idx < A.lo || idx >= A.hi) continue;
                        const double memD = mem_kO(tc, rs, kO, Q);
                        const u64 o = idx - A.lo;
                        if (A.t) A.t[o] = rs.t;
                        if (A.d) A.d[o] = d_kO<UNIT>(tc, us, rs, kO, FG);
                        if (A.mem) A.mem[o] = memD / tc.D;
                        if (A.feas)
                            A.feas[o] = memD <= tc.DMB && in_unit && kG <= (unsigned)P.kmax[1] &&
                                        k <= P.kmax[2];
                    }
                } else {
                    FiltView fv;
                    fv.t = A.f_t; fv.y = A.f_y; fv.idx = A.f_idx; fv.off = A.f_off;
                    const RunCand rc = frontier_run<UNIT, MODE>(P, A, tc, us, kW, kG, kA, radix, Q, Q1, grp, FG, cv,
                                                                ct, cy, nrows, brows, nph, nlb, fcnt, fhash, fv, ctr);
                    has = rc.has; best_y = rc.y; best_i = rc.idx; best_m = rc.m; rs.t = rc.t;
                }
                if (MODE != 1 && has) {
                    const double rt = rs.t, rm = best_m / tc.D;
                    if (!cv) {
                        cv = true; ct = rt; cy = best_y; cm = rm; ci = best_i;
                    } else if (beats(ct, cy, ci, rt, best_y, best_i)) {
                        // new run's best is beaten by the cached point: drop it
                    } else {
                        if (!beats(rt, best_y, best_i, ct, cy, ci)) {   // incomparable: emit the cached one
                            emit = true; et = ct; ey = cy; em = cm; ei = ci;
                        }
                        ct = rt; cy = best_y; cm = rm; ci = best_i;
                    }
                }
            }
            if (MODE != 1) warp_emit(emit, et, ey, em, ei, grp, A, lane);
        }
        if (MODE != 1) {
            warp_emit(cv, ct, cy, cm, ci, grp, A, lane);
            if (A.phases) {                                   // warp-reduced phase-row counts
                unsigned v = nph, b = nlb;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    v += __shfl_xor_sync(0xffffffffu, v, o);
                    b += __shfl_xor_sync(0xffffffffu, b, o);
                }
                if (lane == 0 && v) atomicAdd(A.phases, (u64)v);
                if (lane == 0 && b) atomicAdd(A.phases + 6, (u64)b);
            }
            flush_ctr(A, ctr, lane);
            if (A.fp) {
                // feasible-set fingerprint, warp-aggregated per group
                const bool any = fcnt > 0;
                const unsigned am = __ballot_sync(0xffffffffu, any);
                if (any) {
                    const unsigned peers = __match_any_sync(am, grp);
                    const int leader = __ffs(peers) - 1;
                    u64 c = fcnt, hsh = fhash;
                    // sum over peers via shuffles restricted to the peer set
                    for (unsigned m = peers & ~(1u << leader); m; m &= m - 1) {
                        const int src = __ffs(m) - 1;
                        const u64 oc = __shfl_sync(peers, fcnt, src);
                        const u64 oh = __shfl_sync(peers, fhash, src);
                        if ((int)lane == leader) { c += oc; hsh += oh; }
                    }
                    if ((int)lane == leader) {
                        atomicAdd(A.fp + 2 * (u64)grp, c);
                        atomicAdd(A.fp + 2 * (u64)grp + 1, hsh);
                    }
                }
            }
        }
    }
}

// Frontier mode with a warp-level run queue.  Every lane first finds its
// unit's first run (kG) whose kO = Q config fits the budget; with D*mem
// non-increasing in kG (mG >= gb_k, true for 2-byte gradients) the feasible
// runs of a unit are a suffix in kG (R2').  The warp then deals the feasible
// runs of its 32 units round-robin to its lanes (owner found by binary lifting
// over the warp prefix sum, unit state fetched with shuffles), so no lane idles
// on an infeasible run while another works.
// CQ = true: the queue spans the whole CTA instead of one warp -- the feasible runs
// of all NT units are numbered by a block-wide prefix sum and warps take batches
// of 32 from a shared-memory counter, so every warp of the CTA finishes the
// window at about the same time (less time waiting at the window barrier).
// UPW (CTA queue only): units per thread per window; a window of NT*UPW units
// halves the window boundaries (and their barrier tails) for UPW = 2.
template <bool UNIT, int NT, int MINB, bool CQ, int UPW, bool NI = false, int MODE = 0>
__global__ void __launch_bounds__(NT, MINB)
k_eval_q(DevProblem P, EvalArgs A) {
    static_assert(MODE == 0 || (MODE == 2 && CQ), "the pilot sub-grid (MODE 2) runs on the CTA queue");
    static_assert(CQ || UPW == 1, "several units per thread need the CTA queue");
    constexpr int NW = NT * UPW;                                     // units per window
    static_assert(sizeof(TupleConst) % 16 == 0, "bulk copies move whole tuples in 16-byte units");
    extern __shared__ __align__(128) double smem[];
    FGRow* FG = reinterpret_cast<FGRow*>(smem);
    const int maxt = (NW + (int)A.upt - 1) / (int)A.upt + 1;        // tuples one window touches
    TupleConst* sTbuf = reinterpret_cast<TupleConst*>(smem + 128);  // CQ: two stages of maxt tuples
    TupleConst* sT = sTbuf;
    // per-unit forward state of the CTA's NT units (read by whichever lane runs a run of the unit)
    UnitState* sU = reinterpret_cast<UnitState*>(sTbuf + (CQ ? 2 : 1) * maxt);
    unsigned* s_excl = reinterpret_cast<unsigned*>(sU + NW);     // CQ: exclusive run-count prefix per unit
    unsigned* s_g0 = s_excl + NW;                                 // CQ: first run (kG) per unit
    unsigned* s_uinfo = s_g0 + NW;                                // CQ: tk | kW << 10 | kA << 21
    unsigned* s_wt = s_uinfo + NW;                                // CQ: warp totals [NT/32]
    unsigned* s_ctr = s_wt + NT / 32;                             // CQ: batch counter
    u64* s_bar = reinterpret_cast<u64*>(s_ctr + 2);               // CQ: tuple-stage mbarriers [2]
    unsigned short* s_map = reinterpret_cast<unsigned short*>(s_bar + 2);   // CQ: run -> unit [NT * Q1]
    const int tid = threadIdx.x;
    load_fg(P, FG, tid);
    const double Q = P.Q;
    const int Q1 = P.Q1;
    const unsigned lane = tid & 31;
    UnitState* wU = sU + (tid & ~31);
    // MODE 2 (pilot): ratio indices address the sub-grid values vals[0..nv) on every axis
    const unsigned radix = MODE == 2 ? A.nv : (unsigned)Q1;
    auto val = [&](unsigned i) -> unsigned { return MODE == 2 ? A.vals[i] : i; };
    const unsigned upt = A.upt;
    const u64 n_units = A.n_units;
    unsigned nph = 0, nlb = 0;
    unsigned ctr[5] = {0u, 0u, 0u, 0u, 0u};
    // CQ: the window's tuples arrive by one TMA bulk copy, issued one window ahead
    auto tuples_of = [&](u64 b, u64& t0, int& nt) {
        const u64 lu = min(b + NW, n_units) - 1;
        t0 = b / upt;
        nt = (int)(lu / upt - t0 + 1);
    };
    auto issue_tuples = [&](u64 b, int stg) {
        u64 t0;
        int nt;
        tuples_of(b, t0, nt);
        const unsigned bytes = (unsigned)(nt * sizeof(TupleConst));
        const unsigned bar = (unsigned)__cvta_generic_to_shared(&s_bar[stg]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" :: "r"(bar), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     :: "r"((unsigned)__cvta_generic_to_shared(sTbuf + stg * maxt)), "l"(A.tuples + t0), "r"(bytes),
                        "r"(bar) : "memory");
    };
    if (CQ) {
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"((unsigned)__cvta_generic_to_shared(&s_bar[0])) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"((unsigned)__cvta_generic_to_shared(&s_bar[1])) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            if ((u64)blockIdx.x * NW < n_units) issue_tuples((u64)blockIdx.x * NW, 0);
        }
    }
    int it = 0;
    for (u64 base = (u64)blockIdx.x * NW; base < n_units; base += (u64)gridDim.x * NW, ++it) {
        u64 tb0;
        int ntl;
        tuples_of(base, tb0, ntl);
        __syncthreads();
        if (CQ) {
            const int stg = it & 1;
            sT = sTbuf + stg * maxt;
            const u64 nb = base + (u64)gridDim.x * NW;
            if (tid == 0 && nb < n_units) {          // the other stage was last read before this barrier
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                issue_tuples(nb, stg ^ 1);
            }
            const unsigned bar = (unsigned)__cvta_generic_to_shared(&s_bar[stg]);
            const unsigned par = (unsigned)(it >> 1) & 1u;
            asm volatile("{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
                         " @!P bra WAIT_%=;\n}\n" :: "r"(bar), "r"(par) : "memory");
        } else {
            const double* src = reinterpret_cast<const double*>(A.tuples + tb0);
            double* dst = reinterpret_cast<double*>(sT);
            const int nw = ntl * (int)(sizeof(TupleConst) / 8);
            for (int i = tid; i < nw; i += NT) dst[i] = __ldg(src + i);
            __syncthreads();
        }
        FiltView fv;
        fv.t = A.f_t; fv.y = A.f_y; fv.idx = A.f_idx; fv.off = A.f_off;
        const bool r7 = fv.off != nullptr && A.fp == nullptr && !(A.no_r7 & 1);
        unsigned total = 0;
        // per-thread state of unit j = 0 (the warp queue of the non-CQ path reads it)
        unsigned tk = 0, kW = 0, kA = 0, g0 = radix, excl = 0;
        // 32-bit unit decode: base sits r0 units into tuple tb0, so unit w of the window is
        // unit (r0 + w) mod upt of tuple tb0 + (r0 + w) / upt; both divisions by a float
        // reciprocal with a one-step correction (exact for these small operands)
        const unsigned r0 = (unsigned)(base - tb0 * (u64)upt);
        const float inv_upt = 1.0f / (float)upt, inv_rad = 1.0f / (float)radix;
#pragma unroll
        for (int j = 0; j < UPW; ++j) {
            const unsigned w = (unsigned)(j * NT + tid);                   // unit of the window
            const u64 u = base + w;
            const unsigned off = r0 + w;
            unsigned tq = (unsigned)((float)off * inv_upt);
            tq -= tq * upt > off ? 1u : 0u;
            tq += (tq + 1u) * upt <= off ? 1u : 0u;
            const unsigned tkj = u < n_units ? tq : 0u;
            const unsigned jj = off - tq * upt;
            unsigned kWj = (unsigned)((float)jj * inv_rad);
            kWj -= kWj * radix > jj ? 1u : 0u;
            kWj += (kWj + 1u) * radix <= jj ? 1u : 0u;
            const unsigned iAj = jj - kWj * radix;
            kWj = val(jj < radix * radix ? kWj : 0u);               // ratio values (MODE 2: sub-grid)
            const unsigned kAj = val(jj < radix * radix ? iAj : 0u);
            bool active = u < n_units && jj < radix * radix && kWj <= (unsigned)P.kmax[0] &&
                          kAj <= (unsigned)P.kmax[3];                    // preset ranges
            if (active && sT[tkj].twin_T >= A.twin_floor && sT[tkj].twin_T != ~0ull) active = false;   // L20 twin
            if (A.unit_pass && ((A.unit_pass == 1) != (!(kWj & 1u) && !(kAj & 1u)))) active = false;
            if (active && r7 && !P.ykey && !(A.no_r7 & 2) && tuple_cut(sT[tkj], fv.t, fv.y, fv.off[sT[tkj].group],
                                                     fv.off[sT[tkj].group + 1])) {
                active = false;
                MIST_CTR(4, (unsigned)P.kmax[1] + 1u);
            }
            // runs: kG indices [0, gend) (MODE 2: the sub-grid values within the preset range)
            unsigned gend = (unsigned)P.kmax[1] + 1u;
            if (MODE == 2) {
                gend = 0;
                while (gend < radix && A.vals[gend] <= (unsigned)P.kmax[1]) ++gend;
            }
            unsigned g0j = radix, g1j = gend;
            {
                const TupleConst& tc = sT[tkj];
                if (active) {
                    if (MODE == 2) {
                        // sub-grid: scan its few kG values at the last admitted kO value
                        const double kOv = (double)A.vals[(P.kmax[2] == P.Q ? radix : 1u) - 1u];
                        RunState rm;
                        for (unsigned ig = 0; ig < gend; ++ig) {
                            run_memory(tc, (double)kWj, (double)A.vals[ig], (double)kAj, Q, rm);
                            if (mem_kO(tc, rm, kOv, Q) <= tc.DMB) { g0j = ig; break; }
                        }
                        if (!(tc.mG >= tc.gb_k)) g0j = 0;
                    } else if (tc.mG >= tc.gb_k) {
#ifdef MIST_G0_SCAN
                        RunState rm;
                        for (unsigned ig = 0; ig < gend; ++ig) {
                            run_memory(tc, (double)kWj, (double)ig, (double)kAj, Q, rm);
                            if (mem_kO(tc, rm, (double)P.kmax[2], Q) <= tc.DMB) { g0j = ig; break; }
                        }
#else
                        const unsigned f = first_feasible_kG(tc, (double)kWj, (double)kAj, gend,
                                                             (double)P.kmax[2], Q);
                        g0j = f < gend ? f : radix;
#endif
                    } else {
                        g0j = 0;                       // no kG-suffix property: every run is a task
                    }
                    // A unit without a feasible run, or whose first run a cheap bound (R4 rows of
                    // F in place of the exact ones, R7) already puts past the y = 0 staircase
                    // point, needs no F rows at all.  The cheap bound pays on the long kO axes
                    // only (same-box A/B: cfg3 Q = 20 and cfg5 Q = 50 1-2% faster, cfg2 Q = 10
                    // and cfg4 Q = 8 1-2% slower, profiles/r2/ab_quick_cut_summary.txt).
                    if (g0j < gend && r7 && !P.ykey && P.Q >= 16 &&
                        unit_quick_cut<UNIT, NI>(tc, (double)kWj, (double)kAj,
                                                 (double)(MODE == 2 ? A.vals[g0j] : g0j), FG, fv.t, fv.y,
                                                 fv.off[tc.group], fv.off[tc.group + 1], nlb)) {
                        g1j = g0j;
                        MIST_CTR(4, gend - g0j);
                    }
                    if (g0j < g1j) {
                        UnitState us;
                        unit_forward<UNIT>(tc, (double)kWj, (double)kAj, FG, us);
                        sU[w] = us;
                        nph += (unsigned)(tc.nl0 > 0.0) + (unsigned)(tc.nl1 > 0.0) + (unsigned)(tc.first != 0) +
                               (unsigned)(tc.last != 0);
                        // R7: runs the staircase beats on t alone are never dealt (not with
                        // fingerprints, which count every feasible config)
                        if (r7) {
                            g1j = run_cut<UNIT, NI>(P, tc, us, kWj, kAj, g0j, gend, FG, fv.t, fv.y,
                                                    fv.off[tc.group], fv.off[tc.group + 1], nlb,
                                                    MODE == 2 ? A.vals : nullptr);
                            MIST_CTR(4, gend - g1j);
                        }
                    }
                }
            }
            __syncwarp();
            const unsigned cnt = (active && g0j < g1j) ? g1j - g0j : 0u;
            unsigned incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
                if ((int)lane >= o) incl += v;
            }
            unsigned exj = incl - cnt;
            unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
            if (CQ) {   // block-wide numbering of the runs, after the window's units of earlier j
                if (j > 0) __syncthreads();              // s_wt of the previous j has been read
                if (lane == 31) s_wt[tid >> 5] = incl;
                if (tid == 0 && j == 0) *s_ctr = 0u;
                __syncthreads();
                unsigned before = 0, all = 0;
#pragma unroll
                for (int wq = 0; wq < NT / 32; ++wq) {
                    const unsigned x = s_wt[wq];
                    before += wq < (tid >> 5) ? x : 0u;
                    all += x;
                }
                incl += total + before;
                exj += total + before;
                tot = total + all;
                s_excl[w] = exj;
                s_g0[w] = g0j;
                s_uinfo[w] = tkj | (kWj << 10) | (kAj << 21);
                for (unsigned k = exj; k < incl; ++k) s_map[k] = (unsigned short)w;   // run -> unit
            }
            total = tot;
            if (j == 0) { tk = tkj; kW = kWj; kA = kAj; g0 = g0j; excl = exj; }
        }
        if (CQ) __syncthreads();
#ifdef MIST_DIAG_SETUP_ONLY
        total = 0;                              // diagnostic build: window setup only, no runs
#endif
        bool cv = false;                        // cached candidate (any group; emitted on group change)
        double ct = 0.0, cy = 0.0, cm = 0.0;
        u64 ci = 0;
        unsigned cgrp = 0;
        for (unsigned rb = 0;; rb += 32) {
            if (CQ) {
                unsigned b = 0;
                if (lane == 0) b = atomicAdd(s_ctr, 32u);
                rb = __shfl_sync(0xffffffffu, b, 0);
            }
            if (rb >= total) break;
            const unsigned r = rb + lane;
            unsigned o_tk, o_kW, o_kA, o_g0, o_ex;
            const UnitState* oup;
            if (CQ) {
                const unsigned own = r < total ? s_map[r] : 0u;
                o_ex = s_excl[own];
                o_g0 = s_g0[own];
                const unsigned ui = s_uinfo[own];
                o_tk = ui & 1023u;
                o_kW = (ui >> 10) & 2047u;
                o_kA = ui >> 21;
                oup = sU + own;
            } else {
                unsigned own = 0;                   // largest lane whose excl <= r
#pragma unroll
                for (int s2 = 16; s2 > 0; s2 >>= 1) {
                    const unsigned cand = own + s2;
                    const unsigned e = __shfl_sync(0xffffffffu, excl, cand & 31);
                    if (cand < 32 && e <= r) own = cand;
                }
                o_tk = __shfl_sync(0xffffffffu, tk, own);
                o_kW = __shfl_sync(0xffffffffu, kW, own);
                o_kA = __shfl_sync(0xffffffffu, kA, own);
                o_g0 = __shfl_sync(0xffffffffu, g0, own);
                o_ex = __shfl_sync(0xffffffffu, excl, own);
                oup = wU + own;
            }
            const UnitState& ou = *oup;
            bool emit = false;
            double et = 0.0, ey = 0.0, em = 0.0;
            u64 ei = 0;
            unsigned egrp = 0;
            if (r < total) {
                const TupleConst& tc = sT[o_tk];
                const unsigned grp = tc.group;
                const unsigned kG = val(o_g0 + (r - o_ex));
                const unsigned nrows = (unsigned)(tc.nl0 > 0.0) + (unsigned)(tc.nl1 > 0.0) +
                                       (unsigned)(tc.first != 0) + (unsigned)(tc.last != 0);
                const unsigned brows = nrows * (tc.L.N_Bp != tc.L.N_B ? 2u : 1u);
                const bool same = cv && cgrp == grp;
                u64 fcnt = 0, fhash = 0;
                const RunCand rc = frontier_run<UNIT, MODE, NI>(P, A, tc, ou, o_kW, kG, o_kA, radix, Q, Q1, grp, FG, same,
                                                         ct, cy, nrows, brows, nph, nlb, fcnt, fhash, fv, ctr);
                if (A.fp && fcnt) {
                    atomicAdd(A.fp + 2 * (u64)grp, fcnt);
                    atomicAdd(A.fp + 2 * (u64)grp + 1, fhash);
                }
                if (rc.has) {
                    const double rm = rc.m / tc.D;
                    if (!cv) {
                        cv = true; ct = rc.t; cy = rc.y; cm = rm; ci = rc.idx; cgrp = grp;
                    } else if (same && beats(ct, cy, ci, rc.t, rc.y, rc.idx)) {
                        // the new run's best is beaten by the cached point: drop it
                    } else {
                        if (!same || !beats(rc.t, rc.y, rc.idx, ct, cy, ci)) {   // incomparable: emit the cached one
                            emit = true; et = ct; ey = cy; em = cm; ei = ci; egrp = cgrp;
                        }
                        ct = rc.t; cy = rc.y; cm = rm; ci = rc.idx; cgrp = grp;
                    }
                }
            }
            warp_emit(emit, et, ey, em, ei, egrp, A, lane);
        }
        warp_emit(cv, ct, cy, cm, ci, cgrp, A, lane);
    }
    if (A.phases) {
        unsigned v = nph, b = nlb;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            v += __shfl_xor_sync(0xffffffffu, v, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
        }
        if (lane == 0 && v) atomicAdd(A.phases, (u64)v);
        if (lane == 0 && b) atomicAdd(A.phases + 6, (u64)b);
    }    flush_ctr(A, ctr, lane);
}

// Zero-offload pilot (ykey = d; feeds R7).  A config can have d = 0 only without
// first-microbatch extras: WO = GO = OO = 0 (O6's F' adds OO, GO and WO traffic)
// and no last-microbatch collective or post-update gather (z = 3 or DP = 1).
// The sub-grid pilot samples AO at a few values only, so its y = 0 point can sit
// well right of the group's true one.  One thread per tuple walks every admitted
// kA of (kW, kG, kO) = (0, 0, 0), keeps the feasible config of least (t, idx)
// with d = 0, and the warp emits one candidate per group (leader of the group's
// lanes).  The candidates are real feasible configs, so any point they beat is
// beaten (O10): the staircase they join stays exact.
template <bool UNIT>
__global__ void __launch_bounds__(64)
k_pilot_zero(DevProblem P, EvalArgs A) {
    constexpr int NT = 64;                                  // launched with NT threads
    __shared__ FGRow FG[16];
    __shared__ __align__(16) TupleConst sT[NT];             // the CTA's tuples, loaded coalesced
    load_fg(P, FG, threadIdx.x);
    const double Q = P.Q;
    const unsigned lane = threadIdx.x & 31;
    const u64 nT = A.n_units;
    for (u64 base = (u64)blockIdx.x * NT; base < nT; base += (u64)gridDim.x * NT) {
        __syncthreads();                                    // previous window done with sT
        {
            const int nt = (int)min((u64)NT, nT - base);
            const double* src = reinterpret_cast<const double*>(A.tuples + base);
            double* dst = reinterpret_cast<double*>(sT);
            const int nw = nt * (int)(sizeof(TupleConst) / 8);
            for (int i = threadIdx.x; i < nw; i += NT) dst[i] = __ldg(src + i);
        }
        __syncthreads();
        const u64 T = base + threadIdx.x;
        bool has = false;
        double bt = CUDART_INF, bm = 0.0;
        u64 bi = 0;
        unsigned grp = 0xffffffffu;
        if (T < nT) {
            const TupleConst& tc = sT[threadIdx.x];
            grp = (unsigned)tc.group;
            const bool bp_eq = tc.L.N_Bp == tc.L.N_B && (!tc.first || tc.E.N_Bp == tc.E.N_B) &&
                               (!tc.last || tc.H.N_Bp == tc.H.N_B);
            const bool fp_eq = tc.L.N_Fp == tc.L.N_F && (!tc.first || tc.E.N_Fp == tc.E.N_F) &&
                               (!tc.last || tc.H.N_Fp == tc.H.N_F);
            const bool twin = tc.twin_T != ~0ull && tc.twin_T >= A.twin_floor;
            if (bp_eq && fp_eq && !(tc.DMB < 0.0) && !twin) {
                for (int kA = 0; kA <= P.kmax[3]; ++kA) {
                    RunState rs;
                    run_memory(tc, 0.0, 0.0, (double)kA, Q, rs);
                    const double memD = mem_kO(tc, rs, 0.0, Q);
                    if (!(memD <= tc.DMB)) continue;           // Eq. 4
                    if (has) {
                        // R4 bound of t at this kA (channels at kW = kG = 0): skip the rows when
                        // even the bound cannot beat the best t found (the smaller kA stays on ties)
                        const double dkA = kA;
                        double lb = 0.0;
                        if (tc.nl0 > 0.0)
                            lb += tc.nl0 * (dmax(dmax(tc.L.C_F, tc.L.N_F), dkA * tc.L.sAd) +
                                            dmax(dmax(tc.L.C_B, tc.L.N_B), dkA * tc.L.sAh));
                        if (tc.nl1 > 0.0)
                            lb += tc.nl1 * (dmax(dmax(tc.L.C_F, tc.L.N_F), dkA * tc.L.sAd1) +
                                            dmax(dmax(tc.L.C_B1, tc.L.N_B), dkA * tc.L.sAh1));
                        if (tc.first)
                            lb += dmax(dmax(tc.E.C_F, tc.E.N_F), dkA * tc.E.sAd) +
                                  dmax(dmax(tc.E.C_B, tc.E.N_B), dkA * tc.E.sAh);
                        if (tc.last)
                            lb += dmax(dmax(tc.H.C_F, tc.H.N_F), dkA * tc.H.sAd) +
                                  dmax(dmax(tc.H.C_B, tc.H.N_B), dkA * tc.H.sAh);
                        if ((lb + tc.t_p2p) * (1.0 - 1e-12) >= bt) continue;
                    }
                    UnitState us;
                    unit_forward<UNIT>(tc, 0.0, (double)kA, FG, us);
                    run_backward<UNIT>(tc, us, 0.0, 0.0, (double)kA, FG, rs);
                    if (!(rs.t < bt)) continue;                 // ties: the smaller kA (idx) stays
                    if (d_kO<UNIT>(tc, us, rs, 0.0, FG) != 0.0) continue;
                    has = true; bt = rs.t; bm = memD / tc.D; bi = tc.idx_base + (u64)kA;
                }
            }
        }
        // per group of the warp's lanes: the least (t, idx)
        const unsigned peers = __match_any_sync(0xffffffffu, grp);
        double t = has ? bt : CUDART_INF;
        u64 ix = has ? bi : ~0ull;
        double m = bm;
        for (unsigned rest = peers; rest;) {
            const int src = __ffs(rest) - 1;
            rest &= rest - 1;
            const double ot = __shfl_sync(peers, t, src);
            const u64 oi = __shfl_sync(peers, ix, src);
            const double om = __shfl_sync(peers, m, src);
            if (ot < t || (ot == t && oi < ix)) { t = ot; ix = oi; m = om; }
        }
        const bool emit = (int)lane == __ffs(peers) - 1 && ix != ~0ull;
        warp_emit(emit, t, 0.0, m, ix, grp, A, lane);
    }
}

// Arbitrary index list (test hook): one thread per index, tuple built in registers.
template <bool UNIT>
__global__ void k_eval_at(DevProblem P, const DevGroup* __restrict__ groups, int ng,
                          const double* __restrict__ coef, const u64* __restrict__ idxs, long long n,
                          u64 total, unsigned* __restrict__ bad, double* t, double* d, double* mem,
                          uint8_t* feas) {
    __shared__ FGRow FG[16];
    load_fg(P, FG, threadIdx.x);
    __syncthreads();
    const u64 Q1 = P.Q1, R = Q1 * Q1 * Q1 * Q1;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const u64 idx = idxs[i];
        if (idx >= total) {          // outside the space: flag it (INVALID_ARG), never decode it
            atomicOr(bad, 1u);
            continue;
        }
        const u64 T = idx / R;
        u64 r = idx - T * R;
        const unsigned kA = (unsigned)(r % Q1); r /= Q1;
        const unsigned kO = (unsigned)(r % Q1); r /= Q1;
        const unsigned kG = (unsigned)(r % Q1); r /= Q1;
        const unsigned kW = (unsigned)r;
        TupleConst tc;
        make_tuple(P, groups, ng, coef, T, tc);
        UnitState us;
        RunState rs;
        unit_forward<UNIT>(tc, kW, kA, FG, us);
        run_memory(tc, kW, kG, kA, (double)P.Q, rs);
        run_backward<UNIT>(tc, us, kW, kG, kA, FG, rs);
        const double memD = mem_kO(tc, rs, (double)kO, (double)P.Q);
        if (t) t[i] = rs.t;
        if (d) d[i] = d_kO<UNIT>(tc, us, rs, (double)kO, FG);
        if (mem) mem[i] = memD / tc.D;
        if (feas)
            feas[i] = memD <= tc.DMB && kW <= (unsigned)P.kmax[0] && kG <= (unsigned)P.kmax[1] &&
                      kO <= (unsigned)P.kmax[2] && kA <= (unsigned)P.kmax[3];
    }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
static int sm_count(int device) {
    static std::atomic<int> cached[64];   // zero-initialised (static storage)
    if (device >= 0 && device < 64) {
        const int c = cached[device].load();
        if (c) return c;
    }
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    if (device >= 0 && device < 64) cached[device].store(n);
    return n;
}

cudaError_t launch_precompute(cudaStream_t st, int device, const DevProblem& P, const DevGroup* groups,
                              int ng, const double* coef, u64 T0, u64 nT, TupleConst* out, bool halves) {
    if (nT == 0) return cudaSuccess;
    const int threads = kPreThreads;
    u64 blocks = (nT + threads - 1) / threads;
    const u64 cap = (u64)sm_count(device) * 32;
    if (blocks > cap) blocks = cap;
    k_tuple_precompute<<<(unsigned)blocks, threads, 0, st>>>(P, groups, ng, coef, T0, nT, out, halves);
    return cudaGetLastError();
}

cudaError_t launch_precompute_segs(cudaStream_t st, int device, const DevProblem& P, const DevGroup* groups,
                                   int ng, const double* coef, const u64* seg, int nseg, u64 nT, TupleConst* out,
                                   bool halves) {
    if (nT == 0) return cudaSuccess;
    const int threads = kPreThreads;
    u64 blocks = (nT + threads - 1) / threads;
    const u64 cap = (u64)sm_count(device) * 32;
    if (blocks > cap) blocks = cap;
    k_tuple_precompute_segs<<<(unsigned)blocks, threads, 0, st>>>(P, groups, ng, coef, seg, nseg, nT, out, halves);
    return cudaGetLastError();
}

// shared memory of one eval CTA: factor tables + the tuples its 256 units touch
size_t eval_smem_bytes(unsigned upt) {
    const unsigned maxt = (kEvalThreads + upt - 1) / upt + 1;
    return 128 * sizeof(double) + maxt * sizeof(TupleConst);
}

// units per tuple: radix^2, padded to a multiple of 32 when >= 64 (warp-uniform tuples)
unsigned units_per_tuple(unsigned radix) {
    const unsigned r2 = radix * radix;
    return r2 >= 64 ? (r2 + 31) / 32 * 32 : r2;
}

template <bool UNIT, int MODE, int NT, int MINB>
static cudaError_t launch_eval_t(cudaStream_t st, int device, const DevProblem& P, const EvalArgs& A) {
    const size_t smem = eval_smem_bytes(A.upt);
    if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
    static std::atomic<unsigned long long> attr_set{0};   // the attribute is per device: one bit per device
    if (device >= 64 || !((attr_set.load() >> device) & 1ull)) {
        cudaError_t e = cudaFuncSetAttribute(k_eval<UNIT, MODE, NT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             200 * 1024);
        if (e != cudaSuccess) return e;
        if (device < 64) attr_set.fetch_or(1ull << device);
    }
    // cached occupancy query: one word (device << 40 | smem << 8 | CTAs per SM)
    static std::atomic<unsigned long long> occ{~0ull};
    const unsigned long long key = ((unsigned long long)(device & 0xffff) << 40) | ((unsigned long long)smem << 8);
    int per_sm = 0;
    const unsigned long long w = occ.load();
    if (w != ~0ull && (w & ~0xffull) == key) {
        per_sm = (int)(w & 0xff);
    } else {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_eval<UNIT, MODE, NT, MINB>, NT, smem);
        occ.store(key | (unsigned long long)(per_sm & 0xff));
    }
    if (per_sm < 1) per_sm = 1;
    u64 blocks = (A.n_units + NT - 1) / NT;
    const u64 cap = (u64)sm_count(device) * per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) return cudaSuccess;
    k_eval<UNIT, MODE, NT, MINB><<<(unsigned)blocks, NT, smem, st>>>(P, A);
    return cudaGetLastError();
}

// CTA shape of the frontier-mode eval kernel: threads x min CTAs per SM (register
// budget).  MIST_EVAL_CFG = 256x2 | 256x3 | 128x4 | 128x5 | 128x6 (tuning knob).
static int eval_cfg() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("MIST_EVAL_CFG");
        v = 0;   // default 256x2 (128 registers, no spills): best with the CTA queue (profiles/r1/ab_cq_summary.txt)
        if (s) {
            const char* names[5] = {"256x2", "256x3", "128x4", "128x5", "128x6"};
            for (int i = 0; i < 5; ++i)
                if (!strcmp(s, names[i])) v = i;
        }
    }
    return v;
}

template <bool UNIT, int NT, int MINB, bool CQ, int UPW = 1, bool NI = false, int MODE = 0>
static cudaError_t launch_eval_q(cudaStream_t st, int device, const DevProblem& P, const EvalArgs& A) {
    constexpr size_t NW = (size_t)NT * UPW;
    const size_t maxt = (NW + A.upt - 1) / A.upt + 1;
    const size_t smem = 128 * sizeof(double) + (CQ ? 2 : 1) * maxt * sizeof(TupleConst) + NW * sizeof(UnitState) +
                        (3 * NW + NT / 32 + 2) * sizeof(unsigned) + 2 * sizeof(u64) +
                        (CQ ? NW * P.Q1 * sizeof(unsigned short) : 0);
    if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
    static std::atomic<unsigned long long> attr_set{0};   // the attribute is per device: one bit per device
    if (device >= 64 || !((attr_set.load() >> device) & 1ull)) {
        cudaError_t e = cudaFuncSetAttribute(k_eval_q<UNIT, NT, MINB, CQ, UPW, NI, MODE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return e;
        if (device < 64) attr_set.fetch_or(1ull << device);
    }
    // cached occupancy query: one word (device << 40 | smem << 8 | CTAs per SM)
    static std::atomic<unsigned long long> occ{~0ull};
    const unsigned long long key = ((unsigned long long)(device & 0xffff) << 40) | ((unsigned long long)smem << 8);
    int per_sm = 0;
    const unsigned long long w = occ.load();
    if (w != ~0ull && (w & ~0xffull) == key) {
        per_sm = (int)(w & 0xff);
    } else {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_eval_q<UNIT, NT, MINB, CQ, UPW, NI, MODE>, NT, smem);
        occ.store(key | (unsigned long long)(per_sm & 0xff));
    }
    if (per_sm < 1) per_sm = 1;
    u64 blocks = (A.n_units + NW - 1) / NW;
    const u64 cap = (u64)sm_count(device) * per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) return cudaSuccess;
    k_eval_q<UNIT, NT, MINB, CQ, UPW, NI, MODE><<<(unsigned)blocks, NT, smem, st>>>(P, A);
    return cudaGetLastError();
}

// Units per thread per window of the CTA queue: 2 by default (windows of 512 units;
// cfg2 62.5 -> 60.2 ms, profiles/r1/ab_upw_summary.txt); MIST_EVAL_UPW=1 for 256.
static int eval_upw() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("MIST_EVAL_UPW");
        v = (s && s[0] == '1') ? 1 : 2;
    }
    return v;
}

// MIST_EVAL_QUEUE=0 selects the lockstep kG loop, 1 the warp run queue, 2 (default)
// the CTA-wide run queue.
static int eval_queue() {
    static int v = -1;
    if (v < 0) {
        const char* s = getenv("MIST_EVAL_QUEUE");
        v = (s && s[0] == '0') ? 0 : (s && s[0] == '1') ? 1 : 2;
    }
    return v;
}

// Called (not inlined) bound rows in the frontier kernel unless the kO loops are long:
// Q < 40 by default (measured same-box: cfg4 Q = 8 274 -> 263 ms, cfg2 Q = 10 25.0 ->
// 22.7 ms, cfg3 Q = 20 166 -> 153 ms; cfg5 Q = 50 windows 1.5-3% slower,
// profiles/r2/ab_noinline_summary.txt, ab_chunk_summary.txt); MIST_EVAL_NI=0/1 forces.
static bool eval_ni(int Q) {
    const char* s = getenv("MIST_EVAL_NI");
    if (s && (s[0] == '0' || s[0] == '1')) return s[0] == '1';
    return Q < 40;
}

template <bool UNIT>
static cudaError_t launch_frontier_eval(cudaStream_t st, int device, const DevProblem& P, const EvalArgs& A) {
    if (eval_queue() == 2) {
        if (eval_upw() == 2) {
            if (eval_cfg() == 1) {   // A/B: 3 CTAs per SM (85 registers)
                if (!UNIT && eval_ni(P.Q)) return launch_eval_q<UNIT, 256, 3, true, 2, true>(st, device, P, A);
                return launch_eval_q<UNIT, 256, 3, true, 2>(st, device, P, A);
            }
            if (eval_cfg() == 3) {   // A/B: 128-thread CTAs, 5 per SM (102 registers, 20 warps per SM)
                if (!UNIT && eval_ni(P.Q)) return launch_eval_q<UNIT, 128, 5, true, 2, true>(st, device, P, A);
                return launch_eval_q<UNIT, 128, 5, true, 2>(st, device, P, A);
            }
            if (!UNIT && eval_ni(P.Q)) return launch_eval_q<UNIT, 256, 2, true, 2, true>(st, device, P, A);
            return launch_eval_q<UNIT, 256, 2, true, 2>(st, device, P, A);
        }
        switch (eval_cfg()) {
            case 0: return launch_eval_q<UNIT, 256, 2, true>(st, device, P, A);
            default: return launch_eval_q<UNIT, 256, 3, true>(st, device, P, A);
        }
    }
    if (eval_queue() == 1) {
        switch (eval_cfg()) {
            case 0: return launch_eval_q<UNIT, 256, 2, false>(st, device, P, A);
            default: return launch_eval_q<UNIT, 256, 3, false>(st, device, P, A);
        }
    }
    switch (eval_cfg()) {
        case 1: return launch_eval_t<UNIT, 0, 256, 3>(st, device, P, A);
        case 2: return launch_eval_t<UNIT, 0, 128, 4>(st, device, P, A);
        case 3: return launch_eval_t<UNIT, 0, 128, 5>(st, device, P, A);
        case 4: return launch_eval_t<UNIT, 0, 128, 6>(st, device, P, A);
        default: return launch_eval_t<UNIT, 0, 256, 2>(st, device, P, A);
    }
}

// The pilot sub-grid sweep (MODE 2): the CTA run queue by default (windows of 256
// units); MIST_PILOT_KERNEL=lockstep selects the round-1 lockstep kernel.
static bool pilot_queue() {
    const char* s = getenv("MIST_PILOT_KERNEL");
    return !(s && !strcmp(s, "lockstep"));
}

cudaError_t launch_eval(cudaStream_t st, int device, const DevProblem& P, const EvalArgs& A, int mode) {
    if (P.unit_factors) {
        if (mode == 1) return launch_eval_t<true, 1, 256, 2>(st, device, P, A);
        if (mode == 2) {
            if (pilot_queue()) return launch_eval_q<true, 256, 2, true, 1, false, 2>(st, device, P, A);
            return launch_eval_t<true, 2, 256, 2>(st, device, P, A);
        }
        return launch_frontier_eval<true>(st, device, P, A);
    }
    if (mode == 1) return launch_eval_t<false, 1, 256, 2>(st, device, P, A);
    if (mode == 2) {
        if (pilot_queue()) {
            if (eval_ni(P.Q)) return launch_eval_q<false, 256, 2, true, 1, true, 2>(st, device, P, A);
            return launch_eval_q<false, 256, 2, true, 1, false, 2>(st, device, P, A);
        }
        return launch_eval_t<false, 2, 256, 2>(st, device, P, A);
    }
    return launch_frontier_eval<false>(st, device, P, A);
}

cudaError_t launch_pilot_zero(cudaStream_t st, int device, const DevProblem& P, const EvalArgs& A) {
    if (A.n_units == 0) return cudaSuccess;
    const int threads = 64;                                 // k_pilot_zero's NT
    u64 blocks = (A.n_units + threads - 1) / threads;
    const u64 cap = (u64)sm_count(device) * 16;
    if (blocks > cap) blocks = cap;
    if (P.unit_factors)
        k_pilot_zero<true><<<(unsigned)blocks, threads, 0, st>>>(P, A);
    else
        k_pilot_zero<false><<<(unsigned)blocks, threads, 0, st>>>(P, A);
    return cudaGetLastError();
}

cudaError_t launch_eval_at(cudaStream_t st, int device, const DevProblem& P, const DevGroup* groups,
                           int ng, const double* coef, const u64* idx, long long n, u64 total, unsigned* bad,
                           double* t, double* d, double* mem, uint8_t* feas) {
    if (n <= 0) return cudaSuccess;
    const int threads = 128;
    long long blocks = (n + threads - 1) / threads;
    const long long cap = (long long)sm_count(device) * 8;
    if (blocks > cap) blocks = cap;
    if (P.unit_factors)
        k_eval_at<true><<<(unsigned)blocks, threads, 0, st>>>(P, groups, ng, coef, idx, n, total, bad, t, d, mem,
                                                               feas);
    else
        k_eval_at<false><<<(unsigned)blocks, threads, 0, st>>>(P, groups, ng, coef, idx, n, total, bad, t, d, mem,
                                                                feas);
    return cudaGetLastError();
}

}  // namespace mist
