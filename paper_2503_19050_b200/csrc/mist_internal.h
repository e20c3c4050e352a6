// mist_internal.h -- internal types of libmist (not part of the C ABI).
//
// Device data layout:
//   DevProblem   kernel parameter (by value, constant bank): model, mesh,
//                Q, factor tables F and 1/F, links.
//   DevGroup[]   global, n_groups entries (one per IntraStagePareto key).
//   double coef[6][n_b*n_tp]  profiled time tables, global (read by precompute only).
//   TupleConst[] global, one per tuple of the current chunk (a2 output),
//                staged into shared memory by the eval kernel.
//   candidates   SoA arrays {t, y, mem, idx, group} (a8 output).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "mist.h"

namespace mist {

enum { kAR = 0, kAG = 1, kRS = 2, kP2P = 3 };

struct DevProblem {
    // model (mist_model_t)
    int L, h, a, k, f, V, s, e, g, p, fl, nrm;
    int N, M;
    int Q, Q1, nz;
    int zlev[4];               // enumerated ZeRO levels, ascending
    int n_b, n_tp;
    int ykey;
    int unit_factors;          // all Alg. 1 factors == 1
    int ckpt_ends;             // preset: CKPT c in {0, l} only
    int kmax[4];               // preset: largest admitted kW, kG, kO, kA (0 or Q)
    long long B;
    long long mem_budget;
    double bw[4][2], lat[4][2];
    double bw_h2d, bw_d2h;
    double F[16][4];           // slowdown factors
    double IF[16][4];          // 1 / F
};

struct DevGroup {
    int G, first, last, w, l, n, m, n_splits;
    int tp[MIST_MAX_SPLITS], dp[MIST_MAX_SPLITS], b[MIST_MAX_SPLITS];
    int ti[MIST_MAX_SPLITS];   // row of (b, tp) in the coefficient tables
    unsigned long long tuple_offset, config_offset;
};

// Per-block phase constants of one tuple.  Channel values of a
// configuration are affine in the ratio indices k = Q*ratio:
//   F : [C_F, N_F,  kW sWh,                  kA sAd]
//   B : [C_B, N_B,  kW sWh + kG sGh + kA sAh, kG sGd]
//   F': [C_F, N_Fp, F.H + kO sOh + kG sGh,    F.D + kO sOd + kW sWd]
//   B': [C_B, N_Bp, B.H,                      B.D]
struct BlockConst {
    double C_F, C_B, C_B1;     // C_B1: checkpointed layer (recompute), layers only
    double N_F, N_B, N_Fp, N_Bp;
    double sWh, sGh, sOh, sWd, sGd, sOd;
    double sAh, sAd, sAh1, sAd1;   // activation slopes, r = 0 / r = 1 (layers)
};

struct TupleConst {
    unsigned long long idx_base;   // global config index of ratio tuple (0,0,0,0)
    int group, first, last, c;
    double nl0, nl1;               // l - c, c (layer counts of the two layer kinds)
    double t_p2p;                  // [!last] p2p + [!first] p2p
    BlockConst L, E, H;            // layer, embedding (first), LM head (last)
    // O9 memory, every quantity multiplied by D = Q*TP*DP (exact integers)
    double mW, mG, mO;             // coefficients of (Q-kW), (Q-kG), (Q-kO) in D*M_s
    double wb_c, wb_k;             // D*M_wb = wb_c + wb_k*kW
    double gb_c, gb_k;             // D*M_gb = gb_c + gb_k*kG
    double ob_k;                   // D*M_ob = ob_k*kO
    double ma_k;                   // D*M_a  = ma_k*(Q-kA)
    double DA, DAx;                // D*A_full, [c>0]*D*A_full
    double DMB;                    // D*Mem_Budget
    double D;
    // L20 twin: at DP = 1 every ZeRO level has the same t and d (all sigmas 1, no DP
    // collective) and a memory non-decreasing in z, so a tuple with z above the lowest
    // enumerated level is beaten config by config by its twin at the lowest level
    // (same group, split and c; smaller idx).  twin_T = that twin's global tuple
    // index, or ~0 when the tuple is not such a duplicate.
    unsigned long long twin_T;
    unsigned long long pad_;
};

// Candidate buffer (SoA).  One record per kept OO-run (P13 prefilter).
struct CandBuf {
    double* t = nullptr;
    double* y = nullptr;
    double* mem = nullptr;
    unsigned long long* idx = nullptr;
    unsigned* group = nullptr;
    long long cap = 0;
};

struct SortScratch {
    unsigned long long* key_t[2] = {nullptr, nullptr};
    unsigned* key_g[2] = {nullptr, nullptr};
    unsigned* val[2] = {nullptr, nullptr};
    unsigned* block_hist = nullptr;    // [256][tiles]
    unsigned* digit_hist = nullptr;    // [12][256] global histograms
    double* gy = nullptr;              // y gathered into sorted order
    unsigned long long* gidx = nullptr;   // idx gathered into sorted order
    long long cap = 0;
    long long hist_cap = 0;
};

// k_eval arguments.  MODE 0 (frontier): one candidate per OO-run with a
// feasible config -> cand; MODE 1 (dense): t/d/mem/feas for idx in [lo, hi).
struct EvalArgs {
    const TupleConst* tuples;   // tuples of the chunk
    unsigned long long n_units; // threads of work = tuples * upt
    unsigned upt;               // units (kW, kA) per tuple, radix^2 padded (units_per_tuple)
    CandBuf cand;
    unsigned long long* cand_count;
    unsigned long long* fp;     // [2*n_groups] (count, hash) or null
    unsigned long long* phases; // PredINTF rows evaluated (algorithmic work counter) or null
    unsigned long long lo, hi;
    double *t, *d, *mem;
    uint8_t* feas;
    // MODE 2 (pilot): sub-grid of ratio values vals[0..nv) on every axis; R3 = nv^3
    unsigned nv;
    unsigned vals[16];
    // staircase filter (MODE 0): a per-group frontier of real feasible configs
    // (sorted by t, y strictly decreasing); a candidate beaten by one is dropped
    const double* f_t;
    const double* f_y;
    const unsigned long long* f_idx;
    const int64_t* f_off;       // [n_groups+1], null = no filter
    int no_r7;                  // A/B knob: bit 0 no R7 at all (MIST_R7=0), bit 1 no tuple-level cut (MIST_R7=unit)
    // L20 twins: a tuple with twin_T >= twin_floor is skipped (its twin is swept in
    // the same call); ~0 disables (fingerprints, MIST_DEDUP=0)
    unsigned long long twin_floor;
    // unit passes of the frontier sweep: 0 = every unit; 1 = units with kW and kA both
    // even; 2 = the others (their staircase then includes pass 1's frontier)
    int unit_pass;
};

struct ReduceStats {
    int passes = 0;
    long long launches = 0;
};

}  // namespace mist

// mist_shard_ranges as a vector (mist_enum.cpp)
std::vector<std::pair<uint64_t, uint64_t>> mist_shard_blocks(uint64_t n_tuples, int rank, int world);

namespace mist {
// Host buffer in page-locked memory (D2H at full PCIe speed), grown on demand.
// resize() keeps no contents; release() frees it.
template <typename T>
struct PinnedVec {
    T* p = nullptr;
    size_t n = 0, cap = 0;
    cudaError_t resize(size_t m) {
        if (m > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            const size_t want = std::max<size_t>(m, 1024);
            cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&p), want * sizeof(T));
            if (e != cudaSuccess) { p = nullptr; n = 0; return e; }
            cap = want;
        }
        n = m;
        return cudaSuccess;
    }
    T* data() { return p; }
    const T* data() const { return p; }
    size_t size() const { return n; }
    T& operator[](size_t i) { return p[i]; }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = cap = 0;
    }
};

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};
}  // namespace mist

struct mist_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int timing = 1;
    int rank = 0, world = 1;
    void* nccl = nullptr;          // ncclComm_t
    std::string last_error;
    mist_stats_t stats{};
    // device scratch (grown on demand, freed by mist_ctx_destroy)
    mist::DevBuf cand_mem, sort_mem, tuples, scan_tmp, groups, coef, counters, fp, xfer, out, foff, segs;
    mist::DevBuf seg;   // scratch of the group-bucket frontier reduction (mist_segfront.cu)
    mist::CandBuf cand;            // views into cand_mem
    mist::SortScratch sort;        // views into sort_mem
    // cached last frontier (for BUFFER_TOO_SMALL retries), page-locked
    mist::PinnedVec<mist_point_t> cache_points;
    mist::PinnedVec<int64_t> cache_offsets;
    mist::PinnedVec<uint64_t> cache_fp;
    uint64_t cache_key = 0;
    int cache_valid = 0;
    int64_t cache_nf = 0;          // frontier points of the last computed call
    bool cache_direct = false;     // the last computed call wrote its points to the caller directly
    // inputs of the last validated prepare() (every byte that determines the device
    // tables) and its config count: an identical call skips re-validation
    std::vector<unsigned char> prep_in;
    uint64_t prep_nc = 0;
    int prep_valid = 0;
    mist::PinnedVec<unsigned char> prep_stage;   // page-locked staging of the uploaded tables
    // timing events (pairs)
    struct EvUse { int cat, base; bool done; };
    std::vector<cudaEvent_t> ev_pool;
    std::vector<EvUse> ev_used;   // open and closed intervals (pool index of start; end = base + 1)
    std::vector<int> ev_free;     // pool pairs whose interval has been read
};
