// mist_intf.cu -- Alg. 1 over observation tables and the fitting of its slowdown
// factors, sm_100a, FP64 CUDA cores.
//
// Paper: Alg. 1 "Batched Interference Estimation"; the
// factors are fitted "data-driven": "different shapes and combinations of
// concurrent kernels are sampled and benchmarked, and the resulting runtime
// data is used to train the slowdown factors" (line 561).  Readings F1-F3
// (DESIGN.md 9): squared-relative-error loss, coordinate descent over the 28
// member factors, nested-grid search per coordinate.
//
// k_pred_intf: one thread per observation row, HBM-bound (32 B in, 8 B out).
// k_fit_loss: one pass over the observations evaluates the loss of 32 candidate
// values of one coordinate at once -- lane k of every warp owns candidate k, the
// warp's 32 rows are loaded coalesced and broadcast by shuffles -- so the rows
// are read once per grid level and the FP64 work (32 x Alg. 1 per row) dominates.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <cmath>
#include <string>
#include <vector>

#include "mist.h"
#include "mist_internal.h"

namespace {

constexpr int kGrid = 31;      // F3: grid points per level (lane 0 holds the current value)
constexpr int kLevels = 3;
constexpr int kFitThreads = 256;

struct FactorTable {
    double f[16][4];           // member factors (1 for non-members)
    double g[16][4];           // 1/f for members, 0 for non-members (exact zeros through the update)
};

FactorTable make_table(const double F[16][4]) {
    FactorTable t;
    for (int p = 0; p < 16; ++p)
        for (int j = 0; j < 4; ++j) {
            const bool member = __builtin_popcount(p) >= 2 && ((p >> j) & 1);
            t.f[p][j] = member ? F[p][j] : 1.0;
            t.g[p][j] = member ? 1.0 / F[p][j] : 0.0;
        }
    return t;
}

// Alg. 1 by the nonzero pattern of the row (O7: at most one mask
// matches per round, so the literal loop over masks is a table lookup);
// (po, co) names one factor overridden by (fo, go) (the fitted coordinate).
__device__ __forceinline__ double alg1(double x0, double x1, double x2, double x3,
                                       const double (*f)[4], const double (*g)[4], int po, int co, double fo,
                                       double go) {
    double T = 0.0;
#pragma unroll
    for (int round = 0; round < 3; ++round) {
        const bool q0 = x0 != 0.0, q1 = x1 != 0.0, q2 = x2 != 0.0, q3 = x3 != 0.0;
        const int pat = (int)q0 | ((int)q1 << 1) | ((int)q2 << 2) | ((int)q3 << 3);
        if (__popc(pat) < 2) break;
        double f0 = f[pat][0], f1 = f[pat][1], f2 = f[pat][2], f3 = f[pat][3];
        double g0 = g[pat][0], g1 = g[pat][1], g2 = g[pat][2], g3 = g[pat][3];
        if (pat == po) {
            if (co == 0) { f0 = fo; g0 = go; }
            if (co == 1) { f1 = fo; g1 = go; }
            if (co == 2) { f2 = fo; g2 = go; }
            if (co == 3) { f3 = fo; g3 = go; }
        }
        const double s0 = x0 * f0, s1 = x1 * f1, s2 = x2 * f2, s3 = x3 * f3;
        double ov = q0 ? s0 : CUDART_INF;          // min over the members
        ov = (q1 && s1 < ov) ? s1 : ov;
        ov = (q2 && s2 < ov) ? s2 : ov;
        ov = (q3 && s3 < ov) ? s3 : ov;
        x0 = (s0 - ov) * g0;                       // argmin -> 0, non-members -> 0
        x1 = (s1 - ov) * g1;
        x2 = (s2 - ov) * g2;
        x3 = (s3 - ov) * g3;
        T += ov;
    }
    return T + (((x0 + x1) + x2) + x3);
}

constexpr int kPredRows = 4;   // rows per thread per iteration: their loads are issued together (MLP)

__global__ void k_pred_intf(FactorTable tab, const double4* __restrict__ X, long long n, double* __restrict__ T) {
    __shared__ double sf[16][4], sg[16][4];
    if (threadIdx.x < 64) {
        sf[threadIdx.x >> 2][threadIdx.x & 3] = tab.f[threadIdx.x >> 2][threadIdx.x & 3];
        sg[threadIdx.x >> 2][threadIdx.x & 3] = tab.g[threadIdx.x >> 2][threadIdx.x & 3];
    }
    __syncthreads();
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n; i0 += stride * kPredRows) {
        double4 x[kPredRows];
#pragma unroll
        for (int r = 0; r < kPredRows; ++r) {
            const long long i = i0 + r * stride;
            x[r] = i < n ? X[i] : make_double4(0.0, 0.0, 0.0, 0.0);
        }
#pragma unroll
        for (int r = 0; r < kPredRows; ++r) {
            const long long i = i0 + r * stride;
            if (i < n) T[i] = alg1(x[r].x, x[r].y, x[r].z, x[r].w, sf, sg, -1, -1, 1.0, 1.0);
        }
    }
}

// Observation check: rows with a negative or non-finite channel, or a
// non-positive / non-finite observed total, are counted in *bad.
__global__ void k_check_obs(const double4* __restrict__ X, const double* __restrict__ Tobs, long long n,
                            unsigned long long* bad) {
    unsigned long long b = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double4 x = X[i];
        const bool ok = x.x >= 0.0 && x.y >= 0.0 && x.z >= 0.0 && x.w >= 0.0 && isfinite(x.x) && isfinite(x.y) &&
                        isfinite(x.z) && isfinite(x.w) && (!Tobs || (Tobs[i] > 0.0 && isfinite(Tobs[i])));
        b += ok ? 0 : 1;
    }
    if (b) atomicAdd(bad, b);
}

// Loss of 32 candidate values of factor (po, co): lane k of every warp evaluates
// candidate cand[k] on the warp's rows; per-block partial sums per candidate.
__global__ void __launch_bounds__(kFitThreads)
k_fit_loss(FactorTable tab, const double4* __restrict__ X, const double* __restrict__ Tobs, long long n, int po,
           int co, const double* __restrict__ cand, double* __restrict__ partial) {
    __shared__ double sf[16][4], sg[16][4];
    __shared__ double wsum[kFitThreads / 32][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < 64) {
        sf[threadIdx.x >> 2][threadIdx.x & 3] = tab.f[threadIdx.x >> 2][threadIdx.x & 3];
        sg[threadIdx.x >> 2][threadIdx.x & 3] = tab.g[threadIdx.x >> 2][threadIdx.x & 3];
    }
    __syncthreads();
    const double fo = cand[lane], go = 1.0 / fo;
    double acc = 0.0;
    const long long wstride = (long long)gridDim.x * (kFitThreads / 32) * 32;
    for (long long base = ((long long)blockIdx.x * (kFitThreads / 32) + warp) * 32; base < n; base += wstride) {
        const long long r = base + lane;
        double4 x = make_double4(0.0, 0.0, 0.0, 0.0);
        double ob = 1.0;
        if (r < n) { x = X[r]; ob = Tobs[r]; }
        const int cnt = (int)((n - base) < 32 ? (n - base) : 32);
        for (int j = 0; j < cnt; ++j) {
            const double x0 = __shfl_sync(0xffffffffu, x.x, j), x1 = __shfl_sync(0xffffffffu, x.y, j);
            const double x2 = __shfl_sync(0xffffffffu, x.z, j), x3 = __shfl_sync(0xffffffffu, x.w, j);
            const double o = __shfl_sync(0xffffffffu, ob, j);
            const double e = (alg1(x0, x1, x2, x3, sf, sg, po, co, fo, go) - o) / o;   // F1
            acc += e * e;
        }
    }
    wsum[warp][lane] = acc;
    __syncthreads();
    if (warp == 0) {
        double s = 0.0;
        for (int w = 0; w < kFitThreads / 32; ++w) s += wsum[w][lane];
        partial[(long long)blockIdx.x * 32 + lane] = s;
    }
}

// losses[k] = sum over blocks of partial[b][k] / n: warp w sums blocks b = w (mod 8)
// in order, then the 8 warp sums are added in warp order (deterministic)
__global__ void k_fit_reduce(const double* __restrict__ partial, int nb, long long n, double* __restrict__ losses) {
    __shared__ double ws[8][32];
    const int k = threadIdx.x & 31, w = threadIdx.x >> 5;
    double s = 0.0;
    for (int b = w; b < nb; b += 8) s += partial[(long long)b * 32 + k];
    ws[w][k] = s;
    __syncthreads();
    if (w == 0) {
        double t = 0.0;
        for (int v = 0; v < 8; ++v) t += ws[v][k];
        losses[k] = t / (double)n;
    }
}

int sm_count(int dev) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

mist_status_t fail(mist_ctx_t* ctx, mist_status_t st, const std::string& msg) {
    if (ctx) ctx->last_error = msg;
    return st;
}

bool valid_factors(const double F[16][4]) {
    for (int p = 0; p < 16; ++p)
        for (int j = 0; j < 4; ++j)
            if (__builtin_popcount(p) >= 2 && ((p >> j) & 1) && !(F[p][j] >= 1.0 && std::isfinite(F[p][j])))
                return false;
    return true;
}

// rows valid?  (one check kernel + one 8-byte copy)
mist_status_t check_rows(mist_ctx_t* ctx, const double* X, const double* Tobs, int64_t n) {
    unsigned long long* bad = nullptr;
    if (cudaMallocAsync(&bad, sizeof(*bad), ctx->stream) != cudaSuccess) return fail(ctx, MIST_ERR_OOM, "cudaMalloc");
    cudaMemsetAsync(bad, 0, sizeof(*bad), ctx->stream);
    long long blocks = (n + 255) / 256;
    if (blocks > sm_count(ctx->device) * 8LL) blocks = sm_count(ctx->device) * 8LL;
    k_check_obs<<<(unsigned)blocks, 256, 0, ctx->stream>>>(reinterpret_cast<const double4*>(X), Tobs, n, bad);
    ctx->stats.kernel_launches++;
    unsigned long long h = 0;
    cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream);
    const cudaError_t e = cudaStreamSynchronize(ctx->stream);
    cudaFreeAsync(bad, ctx->stream);
    if (e != cudaSuccess) return fail(ctx, MIST_ERR_CUDA, cudaGetErrorString(e));
    if (h) return fail(ctx, MIST_ERR_INVALID_ARG, std::to_string(h) + " invalid observation rows");
    return MIST_OK;
}

}  // namespace

extern "C" mist_status_t mist_pred_intf(mist_ctx_t* ctx, const double* X, int64_t n, const double intf[16][4],
                                        double* T) {
    if (!ctx || n < 0 || (n > 0 && (!X || !T)) || !intf) return fail(ctx, MIST_ERR_INVALID_ARG, "null argument");
    if (!valid_factors(intf)) return fail(ctx, MIST_ERR_INVALID_ARG, "member factor < 1 or not finite");
    if ((reinterpret_cast<uintptr_t>(X) & 31) != 0) return fail(ctx, MIST_ERR_INVALID_ARG, "X not 32-byte aligned");
    if (n == 0) return MIST_OK;
    cudaSetDevice(ctx->device);
    const FactorTable tab = make_table(intf);
    long long blocks = (n + 255) / 256;
    const long long cap = sm_count(ctx->device) * 8LL;
    if (blocks > cap) blocks = cap;
    k_pred_intf<<<(unsigned)blocks, 256, 0, ctx->stream>>>(tab, reinterpret_cast<const double4*>(X), n, T);
    ctx->stats.kernel_launches++;
    const cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return fail(ctx, MIST_ERR_CUDA, cudaGetErrorString(e));
    return MIST_OK;
}

extern "C" mist_status_t mist_fit_intf(mist_ctx_t* ctx, const double* X, const double* Tobs, int64_t n,
                                       const double init[16][4], int32_t iters, double fmax, double out[16][4],
                                       double* loss) {
    if (!ctx || n < 1 || !X || !Tobs || !init || !out || iters < 0 || !(fmax > 1.0) || !std::isfinite(fmax))
        return fail(ctx, MIST_ERR_INVALID_ARG, "invalid argument");
    if (!valid_factors(init)) return fail(ctx, MIST_ERR_INVALID_ARG, "member factor < 1 or not finite");
    if ((reinterpret_cast<uintptr_t>(X) & 31) != 0) return fail(ctx, MIST_ERR_INVALID_ARG, "X not 32-byte aligned");
    cudaSetDevice(ctx->device);
    mist_status_t st = check_rows(ctx, X, Tobs, n);
    if (st != MIST_OK) return st;
    long long nb = (n + kFitThreads - 1) / kFitThreads;
    const long long cap = sm_count(ctx->device) * 4LL;
    if (nb > cap) nb = cap;
    double *partial = nullptr, *dcand = nullptr, *dloss = nullptr;
    if (cudaMallocAsync(&partial, nb * 32 * sizeof(double), ctx->stream) != cudaSuccess ||
        cudaMallocAsync(&dcand, 64 * sizeof(double), ctx->stream) != cudaSuccess)
        return fail(ctx, MIST_ERR_OOM, "cudaMalloc");
    dloss = dcand + 32;
    double F[16][4];
    for (int p = 0; p < 16; ++p)
        for (int j = 0; j < 4; ++j) F[p][j] = init[p][j];
    std::vector<double> cand(32), losses(32);
    cudaError_t e = cudaSuccess;
    // loss of 32 candidates of coordinate (p, j) around the current table F
    auto eval = [&](int p, int j) -> cudaError_t {
        const FactorTable tab = make_table(F);
        cudaMemcpyAsync(dcand, cand.data(), 32 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream);
        k_fit_loss<<<(unsigned)nb, kFitThreads, 0, ctx->stream>>>(tab, reinterpret_cast<const double4*>(X), Tobs, n,
                                                                    p, j, dcand, partial);
        k_fit_reduce<<<1, 256, 0, ctx->stream>>>(partial, (int)nb, n, dloss);
        ctx->stats.kernel_launches += 2;
        cudaMemcpyAsync(losses.data(), dloss, 32 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
        return cudaStreamSynchronize(ctx->stream);
    };
    double cur_loss = 0.0;
    {
        // loss of the initial table: every lane evaluates an unchanged factor
        for (int k = 0; k < 32; ++k) cand[k] = F[3][0];
        e = eval(3, 0);
        cur_loss = losses[0];
    }
    for (int it = 0; it < iters && e == cudaSuccess; ++it)
        for (int p = 0; p < 16 && e == cudaSuccess; ++p) {
            if (__builtin_popcount(p) < 2) continue;
            for (int j = 0; j < 4 && e == cudaSuccess; ++j) {
                if (!((p >> j) & 1)) continue;
                // F2/F3: nested grids over [1, fmax]; a value replaces the current one only if strictly better
                double best = F[p][j], best_loss = 0.0, lo = 1.0, hi = fmax;
                for (int lev = 0; lev < kLevels && e == cudaSuccess; ++lev) {
                    cand[0] = best;
                    for (int k = 0; k < kGrid; ++k) cand[1 + k] = lo + (hi - lo) * k / (kGrid - 1);
                    e = eval(p, j);
                    if (e != cudaSuccess) break;
                    if (lev == 0) best_loss = losses[0];
                    int kb = 1;
                    for (int k = 2; k <= kGrid; ++k)
                        if (losses[k] < losses[kb]) kb = k;     // first minimum
                    if (losses[kb] < best_loss) { best = cand[kb]; best_loss = losses[kb]; }
                    const double w = (hi - lo) / (kGrid - 1);
                    lo = best - w > 1.0 ? best - w : 1.0;
                    hi = best + w;
                }
                F[p][j] = best;
                cur_loss = best_loss;
            }
        }
    cudaFreeAsync(partial, ctx->stream);
    cudaFreeAsync(dcand, ctx->stream);
    if (e != cudaSuccess) return fail(ctx, MIST_ERR_CUDA, cudaGetErrorString(e));
    for (int p = 0; p < 16; ++p)
        for (int j = 0; j < 4; ++j) out[p][j] = F[p][j];
    if (loss) *loss = cur_loss;
    return MIST_OK;
}
