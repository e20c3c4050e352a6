// mist_sample_dev.cu -- a12 on the device (alpha-sampling
// next to the sweep, so an MILP-only caller never moves the frontier to the host).
//
// Paper: "a series of alpha in [0, 1] are sampled uniformly to construct a
// Pareto frontier" for min alpha*G*t + (1-alpha)*d s.t. the memory budget
// (Eq. 4).  Reading O11 / L29:
// alpha_j = j/(K-1), j = 0..K-1; ties to the smaller t, then the smaller idx;
// distinct picks in order of first appearance.  The score is evaluated as
// ((alpha*G)*t) + ((1-alpha)*y) with every operation rounded separately (no
// FMA contraction), the expression order of the reading, so the argmin is the
// same decision on any conforming implementation.
#include <cuda_runtime.h>
#include <stdint.h>

#include "mist_internal.h"

namespace mist {

namespace {
// one strided view of the frontier: SoA (stride 1) or mist_point_t (stride 4)
struct PtView {
    const double* t;
    const double* y;
    const unsigned long long* idx;
    int stride;
};

__device__ __forceinline__ double score_of(double aG, double om, double t, double y) {
    return __dadd_rn(__dmul_rn(aG, t), __dmul_rn(om, y));
}
}  // namespace

// One warp per group; lane l owns alpha_{j0+l} for j0 = 0, 32, ... < K.  Outputs:
// picked[g*K + k] = frontier position of the k-th distinct pick (-1 padded),
// npick[g] = number of distinct picks.
__global__ void k_sample_alpha(PtView v, const int64_t* __restrict__ off, const double* __restrict__ Gv,
                               long long ng, int K, int64_t* __restrict__ picked, int32_t* __restrict__ npick) {
    const unsigned lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long g = warp; g < ng; g += nw) {
        const int64_t a = off[g], b = off[g + 1];
        const double G = Gv[g];
        int64_t* out = picked + g * (long long)K;
        int cnt = 0;
        for (int j0 = 0; j0 < K; j0 += 32) {
            const int j = j0 + (int)lane;
            int64_t best = -1;
            if (j < K && b > a) {
                const double alpha = __ddiv_rn((double)j, (double)(K - 1));
                const double aG = __dmul_rn(alpha, G), om = __dsub_rn(1.0, alpha);
                best = a;
                double bt = v.t[a * v.stride];
                double bs = score_of(aG, om, bt, v.y[a * v.stride]);
                unsigned long long bi = v.idx[a * v.stride];
                for (int64_t i = a + 1; i < b; ++i) {
                    const double ti = v.t[i * v.stride];
                    const double s = score_of(aG, om, ti, v.y[i * v.stride]);
                    const unsigned long long ii = v.idx[i * v.stride];
                    if (s < bs || (s == bs && (ti < bt || (ti == bt && ii < bi)))) {
                        best = i; bs = s; bt = ti; bi = ii;
                    }
                }
            }
            // distinct picks in order of first appearance (lane 0, j ascending)
            for (int l = 0; l < 32 && j0 + l < K; ++l) {
                const int64_t c = __shfl_sync(0xffffffffu, best, l);
                if (lane == 0 && c >= 0) {
                    bool seen = false;
                    for (int k = 0; k < cnt; ++k) seen |= out[k] == c;
                    if (!seen) out[cnt++] = c;
                }
            }
            cnt = __shfl_sync(0xffffffffu, cnt, 0);
        }
        for (int k = cnt + (int)lane; k < K; k += 32) out[k] = -1;
        if (lane == 0) npick[g] = cnt;
    }
}

cudaError_t sample_alpha(cudaStream_t st, const double* t, const double* y, const unsigned long long* idx,
                         int stride, const int64_t* off, const double* G, long long ng, int K, int64_t* picked,
                         int32_t* npick) {
    if (ng <= 0) return cudaSuccess;
    PtView v{t, y, idx, stride};
    const int threads = 256;
    long long blocks = (ng * 32 + threads - 1) / threads;
    if (blocks > 148LL * 64) blocks = 148LL * 64;
    k_sample_alpha<<<(unsigned)blocks, threads, 0, st>>>(v, off, G, ng, K, picked, npick);
    return cudaGetLastError();
}

// picked positions -> points (padding: idx = ~0, t = y = mem = 0)
__global__ void k_gather_picks(CandBuf c, const int64_t* __restrict__ picked, long long n,
                               mist_point_t* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int64_t p = picked[i];
        mist_point_t q;
        if (p >= 0) { q.idx = c.idx[p]; q.t = c.t[p]; q.y = c.y[p]; q.mem = c.mem[p]; }
        else { q.idx = ~0ull; q.t = 0.0; q.y = 0.0; q.mem = 0.0; }
        out[i] = q;
    }
}

cudaError_t gather_picks(cudaStream_t st, const CandBuf& c, const int64_t* picked, long long n, mist_point_t* out) {
    if (n <= 0) return cudaSuccess;
    long long blocks = (n + 255) / 256;
    if (blocks > 148LL * 32) blocks = 148LL * 32;
    k_gather_picks<<<(unsigned)blocks, 256, 0, st>>>(c, picked, n, out);
    return cudaGetLastError();
}

}  // namespace mist
