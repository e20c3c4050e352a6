// mist_segfront.cu -- a9 + a10 by group buckets: the exact per-group Pareto
// frontier (O10, PAPER.md line 660 / Eq. 3) of a candidate set without a
// global sort.
//
//   level 0  k_seg_count    : per candidate its rank within its group
//                             (warp-aggregated atomics), per-group counts
//            scan           : group offsets
//            k_seg_scatter  : records into group-contiguous order
//   level L  k_chunk_front  : one CTA per chunk of <= kChunk records of one
//                             group: bitonic sort in shared memory by
//                             (t, y, idx), then the frontier flags
//                             y_k < min_{j<k} y_j (exclusive prefix min), and
//                             the chunk's frontier written back in place
//            scan + k_chunk_compact : chunk frontiers packed in group order
//   repeated while some group still spans several chunks: frontier(A u B) =
//   frontier(frontier(A) u frontier(B)) (O12), so every level is exact.
//
// Why the flag rule is the O10 frontier: after the lexicographic sort, an
// earlier element j has t_j <= t_k, and t_j = t_k implies (y_j, idx_j) <
// (y_k, idx_k); so j beats k iff y_j <= y_k, and no later element beats k.
// Output: cand[0, nf) sorted by (group, t), y strictly falling within a group,
// the same order and content as the radix-sort path (frontier_reduce).
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "mist_internal.h"

namespace mist {

typedef unsigned long long u64;
typedef unsigned u32;

cudaError_t scan_u32_exclusive(cudaStream_t st, const u32* in, u32* out, long long n, u32* tmp, u32* grand_total);
long long scan_tmp_words(long long n);

#ifndef MIST_CHUNK
#define MIST_CHUNK 1024
#endif
constexpr int kChunk = MIST_CHUNK;    // records per chunk (one CTA)
constexpr int kChunkThreads = kChunk / 8;
constexpr int kPerThread = kChunk / kChunkThreads;
constexpr int kChunkSmem = (kChunk + 1) * (8 + 8 + 8) + kChunk * 2;   // t, y, idx (+ sentinel), permutation

// per candidate: rank within its group; counts per group (cnt pre-zeroed)
__global__ void k_seg_count(const u32* __restrict__ group, long long n, u32* __restrict__ cnt,
                            u32* __restrict__ rank) {
    const unsigned lane = threadIdx.x & 31;
    for (long long base = (blockIdx.x * (long long)blockDim.x + threadIdx.x) & ~31ll; base < n;
         base += (long long)gridDim.x * blockDim.x) {
        const long long i = base + lane;
        const bool ok = i < n;
        const u32 g = ok ? group[i] : 0xffffffffu;
        const u32 peers = __match_any_sync(0xffffffffu, g);
        const int leader = __ffs(peers) - 1;
        u32 b = 0;
        if (ok && (int)lane == leader) b = atomicAdd(cnt + g, (u32)__popc(peers));
        b = __shfl_sync(0xffffffffu, b, leader);
        if (ok) rank[i] = b + __popc(peers & ((1u << lane) - 1));
    }
}

__global__ void k_seg_scatter(CandBuf src, long long n, const u32* __restrict__ goff, const u32* __restrict__ rank,
                              CandBuf dst) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const u32 g = src.group[i];
        const u32 o = goff[g] + rank[i];
        dst.t[o] = src.t[i]; dst.y[o] = src.y[i]; dst.mem[o] = src.mem[i];
        dst.idx[o] = src.idx[i]; dst.group[o] = g;
    }
}

// chunks per group, a flag when any group needs more than one chunk
__global__ void k_seg_chunks(const u32* __restrict__ cnt, int ng, u32* __restrict__ cpg, u32* __restrict__ multi) {
    if (blockIdx.x == 0 && threadIdx.x == 0) cpg[ng] = 0;   // the scan runs over ng + 1 entries
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x) {
        const u32 c = (cnt[g] + kChunk - 1) / kChunk;
        cpg[g] = c;
        if (c > 1) atomicOr(multi, 1u);
    }
}

__device__ __forceinline__ bool lex_less(double ta, double ya, u64 ia, double tb, double yb, u64 ib) {
    return ta < tb || (ta == tb && (ya < yb || (ya == yb && ia < ib)));
}

__device__ __forceinline__ u32 block_excl_count(u32 mine, u32* s_wcnt, u32& all) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u32 pre = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 v = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += v;
    }
    if (lane == 31) s_wcnt[w] = pre;
    __syncthreads();
    u32 before = pre - mine;
    all = 0;
    for (int q = 0; q < kChunkThreads / 32; ++q) {
        const u32 v = s_wcnt[q];
        before += q < w ? v : 0u;
        all += v;
    }
    __syncthreads();                                      // s_wcnt free for the next use
    return before;
}

// One CTA per chunk (grid-stride over *nchunks).  The chunk's records are
// X[goff[g] + j*kChunk, +len); its frontier goes back to the chunk's start and
// its size to nf[c].  Prefilter: every thread drops the records of its own 8
// that another of its 8 beats (O10, pairwise), so only the survivors are sorted.
__global__ void __launch_bounds__(kChunkThreads)
k_chunk_front(CandBuf X, const u32* __restrict__ cnt, const u32* __restrict__ goff, const u32* __restrict__ co,
              const u32* __restrict__ cmap, const u32* __restrict__ fin, const u32* __restrict__ nchunks,
              u32* __restrict__ nf) {
    extern __shared__ __align__(16) double s_t[];     // [kChunk + 1] t, then y, idx; permutation [kChunk]
    double* s_y = s_t + (kChunk + 1);
    u64* s_i = reinterpret_cast<u64*>(s_y + (kChunk + 1));
    unsigned short* s_p = reinterpret_cast<unsigned short*>(s_i + (kChunk + 1));
    __shared__ double s_wmin[kChunkThreads / 32];
    __shared__ u32 s_wcnt[kChunkThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const u32 total = *nchunks;
    if (blockIdx.x == 0 && tid == 0) nf[total] = 0;      // the scan runs over total + 1 entries
    if (tid == 0) { s_t[kChunk] = CUDART_INF; s_y[kChunk] = CUDART_INF; s_i[kChunk] = ~0ull; }   // sentinel
    for (u32 c = blockIdx.x; c < total; c += gridDim.x) {
        const int g = (int)cmap[c];
        const u32 j = c - co[g];
        const u32 start = goff[g] + j * kChunk;
        const int len = (int)min((u32)kChunk, cnt[g] - j * kChunk);
        if (fin[g]) {                                     // already a final, sorted frontier
            if (tid == 0) nf[c] = (u32)len;
            continue;
        }
        __syncthreads();                                  // previous chunk done with smem
        for (int k = tid; k < len; k += kChunkThreads) {
            s_t[k] = X.t[start + k]; s_y[k] = X.y[start + k]; s_i[k] = X.idx[start + k];
        }
        __syncthreads();
        // thread-local prefilter over records k0 .. k0 + 7
        const int k0 = tid * kPerThread;
        double tt[kPerThread], yy[kPerThread];
        u64 ii[kPerThread];
#pragma unroll
        for (int q = 0; q < kPerThread; ++q) {
            const bool ok = k0 + q < len;
            tt[q] = ok ? s_t[k0 + q] : CUDART_INF;
            yy[q] = ok ? s_y[k0 + q] : CUDART_INF;
            ii[q] = ok ? s_i[k0 + q] : ~0ull;
        }
        unsigned alive = 0;
#pragma unroll
        for (int q = 0; q < kPerThread; ++q) {
            bool beaten = !(k0 + q < len);
#pragma unroll
            for (int r = 0; r < kPerThread; ++r)
                if (r != q)
                    beaten |= tt[r] <= tt[q] && yy[r] <= yy[q] && (tt[r] < tt[q] || yy[r] < yy[q] || ii[r] < ii[q]);
            if (!beaten) alive |= 1u << q;
        }
        u32 ns;
        u32 pos = block_excl_count((u32)__popc(alive), s_wcnt, ns);
#pragma unroll
        for (int q = 0; q < kPerThread; ++q)
            if ((alive >> q) & 1u) s_p[pos++] = (unsigned short)(k0 + q);
        int P = 32;
        while (P < (int)ns) P <<= 1;
        for (int k = (int)ns + tid; k < P; k += kChunkThreads) s_p[k] = (unsigned short)kChunk;   // sentinel
        __syncthreads();
        // bitonic sort of the survivors by (t, y, idx) ascending
        for (int size = 2; size <= P; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int q = tid; q < P / 2; q += kChunkThreads) {
                    const int a = 2 * q - (q & (stride - 1));   // pair (a, a + stride)
                    const int b = a + stride;
                    const bool up = (a & size) == 0;
                    const int pa = s_p[a], pb = s_p[b];
                    const bool gt = lex_less(s_t[pb], s_y[pb], s_i[pb], s_t[pa], s_y[pa], s_i[pa]);
                    if (gt == up) { s_p[a] = (unsigned short)pb; s_p[b] = (unsigned short)pa; }
                }
                __syncthreads();
            }
        }
        // frontier flags over sorted positions [0, ns): y_k < min over earlier y
        // (exclusive prefix min); thread owns kPerThread consecutive positions
        double ys[kPerThread];
        double m = CUDART_INF;
#pragma unroll
        for (int q = 0; q < kPerThread; ++q) {
            const int k = k0 + q;
            ys[q] = k < (int)ns ? s_y[s_p[k]] : CUDART_INF;
            m = fmin(m, ys[q]);
        }
        double incl = m;                                  // warp inclusive min-scan of thread minima
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl = fmin(incl, v);
        }
        if (lane == 31) s_wmin[w] = incl;
        double excl = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) excl = CUDART_INF;
        __syncthreads();
        for (int q = 0; q < w; ++q) excl = fmin(excl, s_wmin[q]);
        unsigned flags = 0;
#pragma unroll
        for (int q = 0; q < kPerThread; ++q) {
            if (k0 + q < (int)ns && ys[q] < excl) flags |= 1u << q;
            excl = fmin(excl, ys[q]);
        }
        u32 all;
        const u32 before = block_excl_count((u32)__popc(flags), s_wcnt, all);
        // read the kept records' mem before any write into the chunk (in place)
        double mm[kPerThread];
#pragma unroll
        for (int q = 0; q < kPerThread; ++q)
            mm[q] = ((flags >> q) & 1u) ? X.mem[start + s_p[k0 + q]] : 0.0;
        __syncthreads();
        u32 o = start + before;
#pragma unroll
        for (int q = 0; q < kPerThread; ++q) {
            if (!((flags >> q) & 1u)) continue;
            const int p = s_p[k0 + q];
            X.t[o] = s_t[p]; X.y[o] = s_y[p]; X.mem[o] = mm[q]; X.idx[o] = s_i[p]; X.group[o] = (u32)g;
            ++o;
        }
        if (tid == 0) nf[c] = all;
    }
}

// chunk c's nf[c] frontier records -> Y[out[c], +nf[c]) (out = exclusive scan of nf)
__global__ void k_chunk_compact(CandBuf X, const u32* __restrict__ goff, const u32* __restrict__ co,
                                const u32* __restrict__ cmap, const u32* __restrict__ nchunks,
                                const u32* __restrict__ nf, const u32* __restrict__ out, CandBuf Y) {
    const u32 total = *nchunks;
    for (u32 c = blockIdx.x; c < total; c += gridDim.x) {
        const int g = (int)cmap[c];
        const u32 start = goff[g] + (c - co[g]) * kChunk, n = nf[c], o = out[c];
        for (u32 k = threadIdx.x; k < n; k += blockDim.x) {
            Y.t[o + k] = X.t[start + k]; Y.y[o + k] = X.y[start + k]; Y.mem[o + k] = X.mem[start + k];
            Y.idx[o + k] = X.idx[start + k]; Y.group[o + k] = X.group[start + k];
        }
    }
}

// chunk -> group map (one thread per group writes its chunks), so a chunk's CTA reads
// its group with one load instead of a binary search over the chunk offsets
__global__ void k_seg_chunk_map(const u32* __restrict__ co, int ng, u32* __restrict__ cmap) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x)
        for (u32 c = co[g]; c < co[g + 1]; ++c) cmap[c] = (u32)g;
}

// next level's per-group counts and offsets from the packed chunk frontiers
// A group that fitted one chunk at this level already holds its final frontier,
// sorted (fin[g] = 1): later levels only carry it along.
__global__ void k_seg_regroup(const u32* __restrict__ co, int ng, const u32* __restrict__ out, u32* __restrict__ cnt,
                              u32* __restrict__ goff, u32* __restrict__ fin) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x) {
        const u32 a = out[co[g]], b = out[co[g + 1]];
        cnt[g] = b - a;
        goff[g] = a;
        if (co[g + 1] - co[g] == 1) fin[g] = 1u;
    }
}

__global__ void k_seg_copy(CandBuf src, long long n, CandBuf dst) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        dst.t[i] = src.t[i]; dst.y[i] = src.y[i]; dst.mem[i] = src.mem[i];
        dst.idx[i] = src.idx[i]; dst.group[i] = src.group[i];
    }
}

static unsigned grid_n(long long n, int threads, int cap = 148 * 8) {
    long long b = (n + threads - 1) / threads;
    return (unsigned)std::max<long long>(1, std::min<long long>(b, cap));
}

// Scratch words for ng groups and n candidates (u32): rank[n], cnt, goff, cpg, co
// (ng + 1 each), nf, out (nchunks + 1 each, nchunks <= n / kChunk + ng), two
// device words, scan tiles.
long long seg_scratch_words(long long n, long long ng) {
    const long long nch = n / kChunk + ng + 2;
    return n + 5 * (ng + 2) + 3 * (nch + 1) + 8 + 2 * scan_tmp_words(std::max(nch, ng + 1)) + 64;
}

cudaError_t frontier_reduce_seg(cudaStream_t st, CandBuf cand, long long n, int ng, u32* ws, long long ws_words,
                                long long* n_out, ReduceStats* rs) {
    cudaError_t err;
    if (n == 0) { *n_out = 0; return cudaSuccess; }
    if (2 * n > cand.cap || n >= (1ll << 32)) return cudaErrorInvalidValue;
    if (ws_words < seg_scratch_words(n, ng)) return cudaErrorInvalidValue;
    const long long nch_max = n / kChunk + ng + 2;
    u32* rank = ws;
    u32* cnt = rank + n;
    u32* goff = cnt + (ng + 2);
    u32* cpg = goff + (ng + 2);
    u32* co = cpg + (ng + 2);
    u32* nf = co + (ng + 2);
    u32* out = nf + (nch_max + 1);
    u32* cmap = out + (nch_max + 1);             // chunk -> group
    u32* fin = cmap + (nch_max + 1);             // group already final (one chunk at a previous level)
    u32* dev = fin + (ng + 2);                   // [0] nchunks, [1] multi, [2] total
    u32* stmp = dev + 8;
    CandBuf A = cand, B = cand;                   // A = [0, n), B = [n, 2n)
    B.t += n; B.y += n; B.mem += n; B.idx += n; B.group += n;
    const int T = 256;
    // level 0: bucket by group
    err = cudaMemsetAsync(cnt, 0, sizeof(u32) * (size_t)ng, st);
    if (err != cudaSuccess) return err;
    err = cudaMemsetAsync(fin, 0, sizeof(u32) * (size_t)ng, st);
    if (err != cudaSuccess) return err;
    k_seg_count<<<grid_n(n, T), T, 0, st>>>(A.group, n, cnt, rank);
    err = scan_u32_exclusive(st, cnt, goff, ng, stmp, nullptr);
    if (err != cudaSuccess) return err;
    k_seg_scatter<<<grid_n(n, T), T, 0, st>>>(A, n, goff, rank, B);
    rs->launches += 5;
    CandBuf X = B, Y = A;
    const unsigned cta = 148 * 8;
    {
        int d = 0;
        cudaGetDevice(&d);
        static std::atomic<unsigned long long> attr{0};   // the attribute is per device: one bit per device
        if (d >= 64 || !((attr.load() >> d) & 1ull)) {
            err = cudaFuncSetAttribute(k_chunk_front, cudaFuncAttributeMaxDynamicSharedMemorySize, kChunkSmem);
            if (err != cudaSuccess) return err;
            if (d < 64) attr.fetch_or(1ull << d);
        }
    }
    long long n_cur = n;                          // records entering the level (an upper bound)
    for (int level = 0;; ++level) {
        // a group whose frontier alone exceeds a chunk never fits one: give up after a few
        // levels and let the caller take the radix-sort path (same result)
        if (level == 8) return cudaErrorNotSupported;
        // one host round trip per level: grids are sized from the bound n_cur / kChunk + ng on
        // chunks (the kernels read the true count from the device), and the multi flag and the
        // frontier total come back together at the end of the level
        const long long nch_bound = n_cur / kChunk + ng + 1;
        err = cudaMemsetAsync(dev, 0, sizeof(u32) * 4, st);
        if (err != cudaSuccess) return err;
        err = cudaMemsetAsync(nf, 0, sizeof(u32) * (size_t)(nch_bound + 1), st);
        if (err != cudaSuccess) return err;
        k_seg_chunks<<<grid_n(ng, T), T, 0, st>>>(cnt, ng, cpg, dev + 1);
        err = scan_u32_exclusive(st, cpg, co, ng + 1, stmp, dev);    // co[ng] = chunks, dev[0] = chunks
        if (err != cudaSuccess) return err;
        const unsigned grid = (unsigned)std::min<long long>(nch_bound, cta);
        k_seg_chunk_map<<<grid_n(ng, T), T, 0, st>>>(co, ng, cmap);
        k_chunk_front<<<grid, kChunkThreads, kChunkSmem, st>>>(X, cnt, goff, co, cmap, fin, dev, nf);
        err = scan_u32_exclusive(st, nf, out, nch_bound + 1, stmp, dev + 2);
        if (err != cudaSuccess) return err;
        k_chunk_compact<<<grid, 128, 0, st>>>(X, goff, co, cmap, dev, nf, out, Y);
        rs->launches += 8;
        rs->passes++;
        u32 h[3] = {0, 0, 0};
        err = cudaMemcpyAsync(h, dev, sizeof(h), cudaMemcpyDeviceToHost, st);
        if (err != cudaSuccess) return err;
        err = cudaStreamSynchronize(st);
        if (err != cudaSuccess) return err;
        if (!h[1]) {                              // every group fitted one chunk: Y holds the frontier
            const u32 tot = h[2];
            if (Y.t != A.t) {
                k_seg_copy<<<grid_n(tot, T), T, 0, st>>>(Y, tot, A);
                rs->launches++;
            }
            *n_out = tot;
            return cudaGetLastError();
        }
        k_seg_regroup<<<grid_n(ng, T), T, 0, st>>>(co, ng, out, cnt, goff, fin);
        rs->launches++;
        n_cur = h[2];
        std::swap(X, Y);
    }
}

}  // namespace mist
