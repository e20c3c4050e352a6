// mist_frontier.cu -- a9 segmented radix sort on (group, t) and a10 segmented
// running-min frontier scan (PAPER.md line 660 / Eq. 3: the per-(stage, l,
// mesh) Pareto frontier; exact dominance definition O10 in DESIGN.md).
//
// Frontier rule on candidates sorted by (group, t): within a group, a run of
// equal t keeps its minimum (y, idx); the run is on the frontier iff that
// minimum y is strictly below the minimum y of every earlier run of the
// group.  Both the run minimum and the "earlier runs" minimum come out of ONE
// segmented scan whose state (pre, cur) is closed under concatenation:
//   pre = min y over elements before the last run head, cur = argmin (y, idx)
//   from the last run head on; group heads reset the state.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <math_constants.h>
#include <stdint.h>

#include <atomic>

#include "mist_internal.h"

namespace mist {

typedef unsigned long long u64;
typedef unsigned u32;

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
// device-wide exclusive scan of u32 (reduce -> scan tile sums -> downsweep)
// ---------------------------------------------------------------------------
constexpr int kScanItems = 8;
constexpr int kScanTile = kThreads * kScanItems;

__device__ __forceinline__ u32 block_excl_sum(u32 v, u32* warp_tot, u32& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    u32 x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
        u32 s = lane < kThreads / 32 ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u32 y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < kThreads / 32) warp_tot[lane] = s;
    }
    __syncthreads();
    total = warp_tot[kThreads / 32 - 1];
    const u32 before = (w ? warp_tot[w - 1] : 0) + x - v;
    __syncthreads();
    return before;
}

__global__ void k_scan_reduce(const u32* __restrict__ in, long long n, u32* __restrict__ tile_sum) {
    __shared__ u32 wt[32];
    const long long base = (long long)blockIdx.x * kScanTile;
    u32 s = 0;
    for (int j = 0; j < kScanItems; ++j) {
        long long i = base + (long long)j * kThreads + threadIdx.x;
        if (i < n) s += in[i];
    }
    u32 total;
    block_excl_sum(s, wt, total);
    if (threadIdx.x == 0) tile_sum[blockIdx.x] = total;
}

__global__ void k_scan_tiles(u32* __restrict__ tile_sum, long long ntiles, u32* __restrict__ grand) {
    __shared__ u32 wt[32];
    u32 carry = 0;
    for (long long b = 0; b < ntiles; b += kThreads) {
        const long long i = b + threadIdx.x;
        const u32 v = i < ntiles ? tile_sum[i] : 0;
        u32 total;
        const u32 ex = block_excl_sum(v, wt, total);
        if (i < ntiles) tile_sum[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0 && grand) *grand = carry;
}

__global__ void k_scan_down(const u32* __restrict__ in, long long n, const u32* __restrict__ tile_off,
                            u32* __restrict__ out) {
    __shared__ u32 wt[32];
    const long long base = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanItems;
    u32 v[kScanItems];
    u32 s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const long long i = base + j;
        v[j] = i < n ? in[i] : 0;
        s += v[j];
    }
    u32 total;
    u32 run = block_excl_sum(s, wt, total) + tile_off[blockIdx.x];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const long long i = base + j;
        if (i < n) out[i] = run;
        run += v[j];
    }
}

// Small arrays (the per-group and per-chunk tables of a reduction): one CTA walks
// the array in tiles of kScanTile with a running carry -- one launch instead of three.
__global__ void k_scan_small(const u32* __restrict__ in, long long n, u32* __restrict__ out,
                             u32* __restrict__ grand) {
    __shared__ u32 wt[32];
    u32 carry = 0;
    for (long long base = 0; base < n; base += kScanTile) {
        const long long b0 = base + (long long)threadIdx.x * kScanItems;
        u32 v[kScanItems];
        u32 s = 0;
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {
            v[j] = b0 + j < n ? in[b0 + j] : 0u;
            s += v[j];
        }
        u32 total;
        u32 run = block_excl_sum(s, wt, total) + carry;
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {
            if (b0 + j < n) out[b0 + j] = run;
            run += v[j];
        }
        carry += total;
    }
    if (threadIdx.x == 0 && grand) *grand = carry;
}

// NOTE k_scan_reduce sums a tile in striped order and k_scan_down in blocked
// order; both cover exactly the same index range [tile*kScanTile, +kScanTile).
cudaError_t scan_u32_exclusive(cudaStream_t st, const u32* in, u32* out, long long n, u32* tmp,
                               u32* grand_total) {
    if (n <= 0) return cudaSuccess;
    if (n <= 16 * kScanTile) {
        k_scan_small<<<1, kThreads, 0, st>>>(in, n, out, grand_total);
        return cudaGetLastError();
    }
    const long long ntiles = (n + kScanTile - 1) / kScanTile;
    k_scan_reduce<<<(unsigned)ntiles, kThreads, 0, st>>>(in, n, tmp);
    k_scan_tiles<<<1, kThreads, 0, st>>>(tmp, ntiles, grand_total);
    k_scan_down<<<(unsigned)ntiles, kThreads, 0, st>>>(in, n, tmp, out);
    return cudaGetLastError();
}

long long scan_tmp_words(long long n) { return (n + kScanTile - 1) / kScanTile + 1; }

// ---------------------------------------------------------------------------
// a9: LSD radix sort of (group, t) with u32 payload, 8-bit digits.
// digit positions: 0..7 = bytes of t (as u64 bits; t >= 0 so the bit pattern
// orders like the value), 8..10 = bytes of the group id.
// ---------------------------------------------------------------------------
constexpr int kSortItems = 8;
constexpr int kSortTile = kThreads * kSortItems;
constexpr int kDigitPositions = 11;

__device__ __forceinline__ u32 digit_of(u64 t, u32 g, int pos) {
    return pos < 8 ? (u32)(t >> (8 * pos)) & 255u : (g >> (8 * (pos - 8))) & 255u;
}

__global__ void k_digit_hist(const u64* __restrict__ t, const u32* __restrict__ g, long long n,
                             u32* __restrict__ hist /*[11][256]*/) {
    __shared__ u32 h[kDigitPositions][256];
    for (int i = threadIdx.x; i < kDigitPositions * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const u64 tv = t[i];
        const u32 gv = g[i];
#pragma unroll
        for (int p = 0; p < kDigitPositions; ++p) atomicAdd(&h[p][digit_of(tv, gv, p)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kDigitPositions * 256; i += blockDim.x) {
        const u32 v = (&h[0][0])[i];
        if (v) atomicAdd(hist + i, v);
    }
}

__global__ void k_radix_upsweep(const u64* __restrict__ t, const u32* __restrict__ g, long long n,
                                int pos, long long ntiles, u32* __restrict__ block_hist) {
    __shared__ u32 h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const long long base = (long long)blockIdx.x * kSortTile;
    u32 dg[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {            // issue every load of the tile first (MLP)
        const long long i = base + (long long)j * kThreads + threadIdx.x;
        dg[j] = i < n ? digit_of(pos < 8 ? t[i] : 0ull, pos < 8 ? 0u : g[i], pos) : 256u;
    }
#pragma unroll
    for (int j = 0; j < kSortItems; ++j)
        if (dg[j] < 256u) atomicAdd(&h[dg[j]], 1u);
    __syncthreads();
    block_hist[(long long)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter of one 2048-key tile: (1) each warp ranks its contiguous
// 256-key sub-tile with __match_any_sync and warp-private digit counters,
// (2) one block scan turns per-warp counts into tile-local positions, (3) the
// tile is reordered by digit in shared memory, (4) threads stream it out so
// consecutive threads write consecutive addresses of each digit bucket.
__global__ void __launch_bounds__(kThreads)
k_radix_scatter(const u64* __restrict__ t_in, const u32* __restrict__ g_in,
                const u32* __restrict__ v_in, u64* __restrict__ t_out,
                u32* __restrict__ g_out, u32* __restrict__ v_out, long long n, int pos,
                long long ntiles, const u32* __restrict__ block_off) {
    constexpr int W = kThreads / 32;
    __shared__ u32 s_cnt[W][256];        // per-warp digit counts, then per-warp tile offsets
    __shared__ u32 s_dstart[256];        // tile-local start of each digit bucket
    __shared__ u32 s_goff[256];          // global start of this tile's part of each bucket
    __shared__ u32 s_wt[32];
    __shared__ u64 sk_t[kSortTile];
    __shared__ u32 sk_g[kSortTile], sk_v[kSortTile];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int i = 0; i < W; ++i) s_cnt[i][tid] = 0;
    s_goff[tid] = block_off[(long long)tid * ntiles + blockIdx.x];
    __syncthreads();
    const long long base = (long long)blockIdx.x * kSortTile;
    const long long wbase = base + (long long)w * 32 * kSortItems;
    u64 tv[kSortItems];
    u32 gv[kSortItems], vv[kSortItems], dg[kSortItems], rk[kSortItems];
    const u32 lt = (1u << lane) - 1;
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {            // issue every load of the sub-tile first (MLP)
        const long long i = wbase + j * 32 + lane;
        const bool valid = i < n;
        tv[j] = valid ? t_in[i] : 0ull;
        gv[j] = valid ? g_in[i] : 0u;
        vv[j] = valid ? v_in[i] : 0u;
    }
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const bool valid = wbase + j * 32 + lane < n;
        dg[j] = valid ? digit_of(tv[j], gv[j], pos) : 0xffffffffu;
        const u32 peers = __match_any_sync(0xffffffffu, dg[j]);
        const u32 before = valid ? s_cnt[w][dg[j]] : 0u;
        rk[j] = before + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers & lt) == 0) s_cnt[w][dg[j]] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {   // thread tid owns digit tid: per-warp prefix and the digit's tile total
        u32 run = 0;
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const u32 c = s_cnt[k][tid];
            s_cnt[k][tid] = run;
            run += c;
        }
        u32 total;
        s_dstart[tid] = block_excl_sum(run, s_wt, total);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        if (dg[j] == 0xffffffffu) continue;
        const u32 o = s_dstart[dg[j]] + s_cnt[w][dg[j]] + rk[j];
        sk_t[o] = tv[j]; sk_g[o] = gv[j]; sk_v[o] = vv[j];
    }
    __syncthreads();
    const int tile_n = (int)min((long long)kSortTile, n - base);
    for (int o = tid; o < tile_n; o += kThreads) {
        const u64 t = sk_t[o];
        const u32 g = sk_g[o];
        const u32 d = digit_of(t, g, pos);
        const u32 gp = s_goff[d] + (u32)o - s_dstart[d];
        t_out[gp] = t; g_out[gp] = g; v_out[gp] = sk_v[o];
    }
}

// Persistent variant of k_radix_scatter with TMA bulk loads (sm_100a): each CTA
// walks tiles blockIdx.x, blockIdx.x + gridDim.x, ...; while it ranks and writes
// tile i, the TMA engine already streams tile i+1 (t, g, v: three contiguous
// cp.async.bulk copies completing on an mbarrier) into the other smem stage, and
// the tile's 256 bucket offsets are prefetched one tile ahead.  Same ranking and
// output as k_radix_scatter.  A partial last tile is loaded with plain loads.
struct ScatterStage {
    u64 t[kSortTile];
    u32 g[kSortTile], v[kSortTile];
};

__device__ __forceinline__ u32 smem_u32(const void* p) {
    return (u32)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
    const u32 a = smem_u32(bar);
    asm volatile("{\n .reg .pred P;\n WAIT_%=:\n"
                 " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
                 " @!P bra WAIT_%=;\n}\n" :: "r"(a), "r"(parity) : "memory");
}

__global__ void __launch_bounds__(kThreads, 2)
k_radix_scatter_tma(const u64* __restrict__ t_in, const u32* __restrict__ g_in,
                    const u32* __restrict__ v_in, u64* __restrict__ t_out,
                    u32* __restrict__ g_out, u32* __restrict__ v_out, long long n, int pos,
                    long long ntiles, const u32* __restrict__ block_off) {
    constexpr int W = kThreads / 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    ScatterStage* stage = reinterpret_cast<ScatterStage*>(smem_raw);          // [2]
    ScatterStage* sk = stage + 2;                                              // reordered tile
    u32 (*s_cnt)[256] = reinterpret_cast<u32 (*)[256]>(sk + 1);                // [W][256]
    u32* s_dstart = &s_cnt[W][0];
    u32* s_goff = s_dstart + 256;
    u32* s_wt = s_goff + 256;
    u64* bar = reinterpret_cast<u64*>(s_wt + 32);                              // [2]
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const long long full_tiles = n / kSortTile;
    auto issue = [&](long long tile, int st) {   // thread 0: TMA the whole tile into stage st
        const long long b = tile * kSortTile;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
                     :: "r"(smem_u32(&bar[st])), "r"((u32)(kSortTile * 16)) : "memory");
        bulk_g2s(stage[st].t, t_in + b, kSortTile * 8, &bar[st]);
        bulk_g2s(stage[st].g, g_in + b, kSortTile * 4, &bar[st]);
        bulk_g2s(stage[st].v, v_in + b, kSortTile * 4, &bar[st]);
    };
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(smem_u32(&bar[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(smem_u32(&bar[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    long long tile = blockIdx.x;
    if (tid == 0 && tile < full_tiles) issue(tile, 0);
    u32 goff_next = tile < ntiles ? block_off[(long long)tid * ntiles + tile] : 0u;
    const u32 lt = (1u << lane) - 1;
    for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it & 1;
        const long long base = tile * kSortTile;
        const long long next = tile + gridDim.x;
        for (int i = 0; i < W; ++i) s_cnt[i][tid] = 0;
        s_goff[tid] = goff_next;
        if (next < ntiles) goff_next = block_off[(long long)tid * ntiles + next];   // one tile ahead
        if (tid == 0 && next < full_tiles) {
            // stage st^1 was last read before the previous iteration's closing barrier
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(next, st ^ 1);
        }
        const bool full = tile < full_tiles;
        if (full) {
            mbar_wait(&bar[st], (u32)(it >> 1) & 1u);   // the (it/2)-th use of stage st
        } else {   // partial last tile: plain loads into the stage
            for (int o = tid; o < kSortTile; o += kThreads) {
                const long long i = base + o;
                if (i < n) { stage[st].t[o] = t_in[i]; stage[st].g[o] = g_in[i]; stage[st].v[o] = v_in[i]; }
            }
        }
        __syncthreads();
        const ScatterStage& S = stage[st];
        const int wbase = w * 32 * kSortItems;
        u64 tv[kSortItems];
        u32 gv[kSortItems], vv[kSortItems], dg[kSortItems], rk[kSortItems];
#pragma unroll
        for (int j = 0; j < kSortItems; ++j) {
            const int o = wbase + j * 32 + lane;
            const bool valid = base + o < n;
            tv[j] = S.t[o]; gv[j] = S.g[o]; vv[j] = S.v[o];
            dg[j] = valid ? digit_of(tv[j], gv[j], pos) : 0xffffffffu;
            const u32 peers = __match_any_sync(0xffffffffu, dg[j]);
            const u32 before = valid ? s_cnt[w][dg[j]] : 0u;
            rk[j] = before + __popc(peers & lt);
            __syncwarp();
            if (valid && (peers & lt) == 0) s_cnt[w][dg[j]] = before + __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        {
            u32 run = 0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const u32 c = s_cnt[k][tid];
                s_cnt[k][tid] = run;
                run += c;
            }
            u32 total;
            s_dstart[tid] = block_excl_sum(run, s_wt, total);
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kSortItems; ++j) {
            if (dg[j] == 0xffffffffu) continue;
            const u32 o = s_dstart[dg[j]] + s_cnt[w][dg[j]] + rk[j];
            sk->t[o] = tv[j]; sk->g[o] = gv[j]; sk->v[o] = vv[j];
        }
        __syncthreads();
        const int tile_n = (int)min((long long)kSortTile, n - base);
        for (int o = tid; o < tile_n; o += kThreads) {
            const u64 t = sk->t[o];
            const u32 g = sk->g[o];
            const u32 d = digit_of(t, g, pos);
            const u32 gp = s_goff[d] + (u32)o - s_dstart[d];
            t_out[gp] = t; g_out[gp] = g; v_out[gp] = sk->v[o];
        }
        __syncthreads();
    }
}

static size_t scatter_tma_smem() {
    return 3 * sizeof(ScatterStage) + (kThreads / 32 + 2) * 256 * sizeof(u32) + 32 * sizeof(u32) + 2 * sizeof(u64);
}

// MIST_SCATTER=plain selects k_radix_scatter (A/B knob); default: the TMA-pipelined kernel.
static bool scatter_tma() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MIST_SCATTER");
        v = (e && !strcmp(e, "plain")) ? 0 : 1;
    }
    return v == 1;
}

// ---------------------------------------------------------------------------
// a10: segmented frontier scan
// ---------------------------------------------------------------------------
struct FS {
    u32 gh, hh;      // contains a group head / a run head
    double pre;      // min y before the last run head (within the last group)
    double cy;       // argmin (y, idx) from the last run head on
    u64 cidx;
    u32 cpos;
};

__device__ __forceinline__ FS fs_empty() {
    FS s; s.gh = 0; s.hh = 0; s.pre = CUDART_INF; s.cy = CUDART_INF; s.cidx = ~0ull; s.cpos = 0;
    return s;
}

__device__ __forceinline__ FS fs_combine(const FS& A, const FS& B) {
    if (B.gh) return B;
    FS R;
    R.gh = A.gh;
    if (B.hh) {
        R.hh = 1;
        R.pre = fmin(fmin(A.pre, A.cy), B.pre);
        R.cy = B.cy; R.cidx = B.cidx; R.cpos = B.cpos;
    } else {
        R.hh = A.hh;
        R.pre = A.pre;
        const bool b_less = B.cy < A.cy || (B.cy == A.cy && B.cidx < A.cidx);
        R.cy = b_less ? B.cy : A.cy;
        R.cidx = b_less ? B.cidx : A.cidx;
        R.cpos = b_less ? B.cpos : A.cpos;
    }
    return R;
}

__device__ __forceinline__ FS fs_shfl_up(const FS& s, int o) {
    FS r;
    r.gh = __shfl_up_sync(0xffffffffu, s.gh, o);
    r.hh = __shfl_up_sync(0xffffffffu, s.hh, o);
    r.pre = __shfl_up_sync(0xffffffffu, s.pre, o);
    r.cy = __shfl_up_sync(0xffffffffu, s.cy, o);
    r.cidx = __shfl_up_sync(0xffffffffu, s.cidx, o);
    r.cpos = __shfl_up_sync(0xffffffffu, s.cpos, o);
    return r;
}

// exclusive block scan of FS (returns the prefix of everything before this thread)
__device__ FS block_excl_fs(const FS& v, FS* warp_tot, FS& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    FS x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        FS y = fs_shfl_up(x, o);
        if (lane >= o) x = fs_combine(y, x);
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
        FS s = lane < kThreads / 32 ? warp_tot[lane] : fs_empty();
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            FS y = fs_shfl_up(s, o);
            if (lane >= o) s = fs_combine(y, s);
        }
        if (lane < kThreads / 32) warp_tot[lane] = s;
    }
    __syncthreads();
    total = warp_tot[kThreads / 32 - 1];
    FS excl_in_warp = fs_shfl_up(x, 1);
    if (lane == 0) excl_in_warp = fs_empty();
    const FS before = w ? fs_combine(warp_tot[w - 1], excl_in_warp) : excl_in_warp;
    __syncthreads();
    return before;
}

constexpr int kFsItems = 4;
constexpr int kFsTile = kThreads * kFsItems;

struct FsIn {
    const u64* t;      // sorted t bits
    const u32* g;      // sorted group
    const u32* v;      // payload (candidate position)
    const double* y;   // y in sorted order (gathered once, k_gather_sorted)
    const u64* idx;    // idx in sorted order
    long long n;
};

// one random-access pass: y and idx into sorted order, so the scans read coalesced
__global__ void k_gather_sorted(const u32* __restrict__ v, long long n, const double* __restrict__ y,
                                const u64* __restrict__ idx, double* __restrict__ ys, u64* __restrict__ xs) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const u32 p = v[i];
        ys[i] = __ldg(y + p);
        xs[i] = __ldg(idx + p);
    }
}

__device__ __forceinline__ FS fs_element(const FsIn& in, long long i) {
    FS s;
    const u64 t = in.t[i];
    const u32 g = in.g[i];
    const bool gh = i == 0 || in.g[i - 1] != g;
    const bool hh = gh || in.t[i - 1] != t;
    const u32 p = in.v[i];
    s.gh = gh; s.hh = hh; s.pre = CUDART_INF;
    s.cy = in.y[i]; s.cidx = in.idx[i]; s.cpos = p;
    return s;
}

__global__ void k_fs_reduce(FsIn in, FS* __restrict__ tile_agg) {
    __shared__ FS wt[kThreads / 32];
    const long long base = (long long)blockIdx.x * kFsTile + (long long)threadIdx.x * kFsItems;
    FS acc = fs_empty();
    for (int j = 0; j < kFsItems; ++j) {
        const long long i = base + j;
        if (i < in.n) acc = fs_combine(acc, fs_element(in, i));
    }
    FS total;
    block_excl_fs(acc, wt, total);
    if (threadIdx.x == 0) tile_agg[blockIdx.x] = total;
}

__global__ void k_fs_tiles(FS* __restrict__ tile_agg, long long ntiles) {
    __shared__ FS wt[kThreads / 32];
    FS carry = fs_empty();
    for (long long b = 0; b < ntiles; b += kThreads) {
        const long long i = b + threadIdx.x;
        const FS v = i < ntiles ? tile_agg[i] : fs_empty();
        FS total;
        const FS ex = block_excl_fs(v, wt, total);
        if (i < ntiles) tile_agg[i] = fs_combine(carry, ex);
        carry = fs_combine(carry, total);
    }
}

// flag[i] = 1 iff i is the tail of a frontier run; pick[i] = that run's argmin payload
__global__ void k_fs_down(FsIn in, const FS* __restrict__ tile_pre, u32* __restrict__ flag,
                          u32* __restrict__ pick) {
    __shared__ FS wt[kThreads / 32];
    const long long base = (long long)blockIdx.x * kFsTile + (long long)threadIdx.x * kFsItems;
    FS el[kFsItems];
    FS acc = fs_empty();
#pragma unroll
    for (int j = 0; j < kFsItems; ++j) {
        const long long i = base + j;
        el[j] = i < in.n ? fs_element(in, i) : fs_empty();
        acc = fs_combine(acc, el[j]);
    }
    FS total;
    FS run = fs_combine(tile_pre[blockIdx.x], block_excl_fs(acc, wt, total));
#pragma unroll
    for (int j = 0; j < kFsItems; ++j) {
        const long long i = base + j;
        if (i >= in.n) break;
        run = fs_combine(run, el[j]);
        const bool tail = i == in.n - 1 || in.g[i + 1] != in.g[i] || in.t[i + 1] != in.t[i];
        const bool fr = tail && run.cy < run.pre;
        flag[i] = fr;
        pick[i] = run.cpos;
    }
}

// compact frontier records into the output SoA (sorted by (group, t))
__global__ void k_fs_compact(const u32* __restrict__ flag, const u32* __restrict__ pick,
                             const u32* __restrict__ outpos, long long n, CandBuf src,
                             CandBuf dst) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        if (!flag[i]) continue;
        const u32 p = pick[i], o = outpos[i];
        dst.t[o] = src.t[p]; dst.y[o] = src.y[p]; dst.mem[o] = src.mem[p];
        dst.idx[o] = src.idx[p]; dst.group[o] = src.group[p];
    }
}

__global__ void k_prepare_keys(CandBuf c, long long n, u64* __restrict__ t, u32* __restrict__ g,
                               u32* __restrict__ v) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        t[i] = __double_as_longlong(c.t[i]);
        g[i] = c.group[i];
        v[i] = (u32)i;
    }
}

__global__ void k_copy_cand(CandBuf src, CandBuf dst, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        dst.t[i] = src.t[i]; dst.y[i] = src.y[i]; dst.mem[i] = src.mem[i];
        dst.idx[i] = src.idx[i]; dst.group[i] = src.group[i];
    }
}

__global__ void k_group_offsets(const u32* __restrict__ g, long long n, int ng, int64_t* __restrict__ off) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q <= ng;
         q += (long long)gridDim.x * blockDim.x) {
        long long lo = 0, hi = n;   // first position with g >= q
        while (lo < hi) {
            const long long mid = (lo + hi) >> 1;
            if (g[mid] < (u32)q) lo = mid + 1; else hi = mid;
        }
        off[q] = lo;
    }
}

__global__ void k_pack_points(CandBuf c, long long n, mist_point_t* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        mist_point_t p;
        p.idx = c.idx[i]; p.t = c.t[i]; p.y = c.y[i]; p.mem = c.mem[i];
        out[i] = p;
    }
}

static unsigned grid_for(long long n, int threads, int max_blocks = 148 * 8) {
    long long b = (n + threads - 1) / threads;
    if (b > max_blocks) b = max_blocks;
    if (b < 1) b = 1;
    return (unsigned)b;
}

// ---------------------------------------------------------------------------
// host: reduce candidates [0, n) of `cand` to their exact frontier, in place
// (cand[0, *n_out) afterwards, sorted by (group, t)).
// ---------------------------------------------------------------------------

cudaError_t frontier_reduce(cudaStream_t st, CandBuf cand, long long n, SortScratch& S, u32* scan_tmp,
                            long long* n_out, ReduceStats* rs) {
    cudaError_t err;
    if (n == 0) { *n_out = 0; return cudaSuccess; }
    const int T = kThreads;
    k_prepare_keys<<<grid_for(n, T), T, 0, st>>>(cand, n, S.key_t[0], S.key_g[0], S.val[0]);
    rs->launches++;
    // global digit histograms for pass skipping
    cudaMemsetAsync(S.digit_hist, 0, sizeof(u32) * kDigitPositions * 256, st);
    k_digit_hist<<<grid_for(n, T, 148 * 4), T, 0, st>>>(S.key_t[0], S.key_g[0], n, S.digit_hist);
    rs->launches++;
    u32 h_hist[kDigitPositions * 256];
    err = cudaMemcpyAsync(h_hist, S.digit_hist, sizeof(h_hist), cudaMemcpyDeviceToHost, st);
    if (err != cudaSuccess) return err;
    err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) return err;
    const long long ntiles = (n + kSortTile - 1) / kSortTile;
    int cur = 0;
    for (int pos = 0; pos < kDigitPositions; ++pos) {
        bool trivial = false;
        for (int d = 0; d < 256; ++d)
            if ((long long)h_hist[pos * 256 + d] == n) { trivial = true; break; }
        if (trivial) continue;   // digit skipping: every key has the same digit
        k_radix_upsweep<<<(unsigned)ntiles, T, 0, st>>>(S.key_t[cur], S.key_g[cur], n, pos, ntiles,
                                                         S.block_hist);
        err = scan_u32_exclusive(st, S.block_hist, S.block_hist, 256 * ntiles, scan_tmp + 8, nullptr);
        if (err != cudaSuccess) return err;
        const bool aligned = ((reinterpret_cast<uintptr_t>(S.key_t[cur]) | reinterpret_cast<uintptr_t>(S.key_g[cur]) |
                               reinterpret_cast<uintptr_t>(S.val[cur])) & 15) == 0;
        if (scatter_tma() && aligned) {
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            static std::atomic<unsigned long long> attr{0};   // the attribute is per device: one bit per device
            if (dev >= 64 || !((attr.load() >> dev) & 1ull)) {
                err = cudaFuncSetAttribute(k_radix_scatter_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)scatter_tma_smem());
                if (err != cudaSuccess) return err;
                if (dev < 64) attr.fetch_or(1ull << dev);
            }
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            long long grid = std::min<long long>(ntiles, 2LL * sms);
            k_radix_scatter_tma<<<(unsigned)grid, T, scatter_tma_smem(), st>>>(
                S.key_t[cur], S.key_g[cur], S.val[cur], S.key_t[cur ^ 1], S.key_g[cur ^ 1], S.val[cur ^ 1], n, pos,
                ntiles, S.block_hist);
        } else {
            k_radix_scatter<<<(unsigned)ntiles, T, 0, st>>>(S.key_t[cur], S.key_g[cur], S.val[cur],
                                                             S.key_t[cur ^ 1], S.key_g[cur ^ 1],
                                                             S.val[cur ^ 1], n, pos, ntiles, S.block_hist);
        }
        rs->launches += 5;
        rs->passes++;
        cur ^= 1;
    }
    // segmented frontier scan over the sorted keys
    k_gather_sorted<<<grid_for(n, T), T, 0, st>>>(S.val[cur], n, cand.y, cand.idx, S.gy, S.gidx);
    rs->launches++;
    FsIn in;
    in.t = S.key_t[cur]; in.g = S.key_g[cur]; in.v = S.val[cur];
    in.y = S.gy; in.idx = S.gidx; in.n = n;
    const long long ftiles = (n + kFsTile - 1) / kFsTile;
    FS* tile_agg = reinterpret_cast<FS*>(S.block_hist);   // reuse (ntiles*256 u32 >= ftiles FS)
    u32* flag = S.val[cur ^ 1];
    u32* pick = S.key_g[cur ^ 1];
    u32* outpos = reinterpret_cast<u32*>(S.key_t[cur ^ 1]);
    k_fs_reduce<<<(unsigned)ftiles, T, 0, st>>>(in, tile_agg);
    k_fs_tiles<<<1, T, 0, st>>>(tile_agg, ftiles);
    k_fs_down<<<(unsigned)ftiles, T, 0, st>>>(in, tile_agg, flag, pick);
    // scan_tmp[0] holds the grand total, tile sums start at scan_tmp + 8
    err = scan_u32_exclusive(st, flag, outpos, n, scan_tmp + 8, scan_tmp);
    if (err != cudaSuccess) return err;
    u32 h_total = 0;
    err = cudaMemcpyAsync(&h_total, scan_tmp, sizeof(u32), cudaMemcpyDeviceToHost, st);
    if (err != cudaSuccess) return err;
    err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) return err;
    const long long nf = h_total;
    // destination: the candidate buffer beyond n (the caller keeps 2n <= cap), then move to [0, nf)
    if (2 * n > cand.cap) return cudaErrorInvalidValue;
    CandBuf dst;
    dst.t = cand.t + n; dst.y = cand.y + n; dst.mem = cand.mem + n; dst.idx = cand.idx + n;
    dst.group = cand.group + n;
    k_fs_compact<<<grid_for(n, T), T, 0, st>>>(flag, pick, outpos, n, cand, dst);
    k_copy_cand<<<grid_for(nf, T), T, 0, st>>>(dst, cand, nf);
    rs->launches += 3 + 3 + 2;
    *n_out = nf;
    return cudaGetLastError();
}

cudaError_t frontier_group_offsets(cudaStream_t st, const u32* g, long long n, int ng, int64_t* off) {
    k_group_offsets<<<grid_for(ng + 1, kThreads), kThreads, 0, st>>>(g, n, ng, off);
    return cudaGetLastError();
}

cudaError_t pack_points(cudaStream_t st, CandBuf c, long long n, mist_point_t* out) {
    if (n <= 0) return cudaSuccess;
    k_pack_points<<<grid_for(n, kThreads), kThreads, 0, st>>>(c, n, out);
    return cudaGetLastError();
}

}  // namespace mist
