// mist_enum.cpp -- a1 enumerate_space (host, integer) and problem packing.
//
// Paper: "given a model, a global batch size B, and a device mesh (N, M)"
// (PAPER.md line 625); intra-stage tuning runs "for all possible pipeline
// partitioning candidates" (line 628) for every gradient-accumulation step
// G, which is independent and parallelisable (line 879).  Groups are the keys
// of IntraStagePareto(i, l_i, (n_i, m_i)) (Eq. 3) with the stage
// index i replaced by what memory/time actually read from it: first, last and
// the 1F1B in-flight count w = min(G, S - i + 1) (readings O2, L33,
// L34).  Splits follow b * DP * G = B (L18), TP = 2^j <= m dividing heads and
// kv heads (L27).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>

#include "mist_internal.h"

namespace mist {

static bool model_ok(const mist_model_t* m) {
    if (!m) return false;
    if (m->num_layers < 1 || m->hidden < 1 || m->heads < 1 || m->kv_heads < 1 || m->ffn < 1 ||
        m->vocab < 1 || m->seq < 1 || m->elem_bytes < 1)
        return false;
    if (((int64_t)m->kv_heads * m->hidden) % m->heads != 0) return false;
    if (m->gated_mlp < 0 || m->gated_mlp > 1 || m->parallel_attn < 0 || m->parallel_attn > 1 ||
        m->flash_attn < 0 || m->flash_attn > 1 || m->norm_vecs_per_layer < 0)
        return false;
    return true;
}

int coef_row(const mist_coeffs_t* c, int b, int tp) {
    int ib = -1, it = -1;
    for (int i = 0; i < c->n_b; ++i)
        if (c->b_values[i] == b) { ib = i; break; }
    for (int i = 0; i < c->n_tp; ++i)
        if (c->tp_values[i] == tp) { it = i; break; }
    return (ib < 0 || it < 0) ? -1 : ib * c->n_tp + it;
}

mist_status_t validate(const mist_model_t* model, int64_t B, const mist_mesh_t* mesh,
                       const mist_space_t* space, const mist_coeffs_t* coeffs, std::string* why) {
    if (!model_ok(model)) { *why = "invalid model shape"; return MIST_ERR_INVALID_ARG; }
    if (B < 1 || B > (1LL << 30)) { *why = "global batch out of range"; return MIST_ERR_INVALID_ARG; }
    if (!mesh || mesh->nodes < 1 || mesh->gpus_per_node < 1 ||
        (int64_t)mesh->nodes * mesh->gpus_per_node > 4096) {
        *why = "invalid mesh"; return MIST_ERR_INVALID_ARG;
    }
    if (mesh->mem_budget_bytes <= 0 || mesh->mem_budget_bytes >= (1LL << 46)) {
        *why = "memory budget out of range"; return MIST_ERR_INVALID_ARG;
    }
    if (space && (double)mesh->mem_budget_bytes * space->offload_steps * mesh->nodes *
                         mesh->gpus_per_node >= 9007199254740992.0) {
        // D * Mem_Budget must be an exact double (O9 exactness argument)
        *why = "budget * Q * N * M must be < 2^53"; return MIST_ERR_INVALID_ARG;
    }
    if (!space || space->offload_steps < 1 || space->offload_steps > 1000 ||
        (space->zero_mask & 0xF) == 0 || (space->zero_mask & ~0xF) || space->max_stages < 0 ||
        space->n_grad_accum < 0 || (space->n_grad_accum > 0 && !space->grad_accum) ||
        (space->ckpt_ends_only != 0 && space->ckpt_ends_only != 1) || (space->offload_off & ~0xF)) {
        *why = "invalid search space options"; return MIST_ERR_INVALID_ARG;
    }
    if (coeffs) {
        if (coeffs->n_b < 1 || coeffs->n_tp < 1 || !coeffs->b_values || !coeffs->tp_values ||
            !coeffs->t_layer_fwd || !coeffs->t_layer_bwd || !coeffs->t_emb_fwd ||
            !coeffs->t_emb_bwd || !coeffs->t_head_fwd || !coeffs->t_head_bwd) {
            *why = "incomplete coefficient tables"; return MIST_ERR_INVALID_ARG;
        }
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 2; ++j)
                if (!(coeffs->bw[i][j] > 0) || !(coeffs->lat[i][j] >= 0)) {
                    *why = "bandwidth must be > 0 and latency >= 0"; return MIST_ERR_INVALID_ARG;
                }
        if (!(coeffs->bw_h2d > 0) || !(coeffs->bw_d2h > 0)) {
            *why = "PCIe bandwidth must be > 0"; return MIST_ERR_INVALID_ARG;
        }
        for (int mask = 0; mask < 16; ++mask) {
            if (__builtin_popcount(mask) < 2) continue;
            for (int j = 0; j < 4; ++j)
                if ((mask >> j & 1) && !(coeffs->intf[mask][j] >= 1.0 && coeffs->intf[mask][j] < 1e6)) {
                    *why = "interference factors must be >= 1"; return MIST_ERR_INVALID_ARG;
                }
        }
    }
    return MIST_OK;
}

// Build the per-problem kernel parameter block.
void pack_problem(const mist_model_t* m, int64_t B, const mist_mesh_t* mesh,
                  const mist_space_t* sp, const mist_coeffs_t* c, int ykey, DevProblem* P) {
    std::memset(P, 0, sizeof(*P));
    P->L = m->num_layers; P->h = m->hidden; P->a = m->heads; P->k = m->kv_heads; P->f = m->ffn;
    P->V = m->vocab; P->s = m->seq; P->e = m->elem_bytes; P->g = m->gated_mlp;
    P->p = m->parallel_attn; P->fl = m->flash_attn; P->nrm = m->norm_vecs_per_layer;
    P->N = mesh->nodes; P->M = mesh->gpus_per_node;
    P->Q = sp->offload_steps; P->Q1 = sp->offload_steps + 1;
    P->nz = 0;
    for (int z = 0; z < 4; ++z)
        if (sp->zero_mask >> z & 1) P->zlev[P->nz++] = z;
    P->n_b = c->n_b; P->n_tp = c->n_tp;
    P->ykey = ykey;
    P->ckpt_ends = sp->ckpt_ends_only;
    for (int r = 0; r < 4; ++r) P->kmax[r] = (sp->offload_off >> r & 1) ? 0 : sp->offload_steps;
    P->B = B;
    P->mem_budget = mesh->mem_budget_bytes;
    std::memcpy(P->bw, c->bw, sizeof(P->bw));
    std::memcpy(P->lat, c->lat, sizeof(P->lat));
    P->bw_h2d = c->bw_h2d; P->bw_d2h = c->bw_d2h;
    int unit = 1;
    for (int mask = 0; mask < 16; ++mask)
        for (int j = 0; j < 4; ++j) {
            bool member = __builtin_popcount(mask) >= 2 && (mask >> j & 1);
            double f = member ? c->intf[mask][j] : 1.0;
            P->F[mask][j] = f;
            P->IF[mask][j] = 1.0 / f;
            if (member && f != 1.0) unit = 0;
        }
    P->unit_factors = unit;
}

}  // namespace mist

using namespace mist;

extern "C" mist_status_t mist_enumerate_space(const mist_model_t* model, int64_t global_batch,
                                              const mist_mesh_t* mesh, const mist_space_t* space,
                                              const mist_coeffs_t* coeffs_or_null,
                                              mist_group_t* groups, int64_t groups_cap,
                                              int64_t* n_groups, uint64_t* n_configs) {
    std::string why;
    if (!n_groups || !n_configs) return MIST_ERR_INVALID_ARG;
    mist_status_t st = validate(model, global_batch, mesh, space, coeffs_or_null, &why);
    if (st != MIST_OK) return st;
    const int L = model->num_layers, N = mesh->nodes, M = mesh->gpus_per_node;
    const int devices = N * M;
    const int64_t B = global_batch;

    // gradient accumulation steps
    std::vector<int> Gs;
    if (space->n_grad_accum > 0) {
        Gs.assign(space->grad_accum, space->grad_accum + space->n_grad_accum);
        for (int G : Gs)
            if (G < 1) return MIST_ERR_INVALID_ARG;
        std::sort(Gs.begin(), Gs.end());
        Gs.erase(std::unique(Gs.begin(), Gs.end()), Gs.end());
    } else {
        for (int64_t d = 1; d * d <= B; ++d)
            if (B % d == 0) {
                Gs.push_back((int)d);
                if (d != B / d) Gs.push_back((int)(B / d));
            }
        std::sort(Gs.begin(), Gs.end());
    }

    // submesh shapes (1, 2^j | M) and (n >= 2, M)
    std::vector<std::array<int, 2>> shapes;
    for (int j = 0; (1 << j) <= M; ++j)
        if (M % (1 << j) == 0) shapes.push_back({1, 1 << j});
    for (int n = 2; n <= N; ++n) shapes.push_back({n, M});

    int S_max = std::min(L, devices);
    if (space->max_stages > 0) S_max = std::min(S_max, (int)space->max_stages);

    // reach[k][r]: r devices can be covered by exactly k submeshes (L34)
    std::vector<std::vector<uint8_t>> reach(S_max, std::vector<uint8_t>(devices + 1, 0));
    reach[0][0] = 1;
    for (int k = 1; k < S_max; ++k)
        for (int r = 0; r <= devices; ++r) {
            if (!reach[k - 1][r]) continue;
            for (auto& sh : shapes) {
                int nr = r + sh[0] * sh[1];
                if (nr <= devices) reach[k][nr] = 1;
            }
        }

    // keys (G, first, last, w, l, n, m), deduplicated, in lexicographic order.  Stage i
    // of S matters only through its context (first = [i = 1], last = [i = S], w =
    // min(G, S - i + 1)), and for S >= 2 it admits l = 1 .. L - S + 1, so per G the
    // key set is: for every (context, shape) the l range of the smallest valid S,
    // plus the single-stage key (l = L on the full mesh).  Generated directly in
    // sorted order (no sort of the per-(S, i, l) candidates).
    std::vector<std::array<int, 7>> keys;
    const int nsh = (int)shapes.size();   // sorted by (n, m): (1, 2^j) ascending, then (n >= 2, M)
    const int W = S_max + 1;
    std::vector<int> ml((size_t)4 * W * nsh);
    std::vector<uint8_t> single((size_t)nsh);
    auto at = [&](int first, int last, int w, int sh) -> int& {
        return ml[(((size_t)(first * 2 + last) * W + w) * nsh) + sh];
    };
    for (int G : Gs) {
        std::fill(ml.begin(), ml.end(), 0);
        std::fill(single.begin(), single.end(), 0);
        for (int S = 1; S <= S_max; ++S)
            for (int sh = 0; sh < nsh; ++sh) {
                const int rest = devices - shapes[sh][0] * shapes[sh][1];
                if (rest < 0 || !reach[S - 1][rest]) continue;
                if (S == 1) { single[sh] = 1; continue; }
                const int lmax = L - S + 1;
                auto upd = [&](int first, int last, int w) {
                    int& v = at(first, last, w, sh);
                    if (lmax > v) v = lmax;
                };
                upd(1, 0, std::min(G, S));                                   // i = 1
                upd(0, 1, 1);                                                // i = S
                for (int v = 2; v <= S - 1; ++v) upd(0, 0, std::min(G, v));  // 1 < i < S
            }
        for (int first = 0; first <= 1; ++first)
            for (int last = 0; last <= 1; ++last)
                for (int w = 1; w <= S_max; ++w)
                    for (int l = 1; l <= L; ++l)
                        for (int sh = 0; sh < nsh; ++sh) {
                            const bool ok = (first && last) ? (single[sh] && w == 1 && l == L)
                                                            : l <= at(first, last, w, sh);
                            if (ok) keys.push_back({G, first, last, w, l, shapes[sh][0], shapes[sh][1]});
                        }
    }

    int nz = 0;
    for (int z = 0; z < 4; ++z) nz += space->zero_mask >> z & 1;
    const uint64_t Q1 = (uint64_t)space->offload_steps + 1;
    const uint64_t R = Q1 * Q1 * Q1 * Q1;

    int64_t ng = 0;
    uint64_t tup = 0, cfg = 0;
    for (auto& key : keys) {
        mist_group_t gr;
        std::memset(&gr, 0, sizeof(gr));
        gr.G = key[0]; gr.first = key[1]; gr.last = key[2]; gr.w = key[3];
        gr.layers = key[4]; gr.n = key[5]; gr.m = key[6];
        const int nm = gr.n * gr.m;
        for (int tp = 1; tp <= gr.m; tp <<= 1) {
            if (nm % tp || model->heads % tp || model->kv_heads % tp) continue;
            const int dp = nm / tp;
            const int64_t gdp = (int64_t)gr.G * dp;
            if (B % gdp) continue;
            const int b = (int)(B / gdp);
            if (coeffs_or_null && coef_row(coeffs_or_null, b, tp) < 0) return MIST_ERR_INVALID_ARG;
            if (gr.n_splits == MIST_MAX_SPLITS) return MIST_ERR_INVALID_ARG;
            gr.tp[gr.n_splits] = tp; gr.dp[gr.n_splits] = dp; gr.b[gr.n_splits] = b;
            gr.n_splits++;
        }
        if (!gr.n_splits) continue;
        const uint64_t nt = (uint64_t)gr.n_splits * nz * (gr.layers + 1);
        gr.tuple_offset = tup;
        gr.config_offset = cfg;
        gr.count = nt * R;
        if (groups && ng < groups_cap) groups[ng] = gr;
        ++ng;
        tup += nt;
        cfg += gr.count;
    }
    *n_groups = ng;
    *n_configs = cfg;
    if (ng == 0) return MIST_ERR_EMPTY_SPACE;
    if (groups && ng > groups_cap) return MIST_ERR_BUFFER_TOO_SMALL;
    return MIST_OK;
}

// Size of the preset space (fig:search-space P:364-370):
// per group n_splits * |z| * |c| * prod(ratio counts), |c| = l + 1 or 2 (c in {0, l}).
extern "C" mist_status_t mist_count_space(const mist_model_t* model, int64_t global_batch, const mist_mesh_t* mesh,
                                          const mist_space_t* space, uint64_t* n_in_space, uint64_t* n_configs) {
    if (!n_in_space || !n_configs) return MIST_ERR_INVALID_ARG;
    int64_t ng = 0;
    uint64_t nc = 0;
    mist_status_t st = mist_enumerate_space(model, global_batch, mesh, space, nullptr, nullptr, 0, &ng, &nc);
    if (st != MIST_OK) return st;
    std::vector<mist_group_t> groups((size_t)ng);
    st = mist_enumerate_space(model, global_batch, mesh, space, nullptr, groups.data(), ng, &ng, &nc);
    if (st != MIST_OK) return st;
    int nz = 0;
    for (int z = 0; z < 4; ++z) nz += space->zero_mask >> z & 1;
    uint64_t per_ratio = 1;
    for (int r = 0; r < 4; ++r) per_ratio *= (space->offload_off >> r & 1) ? 1u : (uint64_t)space->offload_steps + 1;
    uint64_t total = 0;
    for (const mist_group_t& g : groups) {
        const uint64_t nc_ckpt = space->ckpt_ends_only ? 2u : (uint64_t)g.layers + 1;
        total += (uint64_t)g.n_splits * nz * nc_ckpt * per_ratio;
    }
    *n_in_space = total;
    *n_configs = nc;
    return MIST_OK;
}

namespace {
// the ranges of mist_shard_ranges (block-cyclic, coalesced)
std::vector<std::pair<uint64_t, uint64_t>> shard_blocks(uint64_t n, int rank, int world) {
    const uint64_t W = (uint64_t)world;
    uint64_t K = n / (W * 2048);
    K = std::max<uint64_t>(1, std::min<uint64_t>(512, K));
    const uint64_t nb = W * K;
    std::vector<std::pair<uint64_t, uint64_t>> out;
    for (uint64_t i = (uint64_t)rank; i < nb; i += W) {
        const uint64_t a = (uint64_t)((unsigned __int128)n * i / nb);
        const uint64_t b = (uint64_t)((unsigned __int128)n * (i + 1) / nb);
        if (b <= a) continue;
        if (!out.empty() && out.back().second == a) out.back().second = b;
        else out.push_back({a, b});
    }
    return out;
}
}  // namespace

std::vector<std::pair<uint64_t, uint64_t>> mist_shard_blocks(uint64_t n_tuples, int rank, int world) {
    return shard_blocks(n_tuples, rank, world);
}

extern "C" mist_status_t mist_shard_ranges(uint64_t n_tuples, int rank, int world, uint64_t* begins,
                                           uint64_t* ends, int64_t cap, int64_t* n_ranges) {
    if (!n_ranges || world < 1 || rank < 0 || rank >= world) return MIST_ERR_INVALID_ARG;
    const auto r = shard_blocks(n_tuples, rank, world);
    *n_ranges = (int64_t)r.size();
    if (!begins || !ends || cap < (int64_t)r.size()) return (begins || ends) ? MIST_ERR_BUFFER_TOO_SMALL : MIST_OK;
    for (size_t i = 0; i < r.size(); ++i) {
        begins[i] = r[i].first;
        ends[i] = r[i].second;
    }
    return MIST_OK;
}

extern "C" const char* mist_status_string(mist_status_t st) {
    switch (st) {
        case MIST_OK: return "MIST_OK";
        case MIST_ERR_INVALID_ARG: return "MIST_ERR_INVALID_ARG";
        case MIST_ERR_EMPTY_SPACE: return "MIST_ERR_EMPTY_SPACE";
        case MIST_ERR_BUFFER_TOO_SMALL: return "MIST_ERR_BUFFER_TOO_SMALL";
        case MIST_ERR_CUDA: return "MIST_ERR_CUDA";
        case MIST_ERR_NCCL: return "MIST_ERR_NCCL";
        case MIST_ERR_OOM: return "MIST_ERR_OOM";
    }
    return "MIST_ERR_UNKNOWN";
}
