// mist_sample.cpp -- a12 sample_frontier (host consumer of the frontiers).
//
// Paper: "a series of alpha in [0, 1] are sampled uniformly to construct a
// Pareto frontier" for the objective alpha*G*t + (1-alpha)*d (Eq. 4, PAPER.md
// lines 679-687); the inter-stage MILP indexes the sampled points as
// IntraStagePareto(i, l_i, (n_i, m_i))[f_i] (Eq. 3).  Reading O11 /
// L29 in DESIGN.md: alpha_j = j/(K-1), ties to smaller t then smaller idx,
// distinct picks in order of first appearance.
#include <vector>

#include "mist.h"

extern "C" mist_status_t mist_sample_frontier(const mist_point_t* frontier, const int64_t* group_offsets,
                                              int64_t n_groups, const mist_group_t* groups, int32_t K,
                                              int64_t* picked, int64_t picked_cap, int64_t* n_picked,
                                              int64_t* picked_offsets) {
    if (K < 2 || n_groups < 0 || !group_offsets || !groups || !n_picked) return MIST_ERR_INVALID_ARG;
    if (group_offsets[0] != 0) return MIST_ERR_INVALID_ARG;
    for (int64_t g = 0; g < n_groups; ++g)
        if (group_offsets[g + 1] < group_offsets[g]) return MIST_ERR_INVALID_ARG;
    if (group_offsets[n_groups] > 0 && !frontier) return MIST_ERR_INVALID_ARG;
    int64_t total = 0;
    std::vector<int64_t> mine;
    for (int64_t g = 0; g < n_groups; ++g) {
        if (picked_offsets) picked_offsets[g] = total;
        const int64_t a = group_offsets[g], b = group_offsets[g + 1];
        const double G = groups[g].G;
        mine.clear();
        for (int32_t j = 0; j < K && b > a; ++j) {
            const double alpha = (double)j / (K - 1);
            int64_t best = a;
            double best_s = alpha * G * frontier[a].t + (1.0 - alpha) * frontier[a].y;
            for (int64_t i = a + 1; i < b; ++i) {
                const double s = alpha * G * frontier[i].t + (1.0 - alpha) * frontier[i].y;
                const mist_point_t& p = frontier[i];
                const mist_point_t& q = frontier[best];
                if (s < best_s || (s == best_s && (p.t < q.t || (p.t == q.t && p.idx < q.idx)))) {
                    best = i;
                    best_s = s;
                }
            }
            bool seen = false;
            for (int64_t v : mine) seen |= (v == best);
            if (!seen) mine.push_back(best);
        }
        for (int64_t v : mine) {
            if (picked && total < picked_cap) picked[total] = v;
            ++total;
        }
    }
    if (picked_offsets) picked_offsets[n_groups] = total;
    *n_picked = total;
    if (total > picked_cap || (!picked && total > 0)) return MIST_ERR_BUFFER_TOO_SMALL;
    return MIST_OK;
}
