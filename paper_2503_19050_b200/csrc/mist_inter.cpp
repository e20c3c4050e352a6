// mist_inter.cpp -- inter-stage consumer of the frontiers.
//
// Paper: Eq. 2-3: choose G, the number of stages S,
// and per stage i a layer count l_i, a submesh (n_i, m_i) and a point f_i of
// IntraStagePareto(i, l_i, (n_i, m_i)) minimising
//     (G-1) max_i t_i + sum_i t_i + max_i (d_i - sum_{j<i} t_j)      (reading L4)
// subject to sum l_i = L and sum n_i m_i = N*M.  The paper solves an
// MILP with CBC; this is an exact label-setting dynamic program instead
// (DESIGN.md 8), host C++, since the MILP is a host-side consumer of the
// frontiers and not the optimisation target (BASELINE north_star).
//
// Rewriting the objective with suffix sums s_i = sum_{j>=i} t_j:
//     sum_i t_i + max_i (d_i - sum_{j<i} t_j) = max_i (d_i + s_i),
// so a partial plan of the LAST k stages is summarised by the label
// (Ssum = s_{S-k+1}, Mx = max over its stages of d_i + s_i, Tm = max t_i), and
// prepending a stage (t, d) gives (Ssum + t, max(Mx, d + Ssum + t), max(Tm, t)),
// monotone in every component.  A label that another label of the same state
// (layers used, devices used, k) matches or beats in all three can therefore
// never lead to a better plan, and a label whose (G-1) Tm + Mx already reaches
// the incumbent cannot either.  Stage i's group key depends on its distance from
// the end (w = min(G, S-i+1), last = [i = S], O2), so building plans from the
// last stage backwards lets one DP per G serve every S: closing the plan with a
// "first" stage at step k gives S = k.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <cmath>
#include <limits>
#include <map>
#include <thread>
#include <unordered_map>
#include <vector>

#include "mist.h"

namespace {

struct Label {
    double S, M, T;      // suffix sum of t, max_i (d_i + s_i), max t_i
    int32_t parent;      // node of the partial plan this extends (-1: empty)
    int32_t g, p;        // this stage: group, candidate position within the group
};

struct Node {
    int32_t parent, g, p;
};

struct State {
    std::vector<Label> v;
    size_t thr = 4096;      // filter again once v has grown past this
};

struct Result {
    double val = std::numeric_limits<double>::infinity();
    int32_t G = 0, S = 0;
    std::vector<int32_t> g;   // stage 1..S
    std::vector<int32_t> p;
    int64_t labels = 0;
};

inline uint64_t pack_key(int G, int first, int last, int w, int l, int n, int m) {
    // G <= 2^20, w, l <= 2^10, n, m <= 2^10
    return ((uint64_t)G << 42) | ((uint64_t)first << 41) | ((uint64_t)last << 40) | ((uint64_t)w << 30) |
           ((uint64_t)l << 20) | ((uint64_t)n << 10) | (uint64_t)m;
}

struct Problem {
    const mist_group_t* groups;
    const mist_point_t* pts;
    const int64_t* offs;
    int L, devices;
    std::unordered_map<uint64_t, int32_t> key;     // group key -> index (non-empty groups only)
    std::vector<std::pair<int, int>> meshes;       // distinct (n, m)

    int32_t find(int G, int first, int last, int w, int l, int n, int m) const {
        auto it = key.find(pack_key(G, first, last, w, l, n, m));
        return it == key.end() ? -1 : it->second;
    }
};

// Keep the labels of one state that no other label matches or beats in (T, S, M);
// drop labels whose bound reaches the incumbent.  Sorted by (T, S, M); a staircase
// over (S -> min M) of the labels kept so far answers "is there one with S' <= S
// and M' <= M".
void pareto_filter(std::vector<Label>& v, double G1, double inc) {
    std::sort(v.begin(), v.end(), [](const Label& a, const Label& b) {
        if (a.T != b.T) return a.T < b.T;
        if (a.S != b.S) return a.S < b.S;
        if (a.M != b.M) return a.M < b.M;
        if (a.parent != b.parent) return a.parent < b.parent;
        if (a.g != b.g) return a.g < b.g;
        return a.p < b.p;
    });
    std::map<double, double> stair;   // S ascending, M strictly decreasing
    size_t out = 0;
    for (size_t i = 0; i < v.size(); ++i) {
        const Label& a = v[i];
        if (G1 * a.T + a.M >= inc) continue;
        auto it = stair.upper_bound(a.S);
        if (it != stair.begin()) {
            auto pv = std::prev(it);
            if (pv->second <= a.M) continue;        // matched or beaten
        }
        // entries with S'' >= S and M'' >= M are covered by this one for later queries
        auto jt = stair.lower_bound(a.S);
        while (jt != stair.end() && jt->second >= a.M) jt = stair.erase(jt);
        stair[a.S] = a.M;
        v[out++] = a;
    }
    v.resize(out);
}

// The DP of one G.  Plans whose value does not beat `inc` are not reported.
Result solve_G(const Problem& pb, int G, double inc) {
    Result best;
    best.val = inc;
    const double G1 = (double)(G - 1);
    const int L = pb.L, D = pb.devices;
    const int Smax = std::min(L, D);
    std::vector<Node> nodes;
    // states of step k: (layers used, devices used) -> labels
    std::map<std::pair<int, int>, State> cur, nxt;
    cur[{0, 0}].v.push_back(Label{0.0, 0.0, 0.0, -1, -1, -1});
    int32_t close_parent = -1, close_g = -1, close_p = -1, close_k = 0;
    for (int k = 1; k <= Smax && !cur.empty(); ++k) {
        const int w = std::min(G, k), last = k == 1;
        nxt.clear();
        for (auto& st : cur) {
            const int lu = st.first.first, du = st.first.second;
            std::vector<Label>& labs = st.second.v;
            // node ids of this state's labels (created once the labels survived filtering)
            std::vector<int32_t> nid(labs.size());
            for (size_t i = 0; i < labs.size(); ++i) {
                if (labs[i].g < 0) { nid[i] = -1; continue; }
                nid[i] = (int32_t)nodes.size();
                nodes.push_back(Node{labs[i].parent, labs[i].g, labs[i].p});
            }
            const int lrem = L - lu, drem = D - du;
            // close the plan: this stage is stage 1 (first) and S = k
            for (auto& nm : pb.meshes) {
                if (nm.first * nm.second != drem) continue;
                const int32_t g = pb.find(G, 1, last, w, lrem, nm.first, nm.second);
                if (g < 0) continue;
                const int64_t a = pb.offs[g], b = pb.offs[g + 1];
                for (size_t i = 0; i < labs.size(); ++i) {
                    const Label& lb = labs[i];
                    for (int64_t q = a; q < b; ++q) {
                        const double t = pb.pts[q].t, d = pb.pts[q].y;
                        const double S2 = lb.S + t, M2 = std::max(lb.M, d + S2), T2 = std::max(lb.T, t);
                        const double val = G1 * T2 + M2;
                        if (val < best.val) {
                            best.val = val;
                            close_parent = nid[i]; close_g = g; close_p = (int32_t)(q - a); close_k = k;
                        }
                    }
                }
            }
            if (k == Smax) continue;
            // extend: this stage is stage S-k+1 > 1; at least one layer and one device stay for the first
            for (int l = 1; l <= lrem - 1; ++l)
                for (auto& nm : pb.meshes) {
                    const int sz = nm.first * nm.second;
                    if (sz > drem - 1) continue;
                    const int32_t g = pb.find(G, 0, last, w, l, nm.first, nm.second);
                    if (g < 0) continue;
                    const int64_t a = pb.offs[g], b = pb.offs[g + 1];
                    State& ns = nxt[{lu + l, du + sz}];
                    std::vector<Label>& out = ns.v;
                    for (size_t i = 0; i < labs.size(); ++i) {
                        const Label& lb = labs[i];
                        if (G1 * lb.T + lb.M >= best.val) continue;
                        for (int64_t q = a; q < b; ++q) {
                            const double t = pb.pts[q].t, d = pb.pts[q].y;
                            const double S2 = lb.S + t, M2 = std::max(lb.M, d + S2), T2 = std::max(lb.T, t);
                            if (G1 * T2 + M2 >= best.val) continue;
                            out.push_back(Label{S2, M2, T2, nid[i], g, (int32_t)(q - a)});
                        }
                    }
                    if (out.size() > ns.thr) {
                        pareto_filter(out, G1, best.val);
                        ns.thr = 2 * out.size() + 4096;
                    }
                }
        }
        for (auto it = nxt.begin(); it != nxt.end();) {
            pareto_filter(it->second.v, G1, best.val);
            best.labels += (int64_t)it->second.v.size();
            if (it->second.v.empty()) it = nxt.erase(it); else ++it;
        }
        std::swap(cur, nxt);
    }
    if (close_k > 0) {
        best.G = G;
        best.S = close_k;
        best.g.push_back(close_g);
        best.p.push_back(close_p);
        for (int32_t nd = close_parent; nd >= 0; nd = nodes[nd].parent) {
            best.g.push_back(nodes[nd].g);
            best.p.push_back(nodes[nd].p);
        }
    }
    return best;
}

// The same DP with the work of each step spread over threads (OpenMP), results
// independent of the thread count.  Per step: (1) node ids of the current labels,
// in state order; (2) closing stages, per source state in parallel, reduced in
// state order with strict < (the plan the sequential loop finds first among
// equal values); (3) extensions grouped by destination state, each destination
// built by one thread from its sources in state order and filtered.  The
// incumbent of (3) is the one after all of step k's closes, tighter than or equal
// to the sequential loop's: pruning stays exact.
Result solve_G_par(const Problem& pb, int G, double inc, int nthreads) {
    Result best;
    best.val = inc;
    const double G1 = (double)(G - 1);
    const int L = pb.L, D = pb.devices;
    const int Smax = std::min(L, D);
    std::vector<Node> nodes;
    std::map<std::pair<int, int>, State> cur, nxt;
    cur[{0, 0}].v.push_back(Label{0.0, 0.0, 0.0, -1, -1, -1});
    int32_t close_parent = -1, close_g = -1, close_p = -1, close_k = 0;
    struct Src { int lu, du; std::vector<Label>* labs; std::vector<int32_t> nid; };
    struct Task { int si; int32_t g; };
    struct Close { double val; int32_t parent, g, p; };
    for (int k = 1; k <= Smax && !cur.empty(); ++k) {
        const int w = std::min(G, k), last = k == 1;
        std::vector<Src> src;
        src.reserve(cur.size());
        for (auto& st : cur) {
            Src sc{st.first.first, st.first.second, &st.second.v, {}};
            sc.nid.resize(sc.labs->size());
            for (size_t i = 0; i < sc.labs->size(); ++i) {
                const Label& lb = (*sc.labs)[i];
                if (lb.g < 0) { sc.nid[i] = -1; continue; }
                sc.nid[i] = (int32_t)nodes.size();
                nodes.push_back(Node{lb.parent, lb.g, lb.p});
            }
            src.push_back(std::move(sc));
        }
        // (2) close the plan: this stage is stage 1 (first) and S = k
        std::vector<Close> closes(src.size(), Close{std::numeric_limits<double>::infinity(), -1, -1, -1});
        const double inc_k = best.val;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
        for (long long si = 0; si < (long long)src.size(); ++si) {
            const Src& sc = src[(size_t)si];
            Close c{inc_k, -1, -1, -1};
            const int lrem = L - sc.lu, drem = D - sc.du;
            for (auto& nm : pb.meshes) {
                if (nm.first * nm.second != drem) continue;
                const int32_t g = pb.find(G, 1, last, w, lrem, nm.first, nm.second);
                if (g < 0) continue;
                const int64_t a = pb.offs[g], b = pb.offs[g + 1];
                for (size_t i = 0; i < sc.labs->size(); ++i) {
                    const Label& lb = (*sc.labs)[i];
                    for (int64_t q = a; q < b; ++q) {
                        const double t = pb.pts[q].t, d = pb.pts[q].y;
                        const double S2 = lb.S + t, M2 = std::max(lb.M, d + S2), T2 = std::max(lb.T, t);
                        const double val = G1 * T2 + M2;
                        if (val < c.val) c = Close{val, sc.nid[i], g, (int32_t)(q - a)};
                    }
                }
            }
            closes[(size_t)si] = c;
        }
        for (size_t si = 0; si < src.size(); ++si)
            if (closes[si].g >= 0 && closes[si].val < best.val) {
                best.val = closes[si].val;
                close_parent = closes[si].parent; close_g = closes[si].g; close_p = closes[si].p; close_k = k;
            }
        nxt.clear();
        if (k < Smax) {
            // (3) extensions, grouped by destination state
            std::map<std::pair<int, int>, std::vector<Task>> dest;
            for (size_t si = 0; si < src.size(); ++si) {
                const int lrem = L - src[si].lu, drem = D - src[si].du;
                for (int l = 1; l <= lrem - 1; ++l)
                    for (auto& nm : pb.meshes) {
                        const int sz = nm.first * nm.second;
                        if (sz > drem - 1) continue;
                        const int32_t g = pb.find(G, 0, last, w, l, nm.first, nm.second);
                        if (g < 0) continue;
                        dest[{src[si].lu + l, src[si].du + sz}].push_back(Task{(int)si, g});
                    }
            }
            std::vector<std::pair<std::pair<int, int>, std::vector<Task>*>> dl;
            dl.reserve(dest.size());
            for (auto& e : dest) dl.push_back({e.first, &e.second});
            std::vector<std::vector<Label>> out(dl.size());
            const double inc_x = best.val;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
            for (long long di = 0; di < (long long)dl.size(); ++di) {
                std::vector<Label>& o = out[(size_t)di];
                size_t thr = 4096;
                for (const Task& tk : *dl[(size_t)di].second) {
                    const Src& sc = src[(size_t)tk.si];
                    const int64_t a = pb.offs[tk.g], b = pb.offs[tk.g + 1];
                    for (size_t i = 0; i < sc.labs->size(); ++i) {
                        const Label& lb = (*sc.labs)[i];
                        if (G1 * lb.T + lb.M >= inc_x) continue;
                        for (int64_t q = a; q < b; ++q) {
                            const double t = pb.pts[q].t, d = pb.pts[q].y;
                            const double S2 = lb.S + t, M2 = std::max(lb.M, d + S2), T2 = std::max(lb.T, t);
                            if (G1 * T2 + M2 >= inc_x) continue;
                            o.push_back(Label{S2, M2, T2, sc.nid[i], tk.g, (int32_t)(q - a)});
                        }
                    }
                    if (o.size() > thr) {
                        pareto_filter(o, G1, inc_x);
                        thr = 2 * o.size() + 4096;
                    }
                }
                pareto_filter(o, G1, inc_x);
            }
            for (size_t di = 0; di < dl.size(); ++di) {
                if (out[di].empty()) continue;
                best.labels += (int64_t)out[di].size();
                nxt[dl[di].first].v = std::move(out[di]);
            }
        }
        std::swap(cur, nxt);
    }
    if (close_k > 0) {
        best.G = G;
        best.S = close_k;
        best.g.push_back(close_g);
        best.p.push_back(close_p);
        for (int32_t nd = close_parent; nd >= 0; nd = nodes[nd].parent) {
            best.g.push_back(nodes[nd].g);
            best.p.push_back(nodes[nd].p);
        }
    }
    return best;
}

}  // namespace

extern "C" mist_status_t mist_solve_inter(const mist_group_t* groups, int64_t n_groups, const mist_point_t* points,
                                          const int64_t* group_offsets, int32_t num_layers, int32_t n_devices,
                                          int32_t n_threads, mist_plan_t* plan) {
    if (!groups || n_groups < 1 || !group_offsets || !plan || num_layers < 1 || n_devices < 1)
        return MIST_ERR_INVALID_ARG;
    if (group_offsets[0] != 0) return MIST_ERR_INVALID_ARG;
    for (int64_t g = 0; g < n_groups; ++g)
        if (group_offsets[g + 1] < group_offsets[g]) return MIST_ERR_INVALID_ARG;
    if (group_offsets[n_groups] > 0 && !points) return MIST_ERR_INVALID_ARG;
    Problem pb;
    pb.groups = groups; pb.pts = points; pb.offs = group_offsets;
    pb.L = num_layers; pb.devices = n_devices;
    std::vector<int> Gs;
    for (int64_t g = 0; g < n_groups; ++g) {
        const mist_group_t& gr = groups[g];
        if (gr.G < 1 || gr.G >= (1 << 20) || gr.w < 1 || gr.w >= 1024 || gr.layers < 1 || gr.layers >= 1024 ||
            gr.n < 1 || gr.n >= 1024 || gr.m < 1 || gr.m >= 1024)
            return MIST_ERR_INVALID_ARG;
        if (std::find(pb.meshes.begin(), pb.meshes.end(), std::make_pair(gr.n, gr.m)) == pb.meshes.end())
            pb.meshes.push_back({gr.n, gr.m});
        if (std::find(Gs.begin(), Gs.end(), gr.G) == Gs.end()) Gs.push_back(gr.G);
        if (group_offsets[g + 1] > group_offsets[g])
            pb.key[pack_key(gr.G, gr.first, gr.last, gr.w, gr.layers, gr.n, gr.m)] = (int32_t)g;
    }
    std::sort(pb.meshes.begin(), pb.meshes.end());
    std::sort(Gs.begin(), Gs.end());

    // incumbent seed: the best single-stage plan over every G (value G t + d, exact DP form)
    double seed = std::numeric_limits<double>::infinity();
    for (int G : Gs)
        for (auto& nm : pb.meshes) {
            if (nm.first * nm.second != n_devices) continue;
            const int32_t g = pb.find(G, 1, 1, 1, num_layers, nm.first, nm.second);
            if (g < 0) continue;
            for (int64_t q = group_offsets[g]; q < group_offsets[g + 1]; ++q) {
                const double t = points[q].t;
                const double v = (double)(G - 1) * t + std::max(0.0, points[q].y + t);
                seed = std::min(seed, v);
            }
        }
    unsigned nt = n_threads > 0 ? (unsigned)n_threads : std::max(1u, std::thread::hardware_concurrency());
    nt = std::min<unsigned>(nt, (unsigned)Gs.size());
    auto run_all = [&](const Problem& q, double inc, std::vector<Result>& res) {
        res.assign(Gs.size(), Result());
        std::atomic<size_t> next{0};
        auto worker = [&]() {
            for (size_t i; (i = next.fetch_add(1)) < Gs.size();) res[i] = solve_G(q, Gs[i], inc);
        };
        std::vector<std::thread> th;
        for (unsigned i = 1; i < nt; ++i) th.emplace_back(worker);
        worker();
        for (auto& t : th) t.join();
    };
    // A tighter incumbent from a thinned candidate set (at most 4 points per group: the
    // ends and two inner points of each frontier): its optimum is a real plan, so the
    // exact DP may prune every label whose bound reaches it.  Pruning with a valid upper
    // bound explores the same plans below it, so the result is unchanged.  Off by default
    // (MIST_INTER_THIN=1 enables it): it halved the solve on a synthetic cfg5-like table,
    // but on cfg5's real frontier it was slower (10.5 -> 11.3 s) for 0.7% fewer labels
    // (profiles/r1/cfg5_r1y_n4.log vs cfg5_r1z_n4.log).
    const int64_t n_pts = group_offsets[n_groups];
    const char* thin_env = getenv("MIST_INTER_THIN");
    const bool thin_on = thin_env && thin_env[0] == '1';
    if (thin_on && n_pts > 8 * n_groups) {
        std::vector<mist_point_t> tp;
        std::vector<int64_t> to(n_groups + 1, 0);
        tp.reserve((size_t)n_groups * 4);
        for (int64_t g = 0; g < n_groups; ++g) {
            const int64_t a = group_offsets[g], n = group_offsets[g + 1] - a;
            if (n <= 4) {
                for (int64_t k = 0; k < n; ++k) tp.push_back(points[a + k]);
            } else {
                const int64_t pick[4] = {0, n / 3, (2 * n) / 3, n - 1};
                for (int64_t k : pick) tp.push_back(points[a + k]);
            }
            to[g + 1] = (int64_t)tp.size();
        }
        Problem thin = pb;
        thin.pts = tp.data();
        thin.offs = to.data();
        std::vector<Result> rt;
        run_all(thin, std::nextafter(seed, std::numeric_limits<double>::infinity()), rt);
        for (const Result& r : rt)
            if (r.S > 0) seed = std::min(seed, r.val);
    }
    // the seed only prunes; a plan equal to it is found again by its own G's DP
    const double inc = std::nextafter(seed, std::numeric_limits<double>::infinity());

    std::vector<Result> res;
    const char* par_env = getenv("MIST_INTER_PAR");
    if (par_env && !strcmp(par_env, "G")) {
        run_all(pb, inc, res);   // round-1 scheme: one G per thread, the single-stage seed as incumbent
    } else {
        // G by G in ascending order, each DP spread over every thread, with the best plan so
        // far as the incumbent: a G whose plans cannot beat it prunes everything early.
        // Strict improvement only, so ties keep the smaller G (processed first).
        const unsigned nthr = n_threads > 0 ? (unsigned)n_threads : std::max(1u, std::thread::hardware_concurrency());
        res.assign(Gs.size(), Result());
        double incumbent = inc;
        for (size_t i = 0; i < Gs.size(); ++i) {
            res[i] = solve_G_par(pb, Gs[i], incumbent, (int)nthr);
            if (res[i].S > 0) incumbent = std::min(incumbent, res[i].val);
        }
    }

    int best = -1;
    int64_t labels = 0;
    for (size_t i = 0; i < res.size(); ++i) {
        labels += res[i].labels;
        if (res[i].S > 0 && (best < 0 || res[i].val < res[best].val)) best = (int)i;   // ties: smaller G
    }
    if (best < 0) return MIST_ERR_EMPTY_SPACE;
    const Result& r = res[best];
    if (r.S > MIST_MAX_STAGES) return MIST_ERR_BUFFER_TOO_SMALL;
    plan->G = r.G;
    plan->S = r.S;
    plan->labels = labels;
    // Eq. 2 of the chosen plan, written out term by term (stage 1 = first)
    double tmax = 0.0, tsum = 0.0, third = -std::numeric_limits<double>::infinity();
    for (int i = 0; i < r.S; ++i) {
        const mist_point_t& pt = points[group_offsets[r.g[i]] + r.p[i]];
        third = std::max(third, pt.y - tsum);
        tsum += pt.t;
        tmax = std::max(tmax, pt.t);
        plan->group[i] = r.g[i];
        plan->point[i] = group_offsets[r.g[i]] + r.p[i];
    }
    plan->t_max = tmax;
    plan->t_sum = tsum;
    plan->d_term = third;
    plan->objective = (double)(r.G - 1) * tmax + tsum + third;
    return MIST_OK;
}
