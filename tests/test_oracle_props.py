"""Property pins of the oracle: invariants the paper's definitions fix at any
size (SURVEY.md Sec. 8(c) P11-P13, O9 monotonicity, O10 transitivity, O12)."""
import numpy as np
import pytest

from oracle.binding import POINT_DTYPE, Oracle, frontier_points
from synth import random_problem, tiny


def _beats(p, q):
    """O10 / P:660: p beats q."""
    return (p["t"] <= q["t"] and p["y"] <= q["y"] and
            (p["t"] < q["t"] or p["y"] < q["y"] or p["idx"] < q["idx"]))


def _random_points(rng, n, ties=True):
    pts = np.zeros(n, dtype=POINT_DTYPE)
    if ties:
        pts["t"] = rng.integers(0, 12, n).astype(float)
        pts["y"] = rng.integers(0, 12, n).astype(float)
    else:
        pts["t"] = rng.uniform(0, 1, n)
        pts["y"] = rng.uniform(0, 1, n)
    pts["idx"] = rng.permutation(n * 3)[:n]
    return pts


def test_sort_scan_equals_pairwise_definition():
    """P11: the O(k^2) pairwise filter (the definition) equals sort+scan."""
    rng = np.random.default_rng(3)
    for trial in range(300):
        pts = _random_points(rng, int(rng.integers(1, 120)), ties=trial % 2 == 0)
        a = frontier_points(pts, 1)
        b = frontier_points(pts, 2)
        assert a.tobytes() == b.tobytes()
        # brute check in python of the definition
        keep = [q for q in pts if not any(_beats(p, q) for p in pts if p["idx"] != q["idx"])]
        assert sorted(int(q["idx"]) for q in keep) == sorted(a["idx"].tolist())
        # output sorted by x ascending with y strictly descending
        assert np.all(np.diff(a["t"]) > 0) and np.all(np.diff(a["y"]) < 0)


def test_merge_associativity():
    """O12: frontier(A u B) = frontier(frontier(A) u frontier(B)) for any split."""
    rng = np.random.default_rng(4)
    for _ in range(200):
        pts = _random_points(rng, int(rng.integers(2, 200)), ties=True)
        cut = rng.random(len(pts)) < 0.5
        fa, fb = frontier_points(pts[cut], 2), frontier_points(pts[~cut], 2)
        merged = frontier_points(np.concatenate([fa, fb]), 2)
        assert merged.tobytes() == frontier_points(pts, 2).tobytes()


def _dense(o):
    r = o.eval_range(0, o.n_configs)
    gt = o.group_table()
    gid = np.repeat(np.arange(o.n_groups), gt[:, 9])
    return r, gid


@pytest.mark.parametrize("seed", range(12))
def test_frontier_invariants_on_problems(seed):
    """P11: no frontier point is beaten; every discarded feasible point of the
    group is beaten by a frontier point.  P12: every alpha-argmin of
    alpha*G*t + (1-alpha)*d over the feasible set lies on the frontier (ties
    broken by smaller t, then smaller d, then smaller idx)."""
    try:
        o = Oracle(random_problem(seed))
    except ValueError:
        pytest.skip("empty space (no valid split) for this seed")
    if o.n_configs > 200_000:
        pytest.skip("space too large for the brute-force check")
    r, gid = _dense(o)
    res = o.sweep(ykey=0, threads=2)
    offs = res["offsets"]
    for g in range(o.n_groups):
        sel = np.nonzero((gid == g) & (r["feasible"] == 1))[0]
        base = int(o.groups[g].config_offset)
        fr = res["points"][offs[g]:offs[g + 1]]
        assert res["fp_count"][g] == len(sel)
        if len(sel) == 0:
            assert len(fr) == 0
            continue
        pts = np.zeros(len(sel), dtype=POINT_DTYPE)
        pts["idx"] = sel.astype(np.uint64) + 0 * base
        pts["t"], pts["y"] = r["t"][sel], r["d"][sel]
        frs = set(fr["idx"].tolist())
        # frontier is exactly the non-beaten set
        for q in pts:
            beaten = any(_beats(fp, q) for fp in fr if fp["idx"] != q["idx"])
            assert beaten != (int(q["idx"]) in frs)
        G = o.groups[g].G
        for alpha in np.linspace(0, 1, 11):
            score = alpha * G * pts["t"] + (1 - alpha) * pts["y"]
            best = np.lexsort((pts["idx"], pts["y"], pts["t"], score))[0]
            assert int(pts["idx"][best]) in frs


def test_t_constant_along_oo_run():
    """P13: t never reads OO, so it is bitwise constant along kO."""
    for seed in range(4):
        try:
            o = Oracle(random_problem(seed))
        except ValueError:
            continue
        n = min(o.n_configs, 100_000)
        r = o.eval_range(0, n)
        Q1 = o.pb.Q + 1
        t = r["t"][: n - n % (Q1 ** 2)].reshape(-1, Q1, Q1)   # [..., kO, kA]
        assert np.all(t == t[:, :1, :])


def test_memory_exact_and_monotone():
    """O9: D*mem is an integer; feasibility is exactly mem <= Mem_Budget; mem
    is non-increasing in each offload ratio and in c for c >= 1."""
    pb = tiny(4, 4, 1, 4, 8, 3, mem_budget=3_000_000)
    o = Oracle(pb)
    Q, Q1 = pb.Q, pb.Q + 1
    for gi, g in enumerate(o.groups[:20]):
        for sp in range(g.n_splits):
            D = pb.Q * g.tp[sp] * g.dp[sp]
            for z in range(4):
                mem = np.zeros((g.l + 1, Q1, Q1, Q1, Q1))
                for c in range(g.l + 1):
                    for kW in range(Q1):
                        for kG in range(Q1):
                            for kO in range(Q1):
                                for kA in range(Q1):
                                    d = o.detail(gi, sp, z, c, kW, kG, kO, kA)
                                    assert d.mem * D == d.mem_fwd_D or d.mem * D == d.mem_bwd_D
                                    assert float(int(d.mem * D)) == d.mem * D
                                    assert d.feasible == (d.mem <= pb.mem_budget)
                                    mem[c, kW, kG, kO, kA] = d.mem
                for ax in (1, 2, 3, 4):
                    assert np.all(np.diff(mem, axis=ax) <= 0)
                if g.l >= 2:
                    assert np.all(np.diff(mem[1:], axis=0) <= 0)


def test_unit_factor_time_monotone():
    """O9 notes: under unit factors t is non-decreasing in WO, GO, AO and d in OO."""
    pb = tiny(4, 4, 1, 4, 8, 2, factors="unit")
    o = Oracle(pb)
    Q1 = pb.Q + 1
    for gi, g in enumerate(o.groups[:25]):
        for sp in range(g.n_splits):
            for z in range(4):
                for c in range(g.l + 1):
                    T = np.zeros((Q1,) * 4)
                    Dd = np.zeros((Q1,) * 4)
                    for k in np.ndindex(*(Q1,) * 4):
                        det = o.detail(gi, sp, z, c, *map(int, k))
                        T[k], Dd[k] = det.t, det.d
                    tol = 1e-15 * T.max()
                    for ax in (0, 1, 3):
                        assert np.all(np.diff(T, axis=ax) >= -tol)
                    assert np.all(np.diff(Dd, axis=2) >= -tol)


def test_budget_honesty():
    """a config rejected at budget B is rejected at every smaller budget."""
    pb = tiny(2, 2, 1, 2, 4, 2, mem_budget=2_000_000)
    hi = Oracle(pb).eval_range(0, 8748)["feasible"]
    lo = Oracle(pb.replace(mem_budget=1_000_000)).eval_range(0, 8748)["feasible"]
    assert np.all(lo <= hi) and lo.sum() < hi.sum()


def test_sampling():
    """O11: picks lie on the frontier, are distinct, alpha=1 picks the
    minimum-t point and alpha=0 the minimum-d point; K < 2 is rejected."""
    o = Oracle(tiny(2, 2, 1, 2, 4, 2, mem_budget=2_000_000))
    res = o.sweep(threads=1)
    picked, poffs = o.sample(res["points"], res["offsets"], K=16)
    for g in range(o.n_groups):
        mine = picked[poffs[g]:poffs[g + 1]]
        a, b = res["offsets"][g], res["offsets"][g + 1]
        if b == a:
            assert len(mine) == 0
            continue
        assert len(set(mine.tolist())) == len(mine)
        assert all(a <= p < b for p in mine)
        assert mine[0] == b - 1          # alpha = 0: minimum d is the last (largest t)
        assert a in mine.tolist()        # alpha = 1: minimum t
    with pytest.raises(ValueError):
        o.sample(res["points"], res["offsets"], K=1)


def test_dp1_zero_level_twins():
    """L20 (DESIGN R9): at DP = 1 all sigmas are 1 and every DP collective is 0
    (O4-O6), so the ZeRO levels of a tuple share t and d exactly while mem is
    non-decreasing in z (O9: z = 3 adds the gathered layers, z >= 2 the
    unsharded grads).  Hence every z above the lowest level is beaten by its
    lowest-level twin (smaller idx), and no frontier point of the oracle has
    DP = 1 and z above the lowest enumerated level."""
    for seed, pb in enumerate([tiny(4, 4, 1, 4, 8, 2), tiny(3, 4, 2, 2, 8, 2, factors="spec"),
                               tiny(5, 4, 2, 4, 12, 2, kv_heads=2, g=1, p=1), random_problem(3)]):
        try:
            o = Oracle(pb)
        except ValueError:
            continue
        Q1 = pb.Q + 1
        rng = np.random.default_rng(seed)
        seen = 0
        for gi, g in enumerate(o.groups):
            for sp in range(g.n_splits):
                if g.dp[sp] != 1:
                    continue
                for _ in range(6):
                    c = int(rng.integers(0, g.l + 1))
                    k = [int(v) for v in rng.integers(0, Q1, 4)]
                    base = o.detail(gi, sp, 0, c, *k)
                    for z in (1, 2, 3):
                        d = o.detail(gi, sp, z, c, *k)
                        assert d.t == base.t and d.d == base.d
                        assert d.mem >= base.mem
                        seen += 1
        if o.n_configs <= 300_000:
            res = o.sweep(ykey=0, threads=2)
            R = Q1 ** 4
            for g in range(o.n_groups):
                G = o.groups[g]
                for p in res["points"][res["offsets"][g]:res["offsets"][g + 1]]:
                    local = int(p["idx"]) // R - int(G.config_offset) // R
                    per_split = 4 * (G.l + 1)
                    sp, z = local // per_split, (local % per_split) // (G.l + 1)
                    assert not (G.dp[sp] == 1 and z > 0)
        assert seen > 0 or seed == 3
