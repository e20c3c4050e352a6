"""CUDA path vs the CPU oracle, element by element, through the C ABI.

Sizes: tiny/random spaces in full (several tiles and a ragged tail, Q=1..3),
cfg1 (47.2M configs) in full, cfg2 (7.3e9) through the bench's launch
configuration with sampled groups and random indices, cfg3-cfg5 by random
indices.  Tolerances: tests/parity.py (north_star: bit-exact feasibility,
1e-9 relative t and mem, frontier identical up to ties)."""
import numpy as np
import pytest

from oracle.binding import POINT_DTYPE as ORC_POINT
from oracle.binding import Oracle
from paper_2503_19050_b200 import mist
from synth import random_problem, tiny, workload
from tests.parity import compare_dense, compare_frontiers, frontier_fp_and_bench

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    from paper_2503_19050_b200 import build
    build.build()
    c = mist.Context(0)
    yield c
    c.close()


def gpu_dense(ctx, spec, begin, end):
    n = end - begin
    dev = torch.device("cuda:0")
    t = torch.empty(n, dtype=torch.float64, device=dev)
    d = torch.empty_like(t)
    m = torch.empty_like(t)
    f = torch.empty(n, dtype=torch.uint8, device=dev)
    mist.mist_eval_stage_costs(ctx, spec, begin, end, t, d, m, f)
    torch.cuda.synchronize()
    return dict(t=t.cpu().numpy(), d=d.cpu().numpy(), mem=m.cpu().numpy(), feasible=f.cpu().numpy())


def gpu_at(ctx, spec, idx):
    dev = torch.device("cuda:0")
    ti = torch.from_numpy(idx.astype(np.int64)).to(dev)
    n = len(idx)
    t = torch.empty(n, dtype=torch.float64, device=dev)
    d, m = torch.empty_like(t), torch.empty_like(t)
    f = torch.empty(n, dtype=torch.uint8, device=dev)
    mist.mist_eval_stage_costs_at(ctx, spec, ti, t, d, m, f)
    torch.cuda.synchronize()
    return dict(t=t.cpu().numpy(), d=d.cpu().numpy(), mem=m.cpu().numpy(), feasible=f.cpu().numpy())


def _problems():
    out = [tiny(2, 2, 1, 2, 2, 1), tiny(2, 2, 1, 2, 4, 2), tiny(4, 4, 1, 4, 8, 1), tiny(4, 4, 1, 4, 8, 2),
           tiny(3, 4, 2, 2, 8, 2, fl=0), tiny(5, 4, 2, 4, 12, 3, kv_heads=2, g=1, p=1),
           tiny(3, 4, 2, 2, 8, 2, factors="unit"), tiny(3, 4, 2, 2, 8, 2, factors="spec")]
    for s in range(12):
        out.append(random_problem(s))
    return out


PROBLEMS = _problems()


@pytest.mark.parametrize("k", range(len(PROBLEMS)))
def test_dense_small_spaces(ctx, k):
    pb = PROBLEMS[k]
    try:
        o = Oracle(pb)
    except ValueError:
        pytest.skip("empty space")
    s = mist.Spec(pb)
    n = o.n_configs
    compare_dense(gpu_dense(ctx, s, 0, n), o.eval_range(0, n), pb.name)
    # a ragged window
    a, b = n // 3 + 1, min(n, n // 3 + 1 + 7777)
    compare_dense(gpu_dense(ctx, s, a, b), o.eval_range(a, b), pb.name + " window")


@pytest.mark.parametrize("k", range(len(PROBLEMS)))
@pytest.mark.parametrize("ykey", [0, 1])
def test_frontier_small_spaces(ctx, k, ykey):
    pb = PROBLEMS[k]
    try:
        o = Oracle(pb)
    except ValueError:
        pytest.skip("empty space")
    s = mist.Spec(pb)
    pts, offs, fc, fh = frontier_fp_and_bench(ctx, s, ykey=ykey)
    ref = o.sweep(ykey=ykey)
    assert np.array_equal(fc, ref["fp_count"]) and np.array_equal(fh, ref["fp_hash"])
    compare_frontiers(pts, offs, ref["points"], ref["offsets"], label=pb.name)


def test_dense_cfg1_full(ctx):
    """All 47,172,500 configs of cfg1 (SURVEY 7 step 4 gate)."""
    pb = workload(1)
    o, s = Oracle(pb), mist.Spec(pb)
    step = 1 << 23
    for a in range(0, o.n_configs, step):
        b = min(o.n_configs, a + step)
        compare_dense(gpu_dense(ctx, s, a, b), o.eval_range(a, b), f"cfg1[{a}:{b}]")


@pytest.mark.parametrize("ykey", [0, 1])
def test_frontier_cfg1_full(ctx, ykey):
    pb = workload(1)
    o, s = Oracle(pb), mist.Spec(pb)
    pts, offs, fc, fh = frontier_fp_and_bench(ctx, s, ykey=ykey)
    ref = o.sweep(ykey=ykey)
    assert np.array_equal(fc, ref["fp_count"]) and np.array_equal(fh, ref["fp_hash"])
    st = compare_frontiers(pts, offs, ref["points"], ref["offsets"], label="cfg1")
    assert st["points"] > 1000


@pytest.mark.parametrize("factors", ["spec", "unit"])
def test_frontier_cfg2_bench_config_sampled_groups(ctx, factors):
    """The bench workload (cfg2, full 7.3e9-config sweep, launch configuration
    of bench.py) -- checked on 16 seeded groups the oracle sweeps in full."""
    pb = workload(2, factors=factors)
    o, s = Oracle(pb), mist.Spec(pb)
    pts, offs, fc, fh = frontier_fp_and_bench(ctx, s, ykey=0)
    rng = np.random.default_rng(11)
    counts = np.array([g.count for g in o.groups])
    small = np.nonzero(counts <= 2_500_000)[0]
    chosen = sorted(set(rng.choice(small, 14, replace=False).tolist()) | {0, o.n_groups - 1})
    for g in chosen:
        ref = o.sweep(g, g + 1)
        assert fc[g] == ref["fp_count"][0] and fh[g] == ref["fp_hash"][0]
        compare_frontiers(pts, offs, ref["points"], ref["offsets"], groups=[g], label=f"cfg2 g{g}")
    # random configs across the whole space
    idx = rng.integers(0, o.n_configs, 200_000, dtype=np.uint64)
    compare_dense(gpu_at(ctx, s, idx), o.eval_indices(idx), "cfg2 random")


@pytest.mark.parametrize("i", [1, 2, 3, 4, 5])
def test_eval_at_random_indices(ctx, i):
    pb = workload(i)
    o, s = Oracle(pb), mist.Spec(pb)
    rng = np.random.default_rng(100 + i)
    idx = rng.integers(0, o.n_configs, 200_000, dtype=np.uint64)
    # plus group boundaries and the last config
    extra = [int(g.config_offset) for g in o.groups[:: max(1, o.n_groups // 500)]] + [o.n_configs - 1]
    idx = np.concatenate([idx, np.array(extra, dtype=np.uint64)])
    compare_dense(gpu_at(ctx, s, idx), o.eval_indices(idx), pb.name)


@pytest.mark.parametrize("i", [3, 4, 5])
def test_frontier_big_configs_sampled_groups(ctx, i):
    """cfg3-cfg5: sweep a seeded tuple range covering whole groups on the
    GPU and compare with the oracle's sweep of the same groups."""
    pb = workload(i)
    o, s = Oracle(pb), mist.Spec(pb)
    rng = np.random.default_rng(200 + i)
    counts = np.array([g.count for g in o.groups])
    # groups the oracle sweeps in seconds: the smallest ones (cfg5's smallest has 5.4e7 configs)
    cand = np.nonzero(counts <= max(3_000_000, int(counts.min() * 1.01)))[0]
    k = 4 if counts.min() <= 3_000_000 else 1
    for g in sorted(rng.choice(cand, k, replace=False).tolist()):
        G = o.groups[g]
        R = (pb.Q + 1) ** 4
        tb = int(G.tuple_offset)
        te = tb + int(G.count) // R
        pts, offs, fc, fh = frontier_fp_and_bench(ctx, s, t_begin=tb, t_end=te)
        ref = o.sweep(g, g + 1)
        assert fc[g] == ref["fp_count"][0] and fh[g] == ref["fp_hash"][0]
        assert offs[g + 1] - offs[g] == offs[-1]   # only group g is non-empty
        compare_frontiers(pts, offs, ref["points"], ref["offsets"], groups=[g], label=f"{pb.name} g{g}")


def test_sharding_invariance(ctx):
    """8(e): the frontier does not depend on how the tuple range is cut.
    Shard frontiers (random cut points, k = 1, 2, 3, 8) merged by the exact
    O12 rule equal the one-shot frontier bit for bit."""
    from oracle.binding import frontier_points
    pb = workload(1)
    s = mist.Spec(pb)
    full, foffs, fc, fh = frontier_fp_and_bench(ctx, s)
    rng = np.random.default_rng(5)
    for k in (2, 3, 8):
        cuts = np.sort(rng.choice(np.arange(1, s.n_tuples), k - 1, replace=False))
        bounds = [0, *cuts.tolist(), s.n_tuples]
        parts, cnt, hsh = [], np.zeros(s.n_groups, np.uint64), np.zeros(s.n_groups, np.uint64)
        for a, b in zip(bounds[:-1], bounds[1:]):
            p, off, c, h = frontier_fp_and_bench(ctx, s, t_begin=a, t_end=b)
            gid = np.repeat(np.arange(s.n_groups), np.diff(off))
            q = np.zeros(len(p), dtype=ORC_POINT)
            for f in ("idx", "t", "y", "mem"):
                q[f] = p[f]
            q["group"] = gid
            parts.append(q)
            cnt += c
            hsh += h
        allp = np.concatenate(parts)
        assert np.array_equal(cnt, fc) and np.array_equal(hsh, fh)
        for g in range(s.n_groups):
            mine = allp[allp["group"] == g]
            merged = frontier_points(mine, 2)
            ref = full[foffs[g]:foffs[g + 1]]
            assert merged["idx"].tolist() == ref["idx"].tolist()
            assert merged["t"].tolist() == ref["t"].tolist()


def test_buffer_too_small_and_retry(ctx):
    pb = tiny(4, 4, 1, 4, 8, 2)
    s = mist.Spec(pb)
    import ctypes as C
    L = mist.lib()
    n = C.c_int64(0)
    offs = np.zeros(s.n_groups + 1, dtype=np.int64)
    small = np.zeros(1, dtype=mist.POINT_DTYPE)
    st = L.mist_pareto_frontier(ctx.handle, *s.args(), 0, 0, 0, small.ctypes.data, 1, C.byref(n),
                                offs.ctypes.data, None, None)
    assert st == 3 and n.value > 1
    big = np.zeros(n.value, dtype=mist.POINT_DTYPE)
    st = L.mist_pareto_frontier(ctx.handle, *s.args(), 0, 0, 0, big.ctypes.data, n.value, C.byref(n),
                                offs.ctypes.data, None, None)
    assert st == 0
    again, offs2, _, _ = mist.mist_pareto_frontier(ctx, s)
    assert again.tobytes() == big.tobytes() and np.array_equal(offs, offs2)


def test_retry_cache_keyed_on_groups(ctx):
    """The BUFFER_TOO_SMALL retry cache is keyed on the group table too: a
    retry with a different (invalid) table is validated, not served stale."""
    import ctypes as C
    pb = tiny(4, 4, 1, 4, 8, 2)
    s = mist.Spec(pb)
    L = mist.lib()
    n = C.c_int64(0)
    offs = np.zeros(s.n_groups + 1, dtype=np.int64)
    small = np.zeros(1, dtype=mist.POINT_DTYPE)
    st = L.mist_pareto_frontier(ctx.handle, *s.args(), 0, 0, 0, small.ctypes.data, 1, C.byref(n),
                                offs.ctypes.data, None, None)
    assert st == 3 and n.value > 1
    s.groups[0].w += 1
    big = np.zeros(n.value, dtype=mist.POINT_DTYPE)
    st = L.mist_pareto_frontier(ctx.handle, *s.args(), 0, 0, 0, big.ctypes.data, n.value, C.byref(n),
                                offs.ctypes.data, None, None)
    assert st == 1


def test_prepare_cache_not_stale(ctx):
    """prepare() skips re-validation for byte-identical inputs; any changed
    input (here one operator-time table) must give that input's result, the
    same as a fresh context computes."""
    import copy
    pb = tiny(4, 4, 1, 4, 8, 2)
    pb2 = copy.deepcopy(pb)
    pb2.Tf = [v * 1.5 for v in pb2.Tf]
    s1, s2 = mist.Spec(pb), mist.Spec(pb2)
    a1, o1, _, _ = mist.mist_pareto_frontier(ctx, s1)
    a1b, _, _, _ = mist.mist_pareto_frontier(ctx, s1)          # cache hit
    a2, o2, _, _ = mist.mist_pareto_frontier(ctx, s2)          # changed table
    assert a1.tobytes() == a1b.tobytes()
    fresh = mist.Context(0)
    try:
        f2, g2, _, _ = mist.mist_pareto_frontier(fresh, s2)
    finally:
        fresh.close()
    assert a2.tobytes() == f2.tobytes() and np.array_equal(o2, g2)
    assert a2.tobytes() != a1.tobytes()


def test_eval_at_out_of_range_index(ctx):
    """Every index is range-checked on the device, at any list length: one bad
    index among 2^21 gives INVALID_ARG and the context stays usable."""
    pb = workload(1)
    s = mist.Spec(pb)
    n = (1 << 21) + 3
    rng = np.random.default_rng(3)
    idx = rng.integers(0, s.n_configs, n, dtype=np.uint64)
    idx[n - 2] = s.n_configs                   # one past the end
    with pytest.raises(mist.MistError) as ei:
        gpu_at(ctx, s, idx)
    assert ei.value.status == 1
    idx[n - 2] = s.n_configs - 1
    out = gpu_at(ctx, s, idx[-1000:])
    assert np.all(out["t"] > 0)


def test_device_output_buffers(ctx):
    """Outputs may be device memory (torch tensors)."""
    pb = tiny(4, 4, 1, 4, 8, 1)
    s = mist.Spec(pb)
    host, hoffs, _, _ = mist.mist_pareto_frontier(ctx, s)
    dev = torch.zeros(len(host) * 4, dtype=torch.float64, device="cuda:0")
    doffs = torch.zeros(s.n_groups + 1, dtype=torch.int64, device="cuda:0")
    mist.mist_pareto_frontier(ctx, s, out=dev, group_offsets=doffs)
    assert dev.cpu().numpy().tobytes() == host.tobytes()
    assert np.array_equal(doffs.cpu().numpy(), hoffs)


def test_invalid_groups_rejected(ctx):
    pb = tiny(2, 2, 1, 2, 4, 2)
    s = mist.Spec(pb)
    s.groups[0].w += 1
    with pytest.raises(mist.MistError) as ei:
        mist.mist_pareto_frontier(ctx, s)
    assert ei.value.status == 1


@pytest.mark.parametrize("reduce", ["seg", "radix"])
@pytest.mark.parametrize("seed", range(10))
def test_frontier_points_vs_oracle(ctx, seed, reduce, monkeypatch):
    """a9 + a10 alone, on both reductions (group buckets + shared-memory chunk
    sorts, the default; global radix sort + segmented scan, MIST_REDUCE=radix):
    random point sets (heavy ties in t and y, many binades, many groups, ragged
    sizes; seeds 6-8: a few groups of up to 1e5 points, so groups span many
    1024-record chunks and several levels; seed 9: one group whose frontier alone
    exceeds a chunk, which the bucket path hands to the radix path) equal the
    oracle's O(k^2)/sort-scan frontier of the same points, bit for bit."""
    from oracle.binding import frontier_points as orc_frontier
    monkeypatch.setenv("MIST_REDUCE", reduce)
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300_000)) if seed else 5
    ng = int(rng.integers(1, 2000)) if seed < 6 else int(rng.integers(1, 9))
    if seed == 9:
        n, ng = 6000, 1
    g = np.sort(rng.integers(0, ng, n)).astype(np.int32) if seed % 2 else rng.integers(0, ng, n).astype(np.int32)
    pts = np.zeros(n, dtype=mist.POINT_DTYPE)
    if seed == 9:          # every point on the frontier: t rises, y falls
        pts["t"] = rng.permutation(n) + 1.0
        pts["y"] = n + 1.0 - pts["t"]
    elif seed % 3 == 0:    # few distinct values: long equal-t runs and y ties
        pts["t"] = rng.integers(0, 50, n) * 0.125
        pts["y"] = rng.integers(0, 50, n) * 0.5
    else:                  # full-precision doubles across many binades
        pts["t"] = np.exp(rng.uniform(-20, 5, n))
        pts["y"] = np.exp(rng.uniform(-20, 5, n))
    pts["idx"] = rng.permutation(n * 4)[:n].astype(np.uint64)
    pts["mem"] = rng.uniform(0, 1e10, n)
    fr, offs = mist.mist_frontier_points(ctx, pts, g, ng)
    if seed == 9:
        assert len(fr) == n
    for q in range(ng):
        sel = g == q
        op = np.zeros(int(sel.sum()), dtype=ORC_POINT)
        for f in ("idx", "t", "y", "mem"):
            op[f] = pts[f][sel]
        want = orc_frontier(op, 2)
        got = fr[offs[q]:offs[q + 1]]
        assert got["idx"].tolist() == want["idx"].tolist(), q
        assert got["t"].tolist() == want["t"].tolist() and got["y"].tolist() == want["y"].tolist()
