"""Search-space presets on the GPU against the oracle.

* Per preset, dense t/d/mem/feasible (feasible bit-exact: the preset gate is
  integer logic) and per-group frontiers + feasible-set fingerprints
  (bit-exact), on small spaces, the pilot-filtered path included (cfg1, cfg2
  sampled groups).
* The nested presets give a non-increasing optimum of Eq. 2 on cfg1 and on a
  memory-tight problem (sweep -> frontier -> mist_solve_inter).
* Imbalance awareness (the ablation's last bar): the Eq. 2 optimum
  is never worse than the true Eq. 2 value of the plan an imbalance-unaware
  tuner picks (d ignored)."""
import numpy as np
import pytest

from oracle import inter
from oracle.binding import Oracle
from paper_2503_19050_b200 import mist
from synth import PRESETS, random_problem, tiny, with_preset, workload
from tests.parity import compare_dense, compare_frontiers, frontier_fp_and_bench

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

NAMES = [n for n, _ in PRESETS]


@pytest.fixture(scope="module")
def ctx():
    from paper_2503_19050_b200 import build
    build.build()
    c = mist.Context(0)
    yield c
    c.close()


def _dense(ctx, s, a, b):
    n = b - a
    dev = torch.device("cuda:0")
    t = torch.empty(n, dtype=torch.float64, device=dev)
    d, m = torch.empty_like(t), torch.empty_like(t)
    f = torch.empty(n, dtype=torch.uint8, device=dev)
    mist.mist_eval_stage_costs(ctx, s, a, b, t, d, m, f)
    torch.cuda.synchronize()
    return dict(t=t.cpu().numpy(), d=d.cpu().numpy(), mem=m.cpu().numpy(), feasible=f.cpu().numpy())


SMALL = [tiny(4, 4, 1, 4, 8, 2), tiny(5, 4, 2, 2, 12, 3, kv_heads=2, g=1, p=1),
         tiny(4, 4, 1, 2, 8, 2, mem_budget=1_200_000, factors="spec"), random_problem(20), random_problem(29)]


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("k", range(len(SMALL)))
def test_dense_and_frontier_presets(ctx, name, k):
    pb = with_preset(SMALL[k], name)
    o, s = Oracle(pb), mist.Spec(pb)
    n = o.n_configs
    compare_dense(_dense(ctx, s, 0, n), o.eval_range(0, n), pb.name)
    for ykey in (0, 1):
        pts, offs, fc, fh = frontier_fp_and_bench(ctx, s, ykey=ykey)
        ref = o.sweep(ykey=ykey)
        assert np.array_equal(fc, ref["fp_count"]) and np.array_equal(fh, ref["fp_hash"])
        compare_frontiers(pts, offs, ref["points"], ref["offsets"], label=pb.name)
    assert int(np.sum(fc)) <= mist.mist_count_space(s)[0]


@pytest.mark.parametrize("name", NAMES)
def test_frontier_cfg1_presets(ctx, name):
    pb = with_preset(workload(1), name)
    o, s = Oracle(pb), mist.Spec(pb)
    pts, offs, fc, fh = frontier_fp_and_bench(ctx, s)
    ref = o.sweep()
    assert np.array_equal(fc, ref["fp_count"]) and np.array_equal(fh, ref["fp_hash"])
    compare_frontiers(pts, offs, ref["points"], ref["offsets"], label=pb.name)


@pytest.mark.parametrize("name", ["+ckpt", "+offload"])
def test_frontier_cfg2_presets_sampled_groups(ctx, name):
    # the bench workload through the pilot-filtered sweep; 24 seeded groups checked against the oracle
    pb = with_preset(workload(2), name)
    o, s = Oracle(pb), mist.Spec(pb)
    pts, offs, fc, fh = frontier_fp_and_bench(ctx, s)
    rng = np.random.default_rng(7)
    for g in sorted(rng.choice(o.n_groups, size=24, replace=False).tolist()):
        ref = o.sweep(g, g + 1)
        assert fc[g] == ref["fp_count"][0] and fh[g] == ref["fp_hash"][0]
        compare_frontiers(pts, offs, ref["points"], ref["offsets"], groups=[g], label=f"{pb.name} g{g}")


def _solve(ctx, pb):
    s = mist.Spec(pb)
    pts, offs, _, _ = mist.mist_pareto_frontier(ctx, s)
    try:
        return mist.mist_solve_inter(s.groups, pts, offs, pb.model.L, pb.N * pb.M), pts, offs, s
    except mist.MistError as e:
        assert e.status == 2
        return None, pts, offs, s


@pytest.mark.parametrize("pb", [workload(1), tiny(4, 4, 1, 2, 8, 2, mem_budget=1_200_000),
                                tiny(4, 4, 1, 2, 8, 2, mem_budget=3_000_000)], ids=lambda p: p.name)
def test_nested_optimum_and_imbalance_awareness(ctx, pb):
    vals = []
    for name in NAMES:
        plan, pts, offs, s = _solve(ctx, with_preset(pb, name))
        vals.append(None if plan is None else plan["objective"])
    finite = [v for v in vals if v is not None]
    assert finite and all(b <= a * (1 + 1e-12) for a, b in zip(finite, finite[1:]))
    # the full space: aware optimum vs the plan an imbalance-unaware tuner picks
    plan, pts, offs, s = _solve(ctx, pb)
    unaware = pts.copy()
    unaware["y"] = 0.0                     # d ignored: each group's frontier point of least t wins
    up = mist.mist_solve_inter(s.groups, unaware, offs, pb.model.L, pb.N * pb.M)
    true_t = [float(pts[q]["t"]) for q in up["point"]]
    true_d = [float(pts[q]["y"]) for q in up["point"]]
    assert plan["objective"] <= inter.objective(up["G"], true_t, true_d) * (1 + 1e-12)
