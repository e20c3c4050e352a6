"""End to end: sweep on the GPU -> per-group frontiers / alpha-samples ->
inter-stage plan (Eq. 2-3), against the oracle.

* Sampled formulation (the paper's, P:687 + Eq. 3): the device sweep's
  alpha-samples (mist_pareto_sample, K = 3) feed mist_solve_inter; the oracle's
  own sweep + sampler feed the exhaustive argmin (oracle/inter.py).  The
  optima agree within L24/L26's tolerance (the two frontiers may differ only
  at near-ties).
* Exact formulation: the whole (t, d) frontier.  The plan's stages are
  re-evaluated one by one by the oracle from their config indices, and its
  objective must equal Eq. 2 on those values; the optimum must not be worse
  than the solver's optimum over the oracle's own frontier (and vice versa),
  within tolerance."""
import numpy as np
import pytest

from oracle import inter
from oracle.binding import Oracle
from paper_2503_19050_b200 import mist
from synth import random_problem, tiny, workload

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

RTOL = 1e-9


@pytest.fixture(scope="module")
def ctx():
    from paper_2503_19050_b200 import build
    build.build()
    c = mist.Context(0)
    yield c
    c.close()


def _validate(o, plan, pts, keys, L, devices):
    """Stage keys, sums, and Eq. 2 of the plan on the oracle's own per-config values."""
    G, S = plan["G"], plan["S"]
    idx = np.array([int(pts[q]["idx"]) for q in plan["point"]], dtype=np.uint64)
    ev = o.eval_indices(idx)
    assert ev["feasible"].all()
    ls = devs = 0
    for i in range(S):
        k = keys[int(plan["group"][i])]
        assert k == inter.stage_key(G, S, i + 1, k[4], k[5], k[6])
        g = o.groups[int(plan["group"][i])]
        assert g.config_offset <= int(idx[i]) < g.config_offset + g.count
        ls += k[4]
        devs += k[5] * k[6]
    assert ls == L and devs == devices
    v = inter.objective(G, list(ev["t"]), list(ev["d"]))
    assert plan["objective"] == pytest.approx(v, rel=RTOL)
    return v


def _problems():
    return [("tiny_a", tiny(4, 4, 1, 4, 8, 2)), ("tiny_b", tiny(5, 4, 2, 2, 12, 3, kv_heads=2, g=1, p=1)),
            ("tiny_c", tiny(4, 8, 1, 4, 16, 2, factors="spec"))] + \
           [(f"rand{s}", random_problem(s)) for s in (0, 2, 20, 22, 29, 33)]


@pytest.mark.parametrize("name,pb", _problems())
def test_sampled_plan_vs_brute_force(ctx, name, pb):
    K = 3
    o = Oracle(pb)
    spec = mist.Spec(pb)
    keys = o.group_keys()
    L, devices = pb.model.L, pb.N * pb.M
    # device: sweep + alpha-sampling in one call
    smp, npk = mist.mist_pareto_sample(ctx, spec, K=K)
    offs = np.zeros(spec.n_groups + 1, dtype=np.int64)
    offs[1:] = np.cumsum(npk)
    pts = np.concatenate([smp[g, :npk[g]] for g in range(spec.n_groups)]) if offs[-1] else \
        np.zeros(0, dtype=mist.POINT_DTYPE)
    # (1) the solver on the device's candidates, re-evaluated one by one by the oracle,
    #     against the exhaustive argmin of Eq. 2 over the same candidates
    ev = o.eval_indices(pts["idx"]) if len(pts) else None
    cands = {}
    for g, k in enumerate(keys):
        cands[k] = [(float(ev["t"][q]), float(ev["d"][q])) for q in range(offs[g], offs[g + 1])]
    want, _ = inter.brute_force_plan(cands, L=L, devices=devices)
    if want is None:
        with pytest.raises(mist.MistError):
            mist.mist_solve_inter(spec.groups, pts, offs, L, devices)
        return
    plan = mist.mist_solve_inter(spec.groups, pts, offs, L, devices)
    v = _validate(o, plan, pts, keys, L, devices)
    assert v == pytest.approx(want, rel=RTOL)
    # (2) the oracle's own pipeline (its sweep, its sampler, brute force): the same optimum
    #     whenever it sampled the same configurations (samples may differ at score near-ties)
    ref = o.sweep()
    picked, poffs = o.sample(ref["points"], ref["offsets"], K)
    same = all(sorted(ref["points"][picked[poffs[g]:poffs[g + 1]]]["idx"].tolist()) ==
               sorted(pts[offs[g]:offs[g + 1]]["idx"].tolist()) for g in range(len(keys)))
    if same:
        own = {k: [(float(p["t"]), float(p["y"])) for p in ref["points"][picked[poffs[g]:poffs[g + 1]]]]
               for g, k in enumerate(keys)}
        want_o, _ = inter.brute_force_plan(own, L=L, devices=devices)
        assert v == pytest.approx(want_o, rel=RTOL)


@pytest.mark.parametrize("name,pb", [("tiny_a", tiny(4, 4, 1, 4, 8, 2)), ("cfg1", workload(1)),
                                     ("cfg1_unit", workload(1, factors="unit"))])
def test_exact_plan_full_frontier(ctx, name, pb):
    o = Oracle(pb)
    spec = mist.Spec(pb)
    keys = o.group_keys()
    L, devices = pb.model.L, pb.N * pb.M
    pts, offs, _, _ = mist.mist_pareto_frontier(ctx, spec, ykey=mist.Y_DELTA)
    plan = mist.mist_solve_inter(spec.groups, pts, offs, L, devices)
    v = _validate(o, plan, pts, keys, L, devices)
    ref = o.sweep()
    plan_o = mist.mist_solve_inter(spec.groups, ref["points"], ref["offsets"], L, devices)
    assert v == pytest.approx(plan_o["objective"], rel=RTOL)
    # no sampled plan can beat the exact one
    smp, npk = mist.mist_pareto_sample(ctx, spec, K=16)
    so = np.zeros(spec.n_groups + 1, dtype=np.int64)
    so[1:] = np.cumsum(npk)
    sp = np.concatenate([smp[g, :npk[g]] for g in range(spec.n_groups)])
    plan_s = mist.mist_solve_inter(spec.groups, sp, so, L, devices)
    assert plan_s["objective"] >= v * (1 - RTOL)
