"""Whole-space sweeps of the big workloads (cfg3, cfg4, cfg5 = BASELINE
configs[2..4]) through the C ABI on one GPU, in the launch configuration
mist_pareto_frontier uses for them (chunking, pilot levels, rollbacks).  The
oracle cannot sweep these spaces (cfg5: 1.86e14 configs), so the check is
("at full size"):
  * properties that hold at any size, on every group: the frontier is sorted
    by t ascending with y strictly descending (O10) and every point lies in
    its group's index range;
  * every frontier point re-evaluated one by one by the oracle (a seeded sample
    of 20,000): feasible, t/d/mem within the north_star tolerance;
  * whole groups the oracle sweeps in seconds (the smallest ones): frontier
    identical to the oracle's up to ties (L26)."""
import os

import numpy as np
import pytest

from oracle.binding import Oracle
from paper_2503_19050_b200 import mist
from synth import workload
from tests.parity import compare_dense, compare_frontiers

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ctx():
    from paper_2503_19050_b200 import build
    build.build()
    c = mist.Context(0)
    yield c
    c.close()


def _at(ctx, spec, idx):
    dev = torch.device("cuda:0")
    ti = torch.from_numpy(idx.astype(np.int64)).to(dev)
    n = len(idx)
    t = torch.empty(n, dtype=torch.float64, device=dev)
    d, m = torch.empty_like(t), torch.empty_like(t)
    f = torch.empty(n, dtype=torch.uint8, device=dev)
    mist.mist_eval_stage_costs_at(ctx, spec, ti, t, d, m, f)
    torch.cuda.synchronize()
    return dict(t=t.cpu().numpy(), d=d.cpu().numpy(), mem=m.cpu().numpy(), feasible=f.cpu().numpy())


@pytest.mark.parametrize("i", [3, 4, 5])
def test_full_sweep_big_config(ctx, i):
    if i == 5 and os.environ.get("MIST_FULLSCALE", "0") != "1":
        pytest.skip("cfg5 whole space takes minutes on one GPU; MIST_FULLSCALE=1 runs it "
                    "(log in profiles/r1/pytest_fullscale_cfg5.log)")
    pb = workload(i)
    o, s = Oracle(pb), mist.Spec(pb)
    pts, offs, _, _ = mist.mist_pareto_frontier(ctx, s, ykey=0)
    assert offs[0] == 0 and offs[-1] == len(pts) and np.all(np.diff(offs) >= 0)
    # O10 order on every group at once: within a group t rises and y falls strictly
    gid = np.repeat(np.arange(o.n_groups), np.diff(offs))
    same = gid[1:] == gid[:-1]
    assert np.all(np.diff(pts["t"])[same] > 0) and np.all(np.diff(pts["y"])[same] < 0)
    # points belong to their group's index range
    cfg_off = np.array([g.config_offset for g in o.groups] + [o.n_configs], dtype=np.uint64)
    assert np.all(pts["idx"] >= cfg_off[gid]) and np.all(pts["idx"] < cfg_off[gid + 1])
    # frontier points re-evaluated one by one (oracle and the GPU's own dense path)
    rng = np.random.default_rng(300 + i)
    pick = rng.choice(len(pts), min(20_000, len(pts)), replace=False)
    idx = pts["idx"][pick]
    ref = o.eval_indices(idx)
    assert np.all(ref["feasible"] == 1)
    compare_dense(dict(t=pts["t"][pick], d=pts["y"][pick], mem=pts["mem"][pick],
                       feasible=np.ones(len(pick), np.uint8)), ref, f"{pb.name} frontier points")
    compare_dense(_at(ctx, s, idx), ref, f"{pb.name} frontier points (dense path)")
    # whole small groups vs the oracle's sweep
    counts = np.array([g.count for g in o.groups])
    cand = np.nonzero(counts <= max(3_000_000, int(counts.min() * 1.01)))[0]
    k = 3 if counts.min() <= 3_000_000 else 1
    for g in sorted(rng.choice(cand, min(k, len(cand)), replace=False).tolist()):
        rs = o.sweep(g, g + 1)
        compare_frontiers(pts, offs, rs["points"], rs["offsets"], groups=[g], label=f"{pb.name} full g{g}")
