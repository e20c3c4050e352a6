"""Search-space presets (fig:search-space P:364-370,
fig:eval-3-ablation P:810-822; readings S1-S3).  CPU tests:

* mist_count_space (closed form over the group table) == the oracle's count of
  admitted configurations one by one, per preset; the full preset == the index
  space; counts grow along the nesting (fig:search-space's growth).
* The oracle's preset gate: every admitted feasible config of a smaller preset
  is feasible in the larger one, and the excluded configs are infeasible.
* Nested presets give a non-increasing optimum of Eq. 2 (the ablation's
  monotone trend as an exact property), on oracle frontiers + the
  exhaustive inter-stage argmin.
The GPU parity per preset is in tests/test_gpu_presets.py."""
import numpy as np
import pytest

from oracle import inter
from oracle.binding import Oracle
from paper_2503_19050_b200 import mist
from synth import PRESETS, random_problem, tiny, with_preset, workload

NAMES = [n for n, _ in PRESETS]


@pytest.mark.parametrize("pb", [tiny(4, 4, 1, 4, 8, 2), tiny(3, 4, 2, 2, 8, 3, kv_heads=2),
                                random_problem(20), random_problem(29)], ids=lambda p: p.name)
def test_count_space(pb):
    prev = 0
    for name in NAMES:
        q = with_preset(pb, name)
        n_in, n_all = mist.mist_count_space(mist.Spec(q))
        o = Oracle(q)
        assert n_all == o.n_configs
        assert n_in == o.count_space()
        assert n_in >= prev
        prev = n_in
    assert prev == o.n_configs                            # +offload admits the whole index space


def test_count_space_workloads():
    # fig:search-space's growth on the five workloads (closed form; exact integers)
    for i in range(1, 6):
        pb = workload(i)
        counts = [mist.mist_count_space(mist.Spec(with_preset(pb, n)))[0] for n in NAMES]
        full, n_all = mist.mist_count_space(mist.Spec(pb))
        assert counts == sorted(counts) and counts[-1] == full == n_all
        q1 = pb.Q + 1
        assert counts[-1] == counts[-2] * q1 ** 4        # offloading multiplies by (Q+1)^4


def test_oracle_gate():
    # presets with the same ZeRO set share the index space: compare config by config
    pb = tiny(4, 4, 1, 4, 8, 2)
    for small, large in (("megatron", "+ckpt"), ("+zero", "+offload")):
        zm = dict(PRESETS)[large]["zero_mask"]
        base_pb = with_preset(pb, large)
        base_pb.ckpt_ends_only, base_pb.offload_off, base_pb.zero_mask = 0, 0, zm
        ob = Oracle(base_pb)
        base = ob.eval_range(0, ob.n_configs)
        evs = []
        for name in (small, large):
            o = Oracle(with_preset(pb, name))
            assert o.n_configs == ob.n_configs
            ev = o.eval_range(0, o.n_configs)
            assert np.array_equal(ev["t"], base["t"]) and np.array_equal(ev["mem"], base["mem"])
            assert not np.any(ev["feasible"] & ~base["feasible"])      # the gate only removes
            evs.append(ev["feasible"].astype(bool))
        assert not np.any(evs[0] & ~evs[1])                          # nesting
        assert evs[0].sum() < evs[1].sum()


def _plan_value(pb):
    o = Oracle(pb)
    ref = o.sweep()
    keys = o.group_keys()
    cands = {}
    for g, k in enumerate(keys):
        P = ref["points"][ref["offsets"][g]:ref["offsets"][g + 1]]
        if len(P) > 3:
            P = P[[0, len(P) // 2, len(P) - 1]]
        cands[k] = [(float(p["t"]), float(p["y"])) for p in P]
    v, _ = inter.brute_force_plan(cands, pb.model.L, pb.N * pb.M)
    return v, cands


@pytest.mark.parametrize("budget", [1_200_000, 3_000_000, 6_000_000])
def test_nested_optimum_monotone(budget):
    # 1.2 MB is memory-tight: only offloading makes a plan fit (S:632's OOM situation)
    pb = tiny(4, 4, 1, 2, 8, 2, mem_budget=budget)
    vals = [_plan_value(with_preset(pb, name))[0] for name in NAMES]
    if budget == 1_200_000:
        assert vals[0] is None and vals[-1] is not None
    finite = [v for v in vals if v is not None]
    assert finite and all(b <= a for a, b in zip(finite, finite[1:]))
    assert all(v is not None for v in vals[vals.index(finite[0]):])   # once feasible, stays feasible
