"""Inter-stage consumer (Eq. 2-3).

CPU tests: the oracle (oracle/inter.py) pinned against hand evaluations of
Eq. 2 and the SPEC's pipeline recurrence, then libmist's host solver
(mist_solve_inter) against the oracle's exhaustive argmin on seeded candidate
tables.  The GPU end-to-end case (sweep -> frontier -> plan) is in
tests/test_gpu_inter.py."""
import itertools
import random

import numpy as np
import pytest

from oracle import inter
from oracle.binding import Oracle
from paper_2503_19050_b200 import mist
from synth import random_candidates, tiny


# ---------------------------------------------------------------- oracle pins
def test_objective_examples():
    # S:362-365, each evaluated by hand from Eq. 2
    assert inter.objective(4, [10, 12], [5, 3]) == 63.0          # 3*12 + 22 + max(5, 3-10)
    assert inter.objective(3, [7], [0]) == 21.0                  # serial: G*t
    assert inter.objective(4, [10, 12], [0, 0]) == 58.0          # fill-drain (G-1) max + sum
    # the third term reads t_j (L4): stage 3's d is offset by t_1 + t_2, not 2*t_3
    assert inter.objective(2, [1, 2, 4], [0, 0, 10]) == 4 + 7 + 7


def test_objective_two_stage_table():
    # all four selections of S:530's two-stage table, evaluated by hand from Eq. 2:
    # (10,5)(12,3): 36+22+5 = 63; (10,5)(10,8): 30+20+5 = 55;
    # (12,0)(12,3): 36+24+0 = 60; (12,0)(10,8): 36+22+0 = 58.
    # (S:530 prints 63, 63, 66, 62; those values do not follow from Eq. 2 -- DESIGN.md 8, I4.)
    s1, s2 = [(10, 5), (12, 0)], [(12, 3), (10, 8)]
    vals = {(a, b): inter.objective(4, [a[0], b[0]], [a[1], b[1]]) for a in s1 for b in s2}
    assert vals == {((10, 5), (12, 3)): 63, ((10, 5), (10, 8)): 55,
                    ((12, 0), (12, 3)): 60, ((12, 0), (10, 8)): 58}
    cands = {inter.stage_key(4, 2, 1, 1, 1, 1): s1, inter.stage_key(4, 2, 2, 1, 1, 1): s2}
    v, plan = inter.brute_force_plan(cands, L=2, devices=2)
    assert v == 55 and plan[0] == 4 and [p for _, p in plan[1]] == [0, 1]


def test_simulate_examples():
    # S:369-372
    assert inter.simulate(1, [3, 4], [0, 10]) == 14.0
    assert inter.simulate(4, [10, 12], [0, 0]) == 3 * 12 + 22
    assert inter.simulate(5, [3], [2]) == 2 + 5 * 3              # S = 1: d_1 + G t_1


def test_simulate_closed_form_and_sandwich():
    rng = random.Random(7)
    for _ in range(600):
        S, G = rng.randint(1, 7), rng.randint(1, 12)
        t = [rng.uniform(0.1, 5.0) for _ in range(S)]
        d = [rng.choice([0.0, rng.uniform(0.0, 20.0)]) for _ in range(S)]
        sim, cf, obj = inter.simulate(G, t, d), inter.closed_form(G, t, d), inter.objective(G, t, d)
        assert cf == pytest.approx(sim, rel=1e-12)
        assert obj >= sim * (1 - 1e-12)                           # objective >= simulate
        assert sim >= G * max(t) * (1 - 1e-12) and sim >= sum(t) * (1 - 1e-12)
        z = [0.0] * S
        assert inter.objective(G, t, z) == pytest.approx(inter.simulate(G, t, z), rel=1e-12)


def test_objective_monotone():
    rng = random.Random(11)
    for _ in range(300):
        S, G = rng.randint(1, 6), rng.randint(1, 9)
        t = [rng.uniform(0.1, 5.0) for _ in range(S)]
        d = [rng.uniform(0.0, 9.0) for _ in range(S)]
        v = inter.objective(G, t, d)
        i = rng.randrange(S)
        t2, d2 = list(t), list(d)
        t2[i] += rng.uniform(0, 2)
        d2[i] += rng.uniform(0, 2)
        lo = v * (1 - 1e-12)     # Eq. 2's literal form cancels (d_i - sum t_j): monotone up to rounding
        assert inter.objective(G, t2, d) >= lo and inter.objective(G, t, d2) >= lo
        assert inter.objective(G + 1, t, d) >= lo


def test_brute_force_single_stage_collapse():
    # S = 1 only (L = 1): Eq. 2 degenerates to min over candidates of G t + d
    cands = {(2, 1, 1, 1, 1, 1, 1): [(3.0, 4.0), (5.0, 0.0)], (4, 1, 1, 1, 1, 1, 1): [(1.0, 9.0)]}
    v, plan = inter.brute_force_plan(cands, L=1, devices=1)
    assert v == min(2 * 3 + 4, 2 * 5 + 0, 4 * 1 + 9) == 10
    assert plan == (2, [((2, 1, 1, 1, 1, 1, 1), 0)])


def test_brute_force_nesting():
    # a restricted candidate table (subset) never gives a lower optimum (Fig. 11 nesting)
    keys = _tiny_keys(tiny(4, 4, 1, 4, 4, 2))
    pts = random_candidates(keys, seed=3)
    full = {k: p for k, p in zip(keys, pts)}
    v_full, _ = inter.brute_force_plan(full, L=4, devices=4)
    rng = random.Random(5)
    for _ in range(5):
        sub = {k: [q for q in p if rng.random() < 0.6] for k, p in full.items()}
        v_sub, _ = inter.brute_force_plan(sub, L=4, devices=4)
        assert v_sub is None or v_sub >= v_full


# ---------------------------------------------------------------- libmist solver vs oracle
def _tiny_keys(pb):
    return Oracle(pb).group_keys()


def _csr(pts):
    offs = np.zeros(len(pts) + 1, dtype=np.int64)
    flat = []
    for g, p in enumerate(pts):
        offs[g + 1] = offs[g] + len(p)
        flat += p
    arr = np.zeros(len(flat), dtype=mist.POINT_DTYPE)
    for i, (t, d) in enumerate(flat):
        arr[i] = (i, t, d, 0.0)
    return arr, offs


def _check_plan(plan, keys, pts, L, devices, want):
    G, S = plan["G"], plan["S"]
    arr, offs = _csr(pts)
    ls, devs, stages = 0, 0, []
    for i in range(S):
        g, q = int(plan["group"][i]), int(plan["point"][i])
        k = keys[g]
        assert k == inter.stage_key(G, S, i + 1, k[4], k[5], k[6]), (i, k)
        assert offs[g] <= q < offs[g + 1]
        ls += k[4]
        devs += k[5] * k[6]
        stages.append((float(arr[q]["t"]), float(arr[q]["y"])))
    assert ls == L and devs == devices
    v = inter.plan_value(G, stages)
    assert plan["objective"] == pytest.approx(v, rel=1e-12)
    assert v == pytest.approx(want, rel=1e-12)


@pytest.mark.parametrize("shape,seed", [((4, 4, 1, 4, 4, 2), 1), ((4, 4, 1, 4, 4, 2), 2),
                                        ((5, 2, 1, 2, 8, 2), 3), ((3, 4, 2, 2, 4, 2), 4),
                                        ((6, 4, 1, 2, 2, 2), 5), ((4, 8, 1, 4, 12, 2), 6)])
def test_solver_matches_brute_force(shape, seed):
    pb = tiny(*shape)
    keys = _tiny_keys(pb)
    L, devices = pb.model.L, pb.N * pb.M
    for rep in range(3):
        pts = random_candidates(keys, seed=100 * seed + rep)
        want, _ = inter.brute_force_plan({k: p for k, p in zip(keys, pts)}, L=L, devices=devices)
        arr, offs = _csr(pts)
        groups = mist.group_array(keys)
        if want is None:
            with pytest.raises(mist.MistError):
                mist.mist_solve_inter(groups, arr, offs, L, devices)
            continue
        for nt in (1, 3):
            plan = mist.mist_solve_inter(groups, arr, offs, L, devices, n_threads=nt)
            _check_plan(plan, keys, pts, L, devices, want)


def test_solver_fractional_values():
    # non-integer candidates (rounding order differs from the oracle's literal Eq. 2)
    pb = tiny(4, 4, 1, 4, 4, 2)
    keys = _tiny_keys(pb)
    for rep in range(3):
        pts = random_candidates(keys, seed=900 + rep, scale=0.0137)
        want, _ = inter.brute_force_plan({k: p for k, p in zip(keys, pts)}, L=4, devices=4)
        arr, offs = _csr(pts)
        plan = mist.mist_solve_inter(mist.group_array(keys), arr, offs, 4, 4)
        _check_plan(plan, keys, pts, 4, 4, want)


def test_solver_errors():
    keys = [(1, 1, 1, 1, 2, 1, 1)]
    arr, offs = _csr([[(1.0, 0.0)]])
    g = mist.group_array(keys)
    with pytest.raises(mist.MistError) as e:
        mist.mist_solve_inter(g, arr, offs, 3, 1)            # no plan covers 3 layers
    assert e.value.status == 2
    with pytest.raises(mist.MistError) as e:
        mist.mist_solve_inter(g, arr, np.array([0, -1], dtype=np.int64), 2, 1)   # non-monotone offsets
    assert e.value.status == 1
    with pytest.raises(mist.MistError) as e:
        mist.mist_solve_inter(g, arr, offs, 0, 1)
    assert e.value.status == 1
    plan = mist.mist_solve_inter(g, arr, offs, 2, 1)
    assert plan["S"] == 1 and plan["objective"] == 1.0


def test_solver_real_frontier_cfg_tiny():
    # oracle frontiers of a real (tiny) problem: exact optimum over the whole space
    pb = tiny(4, 4, 1, 4, 8, 2)
    o = Oracle(pb)
    ref = o.sweep()
    keys = o.group_keys()
    pts = [[(float(p["t"]), float(p["y"])) for p in ref["points"][ref["offsets"][g]:ref["offsets"][g + 1]]]
           for g in range(len(keys))]
    # the brute force is exponential in the points per group: keep <= 3 by alpha-sampling-like thinning
    thin = [p if len(p) <= 3 else [p[0], p[len(p) // 2], p[-1]] for p in pts]
    want, _ = inter.brute_force_plan({k: p for k, p in zip(keys, thin)}, L=4, devices=4)
    arr, offs = _csr(thin)
    plan = mist.mist_solve_inter(mist.group_array(keys), arr, offs, 4, 4)
    _check_plan(plan, keys, thin, 4, 4, want)


@pytest.mark.parametrize("thin", ["0", "1"])
def test_solver_many_points_per_group(monkeypatch, thin):
    # > 8 candidates per group: with MIST_INTER_THIN=1 the solver first solves a thinned
    # table for its incumbent (mist_inter.cpp); the optimum must equal the exhaustive
    # argmin with and without it
    monkeypatch.setenv("MIST_INTER_THIN", thin)
    pb = tiny(3, 4, 1, 2, 4, 2)
    keys = _tiny_keys(pb)
    for rep in range(2):
        pts = random_candidates(keys, seed=700 + rep, max_points=12, p_empty=0.0)
        pts = [p + [(t + 40.0, max(0.0, d - 5.0)) for t, d in p] for p in pts]     # 2..24 points
        assert sum(len(p) for p in pts) > 8 * len(keys)
        want, _ = inter.brute_force_plan({k: p for k, p in zip(keys, pts)}, L=3, devices=2)
        arr, offs = _csr(pts)
        plan = mist.mist_solve_inter(mist.group_array(keys), arr, offs, 3, 2)
        _check_plan(plan, keys, pts, 3, 2, want)


@pytest.mark.parametrize("scheme", ["", "G"])
def test_solver_plan_independent_of_threads(monkeypatch, scheme):
    """The plan (not only its value) is the same for every thread count: the
    per-step parallel DP (default) reduces its closing stages in state order and
    builds each destination state on one thread."""
    monkeypatch.setenv("MIST_INTER_PAR", scheme)
    pb = tiny(6, 4, 1, 2, 2, 2)
    keys = _tiny_keys(pb)
    L, devices = pb.model.L, pb.N * pb.M
    for rep in range(4):
        pts = random_candidates(keys, seed=900 + rep, max_points=6, p_empty=0.05)
        arr, offs = _csr(pts)
        groups = mist.group_array(keys)
        plans = [mist.mist_solve_inter(groups, arr, offs, L, devices, n_threads=nt) for nt in (1, 2, 5)]
        for p in plans[1:]:
            assert (p["G"], p["S"], p["objective"]) == (plans[0]["G"], plans[0]["S"], plans[0]["objective"])
            assert p["group"].tolist() == plans[0]["group"].tolist()
            assert p["point"].tolist() == plans[0]["point"].tolist()
