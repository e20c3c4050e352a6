"""Pins of the CPU oracle against values fixed by the paper, the SPEC's worked
examples, hand arithmetic and closed forms -- never against the oracle itself.

Every test names the passage that fixes its expected value.
P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n; W1/W2, P1-P13 and
L* = SURVEY.md Sec. 8(c).
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle.binding import Oracle, pred_intf
from synth import factor_table, tiny, workload
from tests.helpers import find_group, golden_problem, load_golden

REL = 1e-12


def _close(a, b, rel=REL, abs_=0.0):
    return abs(a - b) <= rel * max(abs(a), abs(b)) + abs_


# --------------------------------------------------------------------------
# P6 -- Alg. 1 PredINTF
# --------------------------------------------------------------------------
def test_intf_single_channel_identity():
    """S:208 '(C=10, others 0), any params -> 10'; Alg. 1 residue sum."""
    for name in ("unit", "spec", "asym"):
        F = factor_table(name)
        assert pred_intf([10.0, 0, 0, 0], F) == 10.0
        for j in range(4):
            X = [0.0] * 4
            X[j] = 0.123456789
            assert pred_intf(X, F) == 0.123456789
        assert pred_intf([0.0, 0, 0, 0], F) == 0.0


def test_intf_spec_pair_example():
    """(C=10, G2G=4), pair factors (1.2, 1.5) -> scaled (12, 6),
    overlap 6, residues (5, 0), total 11."""
    F = [[1.0] * 4 for _ in range(16)]
    F[0b0011] = [1.2, 1.5, 1.0, 1.0]
    assert _close(pred_intf([10.0, 4.0, 0, 0], F), 11.0, 1e-15)


def test_intf_hand_trace_three_channels():
    """Hand trace of Alg. 1 on X=(10, 4, 2, 0) with asymmetric
    factors.  n=4: pattern 0111 != 1111, skip.  n=3, mask {0,1,2}: scaled =
    (11, 4.8, 2.6), overlap 2.6, X = (8.4/1.1, 2.2/1.2, 0), T = 2.6.  n=2,
    mask {0,1}: scaled = (8.4*1.5/1.1, 2.2*1.6/1.2), overlap = 2.2*1.6/1.2,
    X0 = (8.4*1.5/1.1 - 2.2*1.6/1.2)/1.5, T += overlap; then T += X0."""
    F = [[1.0] * 4 for _ in range(16)]
    F[0b0111] = [1.1, 1.2, 1.3, 1.0]
    F[0b0011] = [1.5, 1.6, 1.0, 1.0]
    F[0b0101] = [9.0, 1.0, 9.0, 1.0]     # must NOT be used: pattern after n=3 is 0011
    q = Fraction
    x0 = (q(11) - q(26, 10)) / q(11, 10)
    x1 = (q(48, 10) - q(26, 10)) / q(12, 10)
    ov2 = x1 * q(16, 10)
    expect = q(26, 10) + ov2 + (x0 * q(15, 10) - ov2) / q(15, 10)
    assert _close(pred_intf([10.0, 4.0, 2.0, 0.0], F), float(expect), 1e-14)


def test_intf_unit_factors_is_max():
    """S:210 / S:227: all factors 1 -> max of the channels (perfect overlap);
    ledger L10: not bitwise, within a few ulp."""
    rng = np.random.default_rng(1)
    F = factor_table("unit")
    for _ in range(2000):
        X = rng.uniform(0, 1, 4) * (rng.uniform(0, 1, 4) < 0.7)
        assert _close(pred_intf(list(X), F), float(X.max()), 1e-15)


def test_intf_bounds():
    """S:216-217 (SPEC property): max(channels) <= PredINTF <= sum(factor x channel)."""
    rng = np.random.default_rng(2)
    for name in ("spec", "asym"):
        F = factor_table(name)
        fmax = max(max(r) for r in F)
        for _ in range(2000):
            X = rng.uniform(0, 1, 4) * (rng.uniform(0, 1, 4) < 0.7)
            v = pred_intf(list(X), F)
            assert v >= X.max() * (1 - 1e-15)
            assert v <= fmax * X.sum() * (1 + 1e-15)


# --------------------------------------------------------------------------
# P7 -- collectives (O5)
# --------------------------------------------------------------------------
def _coll_oracle():
    pb = golden_problem(load_golden("w1_gpt3_1.3b.json"))
    return Oracle(pb)


def test_collectives_spec_examples():
    """AR g=1 -> 0; AR 8e9 B, g=4, bw 1e10, lat 0 -> 1.2 s; AG = AR/2.
    P:212: ZeRO-1 'introduces no additional communication': RS + AG = AR."""
    import ctypes as C
    from oracle.binding import lib
    o = _coll_oracle()
    coll = lambda k, x, g: lib().orc_coll(C.byref(o.s), k, x, g, 0)
    assert coll(0, 8e9, 1) == 0.0
    assert _close(coll(0, 8e9, 4), 1.2, 1e-15)
    assert _close(coll(1, 8e9, 4), 0.6, 1e-15)
    for g in (2, 3, 4, 8, 16):
        assert _close(coll(2, 1e9, g) + coll(1, 1e9, g), coll(0, 1e9, g), 1e-15)
        assert _close(2 * coll(1, 1e9, g), coll(0, 1e9, g), 1e-15)


# --------------------------------------------------------------------------
# P9 -- worked examples W1 and W2, every printed digit
# --------------------------------------------------------------------------
PH = {"F": 0, "B": 1, "Fp": 2, "Bp": 3}
BLK = {"0": 0, "1": 1, "E": 2, "H": 3}


def _golden_detail(name, factors):
    gd = load_golden(name)
    o = Oracle(golden_problem(gd, factors))
    gi = find_group(o.group_keys(), gd)
    g = o.groups[gi]
    cf = gd["config"]
    splits = [(g.tp[i], g.dp[i], g.b[i]) for i in range(g.n_splits)]
    sp = splits.index((cf["TP"], cf["DP"], cf["b"]))
    d = o.detail(gi, sp, cf["z"], cf["c"], cf["kW"], cf["kG"], cf["kO"], cf["kA"])
    return gd, d


@pytest.mark.parametrize("name", ["w1_gpt3_1.3b.json", "w2_gpt3_2.7b.json"])
def test_worked_example_phases(name):
    gd, d = _golden_detail(name, "unit")
    for key, (vec, T) in gd["phases_unit"].items():
        ph, blk = PH[key[:-1]], BLK[key[-1]]
        for j in range(4):
            assert _close(d.ch[blk][ph][j], vec[j], 1e-12), (key, j, d.ch[blk][ph][j], vec[j])
        assert _close(d.T[blk][ph], T, 1e-12), (key, d.T[blk][ph], T)
    assert _close(d.p2p, gd["p2p"], 1e-14)


@pytest.mark.parametrize("name", ["w1_gpt3_1.3b.json", "w2_gpt3_2.7b.json"])
@pytest.mark.parametrize("factors", ["unit", "spec"])
def test_worked_example_t_d(name, factors):
    gd, d = _golden_detail(name, factors)
    assert _close(d.t, gd[factors]["t"], 1e-12), (d.t, gd[factors]["t"])
    # d is a difference of phase times: tolerance relative to t (ledger L24)
    assert abs(d.d - gd[factors]["d"]) <= 1e-12 * gd[factors]["t"], (d.d, gd[factors]["d"])


def test_worked_example_w1_memory():
    gd, d = _golden_detail("w1_gpt3_1.3b.json", "unit")
    m = gd["memory"]
    D = m["D"]
    assert d.D == D
    assert d.P_layer == m["P_layer"] and d.P_st == m["P_st"]
    assert d.A_full == m["A_full"] and d.A_bnd == m["A_bnd"]
    assert d.Ms == m["M_s"] * D and d.Mwb == m["M_wb"] * D and d.Mgb == m["M_gb"] * D
    assert d.Mob == m["M_ob"] * D and d.Ma == m["M_a"] * D
    assert d.mem_fwd_D == m["Mem_fwd"] * D and d.mem_bwd_D == m["Mem_bwd"] * D
    assert d.mem == m["mem"] and d.mem * D == m["D_mem"] and d.feasible == 1


def test_worked_example_w2_memory():
    gd, d = _golden_detail("w2_gpt3_2.7b.json", "unit")
    m = gd["memory"]
    D = m["D"]
    assert d.D == D and d.P_st == m["P_st"] and d.A_full == m["A_full"] and d.A_H == m["A_H"]
    assert d.Ms == m["M_s"] * D and d.Mwb == m["M_wb"] * D and d.Mgb == m["M_gb"] * D
    assert d.Mob == m["M_ob"] * D
    assert Fraction(int(d.Ma), D) == Fraction(m["M_a_num"], m["M_a_den"])
    assert Fraction(int(d.mem_fwd_D), D) == Fraction(m["Mem_fwd_num"], m["Mem_fwd_den"])
    assert Fraction(int(d.mem_bwd_D), D) == Fraction(m["Mem_bwd_num"], m["Mem_bwd_den"])
    assert d.mem_bwd_D == m["D_mem"]
    assert d.mem == m["D_mem"] / D  # one IEEE division
    assert d.feasible == 1


# --------------------------------------------------------------------------
# P1-P5, P8 -- closed forms
# --------------------------------------------------------------------------
def _tiny_detail(o, gi, split, z, c, kW=0, kG=0, kO=0, kA=0):
    return o.detail(gi, split, z, c, kW, kG, kO, kA)


def test_model_state_bytes_per_param():
    """P1: ZeRO-0, no offload -> 16 B/param.  P2: ZeRO-3,
    DP=4 -> 4 B/param.  P3: OO=1, ZeRO-0 -> 4 B/param."""
    o = Oracle(workload(2))
    for gi, g in enumerate(o.groups):
        for sp in range(g.n_splits):
            if g.dp[sp] != 4:
                continue
            d0 = _tiny_detail(o, gi, sp, 0, 0)
            assert d0.Ms == 16 * d0.P_st * d0.D
            d3 = _tiny_detail(o, gi, sp, 3, 0)
            assert d3.Ms == 4 * d3.P_st * d3.D
            dO = _tiny_detail(o, gi, sp, 0, 0, kO=o.pb.Q)
            assert dO.Ms == 4 * dO.P_st * dO.D
            return
    pytest.fail("no DP=4 split found")


def test_param_counts_public_models():
    """P4: GPT-3 2.7B layer = 78,653,440 (S:125 '~78.6M'); Llama-2 7B total
    6,738,415,616 (published count; our stage counts exclude the final norm
    vector h); Falcon-40B ~41.8B."""
    o = Oracle(workload(2))
    assert _tiny_detail(o, 0, 0, 0, 0).P_layer == 78_653_440
    for i, target, extra in ((3, 6_738_415_616, 4096), (5, 41.8e9, 0)):
        o = Oracle(workload(i))
        keys = o.group_keys()
        gi = next(k for k, key in enumerate(keys) if key[1] == 1 and key[2] == 1)
        g = o.groups[gi]
        sp = [g.tp[s] for s in range(g.n_splits)].index(1) if 1 in list(g.tp)[:g.n_splits] else None
        if sp is None:  # single-stage group with TP=1 absent -> scale back
            sp = 0
        d = _tiny_detail(o, gi, sp, 0, 0)
        total = d.P_st * g.tp[sp] + extra
        if i == 3:
            assert total == target
        else:
            assert abs(total - target) / target < 0.005


def test_activation_closed_form():
    """P5: non-gated MHA with f = 4h: A_full = sbh(8 + 24/TP) + 2 a s^2 b / TP
    (Korthikanti et al. minus the dropout terms); flash drops the s^2 term."""
    for fl in (0, 1):
        pb = tiny(4, 4, 1, 4, 8, 1, h=64, s=128, fl=fl)
        o = Oracle(pb)
        m = pb.model
        for gi, g in enumerate(o.groups):
            for sp in range(g.n_splits):
                tp, b = g.tp[sp], g.b[sp]
                d = _tiny_detail(o, gi, sp, 0, 0)
                expect = m.s * b * m.h * (8 + Fraction(24, tp)) + (1 - fl) * Fraction(2 * m.a * m.s ** 2 * b, tp)
                assert Fraction(d.A_full) == expect
                assert d.A_bnd == 2 * m.s * b * m.h


def test_degenerate_stage():
    """P8: DP=1, ratios 0, not first/last -> d = 0, and a
    checkpointed layer adds exactly one forward (Tf + ARtp_f) to B's compute."""
    pb = tiny(4, 4, 1, 4, 8, 2)
    o = Oracle(pb)
    seen = 0
    for gi, g in enumerate(o.groups):
        if g.first or g.last:
            continue
        for sp in range(g.n_splits):
            if g.dp[sp] != 1:
                continue
            for z in range(4):
                for c in range(g.l + 1):
                    d = _tiny_detail(o, gi, sp, z, c)
                    assert d.d == 0.0
                    assert _close(d.ch[1][1][0] - d.ch[0][1][0], d.ch[0][0][0], 1e-14)
                    seen += 1
    assert seen > 0


# --------------------------------------------------------------------------
# P10 -- enumeration counts
# --------------------------------------------------------------------------
def test_tiny_enumeration_exact():
    """P10: L=2, heads=2, 1x2, B=2, Q=1 -> 6 groups / 1,088 configs and the
    listed groups; (B=4, Q=2) -> 9 / 8,748; L=4, heads=4, 1x4, B=8, Q=1 -> 68 / 18,496."""
    o = Oracle(tiny(2, 2, 1, 2, 2, 1))
    assert (o.n_groups, o.n_configs) == (6, 1088)
    assert o.group_keys() == [(1, 0, 1, 1, 1, 1, 1), (1, 1, 0, 1, 1, 1, 1), (1, 1, 1, 1, 2, 1, 2),
                              (2, 0, 1, 1, 1, 1, 1), (2, 1, 0, 2, 1, 1, 1), (2, 1, 1, 1, 2, 1, 2)]
    o = Oracle(tiny(2, 2, 1, 2, 4, 2))
    assert (o.n_groups, o.n_configs) == (9, 8748)
    o = Oracle(tiny(4, 4, 1, 4, 8, 1))
    assert (o.n_groups, o.n_configs) == (68, 18496)


@pytest.mark.parametrize("i,groups,tuples,configs", [
    (1, 1066, 75476, 47172500),
    (2, 4569, 501492, 7342344372),
    (3, 11917, 1412836, 274769758116),
    (4, 52784, 9603260, 63006988860),
    (5, 125230, 27496640, 186020296424640),
])
def test_workload_space_sizes(i, groups, tuples, configs):
    """SURVEY Sec. 8(d) table (exact counts from an independent scratch counter)."""
    o = Oracle(workload(i))
    assert o.n_groups == groups
    assert o.n_tuples() == tuples
    assert o.n_configs == configs
    # closed form: sum over groups n_splits * 4 * (l+1) * (Q+1)^4
    R = (o.pb.Q + 1) ** 4
    assert sum(g.n_splits * 4 * (g.l + 1) * R for g in o.groups) == configs


def test_submesh_rule_spec_example():
    """S:533 N=4, M=8 -> submeshes (1,1),(1,2),(1,4),(1,8),(2,8),(3,8),(4,8):
    the set of (n, m) pairs appearing in the groups is exactly that list.  (B is
    chosen divisible by 3 so that the 24-GPU submesh has a valid DP split.)"""
    from synth import make_coeffs
    o = Oracle(make_coeffs(workload(4).replace(B=96)))
    assert sorted({(k[5], k[6]) for k in o.group_keys()}) == [(1, 1), (1, 2), (1, 4), (1, 8), (2, 8), (3, 8), (4, 8)]


# --------------------------------------------------------------------------
# P11/P12 -- frontier
# --------------------------------------------------------------------------
def test_spec_frontier_example():
    """(t,d) = (10,5) and (9,6) both kept; (11,6) dropped."""
    from oracle.binding import POINT_DTYPE, frontier_points
    pts = np.zeros(3, dtype=POINT_DTYPE)
    pts["t"], pts["y"], pts["idx"] = [10, 9, 11], [5, 6, 6], [0, 1, 2]
    for method in (1, 2):
        fr = frontier_points(pts, method)
        assert sorted(fr["idx"].tolist()) == [0, 1]
        assert fr["t"].tolist() == [9.0, 10.0]   # sorted by x, y strictly descending
