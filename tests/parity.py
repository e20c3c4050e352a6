"""Comparison helpers for CUDA-vs-oracle parity (tolerances from BASELINE.json
north_star: 'relative error of 1e-9 (fp64)'; reading L24/L26)."""
import numpy as np

REL = 1e-9


def compare_dense(gpu, orc, label=""):
    """Element-wise: feasibility bit-exact; mem bit-exact wherever the oracle's
    D*mem is below 2^52 (all feasible configs), else 1e-12 relative; t within
    1e-9 relative; d within 1e-9 * (d + t)."""
    fe_g, fe_o = np.asarray(gpu["feasible"]).astype(np.uint8), np.asarray(orc["feasible"]).astype(np.uint8)
    bad = np.nonzero(fe_g != fe_o)[0]
    assert len(bad) == 0, f"{label}: feasibility differs at {bad[:10]}"
    mg, mo = np.asarray(gpu["mem"]), np.asarray(orc["mem"])
    exact = fe_o == 1
    assert np.array_equal(mg[exact], mo[exact]), f"{label}: feasible mem not bit-exact"
    rel = np.abs(mg - mo) / np.maximum(np.abs(mo), 1e-300)
    assert rel.max(initial=0) <= 1e-12, f"{label}: mem rel err {rel.max()}"
    tg, to = np.asarray(gpu["t"]), np.asarray(orc["t"])
    et = np.abs(tg - to) / to
    assert et.max(initial=0) <= REL, f"{label}: t rel err {et.max()} at {np.argmax(et)}"
    dg, do = np.asarray(gpu["d"]), np.asarray(orc["d"])
    ed = np.abs(dg - do) / (do + to)
    assert ed.max(initial=0) <= REL, f"{label}: d err {ed.max()} at {np.argmax(ed)}"
    assert np.all(dg >= 0)
    return dict(t=et.max(initial=0), d=ed.max(initial=0), n=len(to))


def _near_beaten(p, pts):
    """L26: p is acceptable iff the other side has q with x_q <= x_p (1+tol)
    and y_q <= y_p + tol (y_p + t_p)."""
    if len(pts) == 0:
        return False
    ok = (pts["t"] <= p["t"] * (1 + REL)) & (pts["y"] <= p["y"] + REL * (p["y"] + p["t"]))
    ok &= pts["idx"] != p["idx"]
    return bool(ok.any())


def compare_frontiers(g_pts, g_off, o_pts, o_off, groups=None, label=""):
    """Per group: identical membership except ties within tolerance; values of
    common points within tolerance.  g_off/o_off index the two point arrays
    (o_off may cover a subset of groups, given by ``groups``)."""
    ng = len(o_off) - 1
    groups = list(range(ng)) if groups is None else list(groups)
    stats = dict(groups=0, points=0, tie_diffs=0)
    for k, g in enumerate(groups):
        G = g_pts[g_off[g]:g_off[g + 1]]
        O = o_pts[o_off[k]:o_off[k + 1]]
        stats["groups"] += 1
        stats["points"] += len(O)
        gi, oi = set(G["idx"].tolist()), set(O["idx"].tolist())
        if gi != oi:
            for p in G:
                if int(p["idx"]) not in oi:
                    assert _near_beaten(p, O), f"{label} group {g}: GPU-only point {p} not near-beaten"
                    stats["tie_diffs"] += 1
            for p in O:
                if int(p["idx"]) not in gi:
                    assert _near_beaten(p, G), f"{label} group {g}: oracle-only point {p} not near-beaten"
                    stats["tie_diffs"] += 1
        common = np.intersect1d(G["idx"], O["idx"])
        if len(common):
            gm = {int(p["idx"]): p for p in G}
            for p in O:
                q = gm.get(int(p["idx"]))
                if q is None:
                    continue
                assert abs(q["t"] - p["t"]) <= REL * p["t"], (label, g, p, q)
                assert abs(q["y"] - p["y"]) <= REL * (abs(p["y"]) + p["t"]), (label, g, p, q)
                assert q["mem"] == p["mem"], (label, g, p, q)
        # sorted by t ascending, y strictly descending
        assert np.all(np.diff(G["t"]) > 0) and np.all(np.diff(G["y"]) < 0), f"{label} group {g} order"
    return stats


def frontier_fp_and_bench(ctx, spec, **kw):
    """The sweep twice: with fingerprints (feasible-set check; every feasible
    config is visited) and without (the bench's launch path, where the exact
    skips R4/R5/R7 cut whole runs).  Both must return the same frontier bit for
    bit; returns the fingerprinted call's (points, offsets, fp_count, fp_hash)."""
    from paper_2503_19050_b200 import mist
    pts, offs, fc, fh = mist.mist_pareto_frontier(ctx, spec, fingerprints=True, **kw)
    p2, o2, _, _ = mist.mist_pareto_frontier(ctx, spec, **kw)
    assert np.array_equal(offs, o2), "bench-path frontier: group sizes differ from the fingerprinted sweep"
    assert p2.tobytes() == pts.tobytes(), "bench-path frontier differs from the fingerprinted sweep"
    return pts, offs, fc, fh
