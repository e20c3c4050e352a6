"""Diagnostic (not collected): where the GPU and oracle frontiers of one workload
differ in membership, print the differing points and their nearest partners.
    python tests/diag_ties.py 1
"""
import sys

import numpy as np

from oracle.binding import Oracle
from paper_2503_19050_b200 import mist
from synth import workload

i = int(sys.argv[1]) if len(sys.argv) > 1 else 1
pb = workload(i)
o, s = Oracle(pb), mist.Spec(pb)
ref = o.sweep()
ctx = mist.Context(0)
pts, offs, _, _ = mist.mist_pareto_frontier(ctx, s)
ndiff = 0
shown = 0
kinds = {}
R = (pb.Q + 1) ** 4
for g in range(o.n_groups):
    G = pts[offs[g]:offs[g + 1]]
    O = ref["points"][ref["offsets"][g]:ref["offsets"][g + 1]]
    gi, oi = set(G["idx"].tolist()), set(O["idx"].tolist())
    if gi == oi:
        continue
    ndiff += 1
    for p in G:
        if int(p["idx"]) in oi:
            continue
        # partner: oracle point with the same t (closest)
        j = np.argmin(np.abs(O["t"] - p["t"]))
        q = O[j]
        e = o.eval_indices(np.array([p["idx"], q["idx"]], dtype=np.uint64))
        dt = (p["t"] - q["t"]) / q["t"]
        key = ("same_t" if q["t"] == p["t"] else "t_ulps", "same_y" if q["y"] == p["y"] else "y_diff")
        kinds[key] = kinds.get(key, 0) + 1
        if shown < 8:
            shown += 1
            ip, iq = int(p["idx"]), int(q["idx"])
            print(f"g{g} GPU-only idx={ip} (tuple {ip // R}, r {ip % R}) t={p['t']!r} y={p['y']!r}")
            print(f"     oracle idx={iq} (tuple {iq // R}, r {iq % R}) t={q['t']!r} y={q['y']!r}  rel dt={dt:.2e}")
            print(f"     oracle eval of both: t={e['t'].tolist()} d={e['d'].tolist()}")
print("groups with membership differences:", ndiff, "of", o.n_groups, "kinds:", kinds)
ctx.close()
