"""Diagnostic (not collected): GPU dense values vs oracle for given indices.
    python tests/diag_pairs.py 1 205651 205751 55000 55001
"""
import sys

import numpy as np
import torch

from oracle.binding import Oracle
from paper_2503_19050_b200 import mist
from synth import workload

pb = workload(int(sys.argv[1]))
idx = np.array([int(x) for x in sys.argv[2:]], dtype=np.uint64)
o, s = Oracle(pb), mist.Spec(pb)
ctx = mist.Context(0)
ti = torch.from_numpy(idx.astype(np.int64)).cuda()
t = torch.empty(len(idx), dtype=torch.float64, device="cuda")
d, m = torch.empty_like(t), torch.empty_like(t)
f = torch.empty(len(idx), dtype=torch.uint8, device="cuda")
mist.mist_eval_stage_costs_at(ctx, s, ti, t, d, m, f)
e = o.eval_indices(idx)
R = (pb.Q + 1) ** 4
for k, i in enumerate(idx.tolist()):
    r = i % R
    Q1 = pb.Q + 1
    kA = r % Q1; kO = (r // Q1) % Q1; kG = (r // Q1 ** 2) % Q1; kW = r // Q1 ** 3
    print(f"idx {i} tuple {i // R} (kW,kG,kO,kA)=({kW},{kG},{kO},{kA})")
    print(f"   gpu t={t[k].item()!r} d={d[k].item()!r}   oracle t={e['t'][k]!r} d={e['d'][k]!r}")
# the frontier kernel's own values
pts, offs, _, _ = mist.mist_pareto_frontier(ctx, s)
for i in idx.tolist():
    w = np.nonzero(pts["idx"] == i)[0]
    print(i, "in GPU frontier:" , [(pts[j]["t"], pts[j]["y"]) for j in w])
ctx.close()
