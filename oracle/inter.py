"""Inter-stage oracle (Eq. 1-3) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module.  The
product package ``paper_2503_19050_b200`` never imports it; it shares no code
with ``paper_2503_19050_b200/csrc/mist_inter.cpp``.

Plain pure-Python loops, for small instances only.  Every function cites the
passage it follows (``P:n`` = PAPER.md line n, ``S:n`` = SPEC.md line n; the
readings I1-I4 are listed in DESIGN.md section 8).

  objective         Eq. 2 written out (L4 reads the inner sum as t_j)
  simulate          the pipeline recurrence of the SPEC, a second model
  closed_form       its closed form
  stage_key         the IntraStagePareto key of stage i of S (Eq. 3; O2)
  brute_force_plan  argmin of Eq. 2 over every selection: every G, S,
                    layer composition, submesh sequence and candidate point
"""
from __future__ import annotations

import itertools
from typing import Dict, List, Optional, Sequence, Tuple


def objective(G: int, t: Sequence[float], d: Sequence[float]) -> float:
    """Eq. 2: (G-1) max_i t_i + sum_i t_i + max_i (d_i - sum_{j<i} t_j).

    Reading L4: the inner sum of the third term is over t_j (the paper prints t_i)."""
    S = len(t)
    if S == 0 or len(d) != S:
        raise ValueError("objective: empty or mismatched stage list")
    first = (G - 1) * max(t)
    second = 0.0
    for i in range(S):
        second += t[i]
    third = None
    for i in range(S):
        before = 0.0
        for j in range(i):
            before += t[j]
        v = d[i] - before
        third = v if third is None or v > third else third
    return first + second + third


def simulate(G: int, t: Sequence[float], d: Sequence[float]) -> float:
    """SPEC's event recurrence: F(i,k) = max(F(i-1,k), F(i,k-1)) + t_i,
    F(0,k) = 0, F(i,0) = d_i (stage i's first-microbatch extra work runs from time 0,
    hidden in the bubble); makespan = F(S, G)."""
    S = len(t)
    F = [[0.0] * (G + 1) for _ in range(S + 1)]
    for i in range(1, S + 1):
        F[i][0] = d[i - 1]
    for k in range(1, G + 1):
        for i in range(1, S + 1):
            F[i][k] = max(F[i - 1][k], F[i][k - 1]) + t[i - 1]
    return F[S][G]


def closed_form(G: int, t: Sequence[float], d: Sequence[float]) -> float:
    """max over j in {0..S} of d_j + sum_{m>=j} t_m + (G-1) max_{m>=j} t_m,
    with d_0 = 0 and the j = 0 term over the whole pipeline."""
    S = len(t)
    best = None
    for j in range(0, S + 1):
        lo = 0 if j == 0 else j - 1          # stage index (0-based) the suffix starts at
        dj = 0.0 if j == 0 else d[j - 1]
        suf = 0.0
        for m in range(lo, S):
            suf += t[m]
        mx = max(t[lo:])
        v = dj + suf + (G - 1) * mx
        best = v if best is None or v > best else best
    return best


def stage_key(G: int, S: int, i: int, l: int, n: int, m: int) -> Tuple[int, ...]:
    """Stage i (1-based) of S as an IntraStagePareto key (Eq. 3; O2):
    (G, first = [i = 1], last = [i = S], w = min(G, S - i + 1), l, n, m)."""
    return (G, int(i == 1), int(i == S), min(G, S - i + 1), l, n, m)


def brute_force_plan(cands: Dict[Tuple[int, ...], Sequence[Tuple[float, float]]], L: int,
                     devices: int, max_stages: Optional[int] = None):
    """Argmin of Eq. 2 over every selection.

    cands: key (G, first, last, w, l, n, m) -> list of (t, d) candidate points
    (a group's frontier, or its alpha-samples).  A plan picks G, S and, per
    stage i, l_i >= 1, a submesh (n_i, m_i) and a point of cands[stage_key(...)],
    with sum l_i = L and sum n_i m_i = devices.

    Returns (value, plan) where plan = (G, [(key, point position)...]) for stage
    1..S, or (None, None) when no plan exists.  Exhaustive: small inputs only."""
    Gs = sorted({k[0] for k in cands})
    meshes = sorted({(k[5], k[6]) for k in cands})
    Smax = min(L, devices) if max_stages is None else min(L, devices, max_stages)
    best_v, best_p = None, None
    for G in Gs:
        for S in range(1, Smax + 1):
            for comp in _compositions(L, S):
                for ms in itertools.product(meshes, repeat=S):
                    if sum(n * m for n, m in ms) != devices:
                        continue
                    keys = [stage_key(G, S, i + 1, comp[i], ms[i][0], ms[i][1]) for i in range(S)]
                    if any(k not in cands or len(cands[k]) == 0 for k in keys):
                        continue
                    for pick in itertools.product(*[range(len(cands[k])) for k in keys]):
                        t = [cands[keys[i]][pick[i]][0] for i in range(S)]
                        d = [cands[keys[i]][pick[i]][1] for i in range(S)]
                        v = objective(G, t, d)
                        if best_v is None or v < best_v:
                            best_v, best_p = v, (G, list(zip(keys, pick)))
    return best_v, best_p


def _compositions(L: int, S: int):
    """All (l_1..l_S) with l_i >= 1 and sum = L."""
    for cuts in itertools.combinations(range(1, L), S - 1):
        prev, out = 0, []
        for c in cuts + (L,):
            out.append(c - prev)
            prev = c
        yield tuple(out)


def plan_value(G: int, stages: List[Tuple[float, float]]) -> float:
    """Eq. 2 of a plan given as [(t_i, d_i)] for stage 1..S."""
    return objective(G, [s[0] for s in stages], [s[1] for s in stages])
