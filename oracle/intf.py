"""Interference-factor fitting oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` may import this
module; the product (``paper_2503_19050_b200/csrc/mist_intf.cu``) shares no
code with it.

The paper fits Alg. 1's slowdown factors "data-driven": "different shapes and
combinations of concurrent kernels are sampled and benchmarked, and the
resulting runtime data is used to train the slowdown factors".  It
names no procedure.  Reading F1-F3, after S:212-220:

  F1  loss = mean over observations of ((PredINTF(X_i) - T_i) / T_i)^2
      (orc_intf_loss, the literal Alg. 1 row by row);
  F2  coordinate descent over the 28 member factors (masks with >= 2 channels,
      pattern ascending, member channel ascending), ``iters`` sweeps;
  F3  per coordinate, a derivative-free search over [1, fmax]: LEVELS nested
      grids of GRID points, each centred on the best value so far with half-width
      one step of the previous grid (lower end clamped at 1); a grid value
      replaces the current one only if its loss is strictly lower (ties: the
      smallest grid index), so the loss never increases.
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np

from .binding import intf_loss

GRID = 31
LEVELS = 3


def coords() -> List[Tuple[int, int]]:
    """The 28 fitted factors: (pattern, channel) with popcount(pattern) >= 2 and
    the channel a member (F2).  Channel bits C=1, NCCL=2, H2D=4, D2H=8 (O7)."""
    out = []
    for pat in range(16):
        if bin(pat).count("1") < 2:
            continue
        for ch in range(4):
            if pat >> ch & 1:
                out.append((pat, ch))
    return out


def fit(X: np.ndarray, Tobs: np.ndarray, init, iters: int = 2, fmax: float = 4.0):
    """F1-F3 step by step.  Returns (factors[16][4], loss)."""
    F = np.array(init, dtype=np.float64).reshape(16, 4).copy()
    for _ in range(iters):
        for pat, ch in coords():
            best = F[pat, ch]
            best_loss = intf_loss(X, Tobs, F)
            lo, hi = 1.0, fmax
            for _lev in range(LEVELS):
                grid = [lo + (hi - lo) * k / (GRID - 1) for k in range(GRID)]
                losses = []
                for v in grid:
                    G = F.copy()
                    G[pat, ch] = v
                    losses.append(intf_loss(X, Tobs, G))
                k = int(np.argmin(losses))           # first minimum
                if losses[k] < best_loss:
                    best, best_loss = grid[k], losses[k]
                w = (hi - lo) / (GRID - 1)
                lo, hi = max(1.0, best - w), best + w
            F[pat, ch] = best
    return F, intf_loss(X, Tobs, F)
