"""Interference-factor fitting oracle (Alg. 1).

CPU pins of oracle/intf.py (readings F1-F3).  The fitted values
are not unique, so the fit is pinned by what any correct F1-F3 procedure must
do: recover synthetic factors (held-out predictions), never end worse than its
start, keep a table that already fits exactly, and leave the factors alone when
no observation exercises them.  The GPU side is in tests/test_gpu_intf.py."""
import numpy as np
import pytest

from oracle import intf
from oracle.binding import intf_loss, pred_intf, pred_intf_batch
from synth import intf_rows, noise, random_factor_table

UNIT = [[1.0] * 4 for _ in range(16)]


def test_coords():
    c = intf.coords()
    assert len(c) == 28                                  # 6 pairs x 2 + 4 triples x 3 + 1 quad x 4 (D7)
    assert c[0] == (3, 0) and c[-1] == (15, 3)


def test_batch_equals_rows():
    X = intf_rows(1, 200)
    F = random_factor_table(1)
    T = pred_intf_batch(X, F)
    assert all(T[i] == pred_intf(X[i], F) for i in range(len(X)))


def test_loss_definition():
    X = intf_rows(2, 50, min_channels=2)
    F = random_factor_table(2)
    T = pred_intf_batch(X, F)
    assert intf_loss(X, T, F) == 0.0
    assert intf_loss(X, 2.0 * T, F) == pytest.approx(0.25, rel=1e-12)    # ((T - 2T) / 2T)^2


def test_fixed_point_and_never_worse():
    X = intf_rows(3, 120, min_channels=2)
    Ft = random_factor_table(3)
    T = pred_intf_batch(X, Ft)
    F, loss = intf.fit(X, T, Ft, iters=1)
    assert loss == 0.0 and np.array_equal(F, np.array(Ft))          # nothing is strictly better
    Tn = T * noise(3, len(T), 0.05)
    l0 = intf_loss(X, Tn, UNIT)
    F2, l2 = intf.fit(X, Tn, UNIT, iters=1)
    assert l2 <= l0


def test_single_channel_rows_leave_factors():
    X = intf_rows(4, 80)
    X = X * (np.arange(4)[None, :] == (np.arange(80) % 4)[:, None])   # one channel per row
    X[X.sum(1) == 0, 0] = 1e-3
    T = X.sum(1) * 1.1
    F, _ = intf.fit(X, T, UNIT, iters=1)
    assert np.array_equal(F, np.array(UNIT))                          # loss flat in every factor


@pytest.mark.parametrize("trial", [0, 1])
def test_round_trip(trial):
    Ft = random_factor_table(trial)
    X = intf_rows(trial, 300, min_channels=2)
    T = pred_intf_batch(X, Ft)
    Xh = intf_rows(100 + trial, 2000, min_channels=2)
    Th = pred_intf_batch(Xh, Ft)
    F, loss = intf.fit(X, T, UNIT, iters=30, fmax=3.0)
    err = np.abs(pred_intf_batch(Xh, F) - Th) / Th
    assert err.mean() <= 0.01 and np.quantile(err, 0.9) <= 0.01
