"""Alg. 1 over observation tables and its fitting on the GPU
against the oracle (literal Alg. 1, oracle/intf.py's F1-F3 step by step).

* mist_pred_intf == the oracle's Alg. 1 row by row (R3: reciprocal vs division,
  a few ulp), and the identities: one nonzero channel returns it, unit factors
  return the max.
* The loss of a table (iters = 0) == orc_intf_loss.
* The fit == the oracle's fit on the same observations: identical factors up to
  rounding, unless a grid decision met a near-tie of the loss, in which case the
  two losses must still agree.
* Round trip at scale: recovered factors predict held-out rows within 1%."""
import numpy as np
import pytest

from oracle import intf
from oracle.binding import intf_loss, pred_intf_batch
from paper_2503_19050_b200 import mist
from synth import factor_table, intf_rows, noise, random_factor_table

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

UNIT = [[1.0] * 4 for _ in range(16)]


@pytest.fixture(scope="module")
def ctx():
    from paper_2503_19050_b200 import build
    build.build()
    c = mist.Context(0)
    yield c
    c.close()


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


@pytest.mark.parametrize("table", ["unit", "spec", "asym", "rand"])
def test_pred_intf_parity(ctx, table):
    F = random_factor_table(5) if table == "rand" else factor_table(table)
    X = intf_rows(11, 100_003)
    X[:7] = 0.0                                          # all-zero rows
    T = mist.mist_pred_intf(ctx, _dev(X), F).cpu().numpy()
    ref = pred_intf_batch(X, F)
    np.testing.assert_allclose(T, ref, rtol=1e-13, atol=0)
    one = np.count_nonzero(X, axis=1) <= 1
    assert np.array_equal(T[one], X[one].sum(1))         # identity: a single channel is returned
    if table == "unit":
        np.testing.assert_allclose(T, X.max(1), rtol=1e-14, atol=0)


def test_loss_parity(ctx):
    X = intf_rows(12, 5000, min_channels=2)
    Ft = random_factor_table(12)
    Tobs = pred_intf_batch(X, Ft) * noise(12, 5000, 0.05)
    for F in (UNIT, Ft, factor_table("spec")):
        _, loss = mist.mist_fit_intf(ctx, _dev(X), _dev(Tobs), F, iters=0)
        assert loss == pytest.approx(intf_loss(X, Tobs, F), rel=1e-12)


@pytest.mark.parametrize("trial", [0, 1, 2])
def test_fit_parity(ctx, trial):
    Ft = random_factor_table(20 + trial)
    X = intf_rows(20 + trial, 257, min_channels=2)
    Tobs = pred_intf_batch(X, Ft) * noise(20 + trial, 257, 0.03 * trial)
    F, loss = mist.mist_fit_intf(ctx, _dev(X), _dev(Tobs), UNIT, iters=2, fmax=3.0)
    Fo, lo = intf.fit(X, Tobs, UNIT, iters=2, fmax=3.0)
    assert loss == pytest.approx(lo, rel=1e-9)
    if not np.allclose(F, Fo, rtol=1e-9, atol=0):
        # a grid decision met a near-tie: the loss of each side's table must agree
        assert intf_loss(X, Tobs, F) == pytest.approx(intf_loss(X, Tobs, Fo), rel=1e-9)
    assert loss == pytest.approx(intf_loss(X, Tobs, F), rel=1e-12)


@pytest.mark.parametrize("trial", [0, 1, 2, 3])
def test_round_trip_scale(ctx, trial):
    Ft = random_factor_table(40 + trial)
    X = intf_rows(40 + trial, 20_000, min_channels=2)
    T = pred_intf_batch(X, Ft)
    Xh = intf_rows(140 + trial, 5000, min_channels=2)
    Th = pred_intf_batch(Xh, Ft)
    F, loss = mist.mist_fit_intf(ctx, _dev(X), _dev(T), UNIT, iters=30, fmax=3.0)
    err = np.abs(pred_intf_batch(Xh, F) - Th) / Th
    assert err.mean() <= 0.01
    Fn, _ = mist.mist_fit_intf(ctx, _dev(X), _dev(T * noise(40 + trial, len(T), 0.05)), UNIT, iters=30, fmax=3.0)
    errn = np.abs(pred_intf_batch(Xh, Fn) - Th) / Th
    assert errn.mean() <= 0.03


def test_errors(ctx):
    X = intf_rows(13, 64)
    T = np.ones(64)
    bad = X.copy()
    bad[5, 2] = -1.0
    with pytest.raises(mist.MistError):
        mist.mist_fit_intf(ctx, _dev(bad), _dev(T), UNIT)
    T0 = T.copy()
    T0[3] = 0.0
    with pytest.raises(mist.MistError):
        mist.mist_fit_intf(ctx, _dev(X), _dev(T0), UNIT)
    F = [row[:] for row in UNIT]
    F[3][0] = 0.5
    with pytest.raises(mist.MistError):
        mist.mist_pred_intf(ctx, _dev(X), F)
