"""FieldRegressor (estimator.py of the reference) on the device."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _points(n, seed):
    r = np.random.default_rng(seed)
    X = r.random((n, 3))
    y = 3.0 + 2.0 * np.exp(-((X - 0.5) ** 2).sum(1) / (2 * 0.18 ** 2))   # a gaussian blob, offset / scaled
    return X, y


def test_field_regressor_fits_and_predicts(nv):
    from paper_2207_11620_b200.estimator import FieldRegressor
    X, y = _points(20000, 0)
    Xt, yt = _points(2000, 1)
    est = FieldRegressor(n_levels=6, log2_hashmap_size=14, n_steps=300, batch_size=4096, seed=2)
    assert est.fit(X, y) is est
    assert est.n_features_in_ == 3 and len(est.history_.losses) == 300
    assert est.history_.losses[-1] < est.history_.losses[0]
    assert est.score(Xt, yt) > 0.95
    lo, hi = est.value_range_
    assert lo == pytest.approx(y.min()) and hi == pytest.approx(y.max())


def test_field_regressor_protocol_and_errors(nv):
    from paper_2207_11620_b200.estimator import FieldRegressor
    est = FieldRegressor(n_steps=5)
    assert est.get_params()["n_steps"] == 5
    assert repr(est) == "FieldRegressor(n_steps=5)"
    assert est.set_params(seed=3).seed == 3
    with pytest.raises(ValueError, match="invalid parameter"):
        est.set_params(bogus=1)
    with pytest.raises(ValueError, match="not fitted"):
        est.predict(np.zeros((2, 3)))
    with pytest.raises(ValueError, match="unit cube"):
        est.fit(np.full((4, 3), 1.5), np.zeros(4))
    with pytest.raises(ValueError, match="shape"):
        est.fit(np.zeros((4, 2)), np.zeros(4))
    X, y = _points(4096, 3)
    est = FieldRegressor(n_levels=4, log2_hashmap_size=12, batch_size=4096, seed=1)
    est.partial_fit(X, y).partial_fit(X, y)
    assert est.model_.opt.t == 2 and len(est.history_.losses) == 2


def test_field_regressor_same_seed_same_model(nv):
    """Same seed -> the same model bit for bit, and fit() does not resume (test_estimator.py:63-75):
    the estimator trains with ordered reductions; the global mode is restored afterwards."""
    from paper_2207_11620_b200 import encoding
    from paper_2207_11620_b200.estimator import FieldRegressor
    X, y = _points(1024, 4)
    mk = lambda: FieldRegressor(n_levels=4, log2_hashmap_size=12, n_steps=40, batch_size=512, seed=7)  # noqa: E731
    a = mk().fit(X, y).predict(X[:64])
    est = mk()
    b = est.fit(X, y).predict(X[:64])
    c = est.fit(X, y).predict(X[:64])
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(b, c)
    assert not encoding.deterministic()
