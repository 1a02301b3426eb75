"""Host helpers of the product's C ABI that need no device (sigma, q1_shape, detect_cycles), checked
against the oracle's restatements of model.cpp:19-26, fem.cpp:76-96 and solver.cpp:10-22."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def cf():
    import paper_1806_09924_b200 as cf
    return cf


def test_sigma_matches_oracle(cf, orc):
    rng = np.random.default_rng(3)
    for d in (2, 3):
        for _ in range(20):
            g = rng.standard_normal((3, 3))
            kw = dict(E=float(rng.uniform(0.5, 2)), nu=float(rng.uniform(0.0, 0.45)))
            assert np.array_equal(cf.sigma(g, cf.Material(**kw), d), orc.sigma(g, orc.material(**kw), d))


def test_q1_shape_matches_oracle_tables(cf, orc):
    for d in (2, 3):
        pts, _, shape, grads = orc.qp_tables(d)
        for q in range(1 << d):
            v, g = cf.q1_shape(d, pts[q, :d])
            assert np.array_equal(v, shape[q]) and np.array_equal(g, grads[q, :, :d])
        v, g = cf.q1_shape(d, [0.25, 0.5, 0.75][:d])
        assert abs(v.sum() - 1.0) < 1e-15 and np.abs(g.sum(axis=0)).max() < 1e-15


def test_detect_cycles_matches_oracle(cf, orc):
    rng = np.random.default_rng(4)
    hist = {int(k): list(rng.integers(0, 2, int(rng.integers(0, 14)))) for k in rng.choice(1000, 60, replace=False)}
    for window, toggles in ((8, 3), (4, 2), (16, 5), (1, 1)):
        keys = list(hist)
        flags = orc.detect_cycles([hist[k] for k in keys], window, toggles)
        expect = {k for k, f in zip(keys, flags) if f}
        assert cf.detect_cycles(hist, window, toggles) == expect
    assert cf.detect_cycles({}, 8, 3) == set()
