"""Quantisation thresholds (host side of the LUT exactness argument)."""
import numpy as np
import pytest

from paper_2512_16609_b200.quant import compute_thresholds, quantize_chain


@pytest.mark.parametrize("gamma", [1.2, 1.0, 2.0, 0.5, 1.7, 3.3, 0.9])
def test_thresholds_reproduce_chain(gamma):
    thr = compute_thresholds(gamma)
    assert thr.shape == (256,) and np.all(np.diff(thr[1:]) > 0)
    rng = np.random.default_rng(int(gamma * 100))
    x = np.concatenate([rng.random(200_000), thr[1:], np.nextafter(thr[1:], -1.0), [0.0, 1.0, 0.25, 0.5]])
    x = np.clip(x, 0.0, 1.0)
    q = quantize_chain(x, gamma).astype(np.int64)
    assert np.array_equal(q, np.searchsorted(thr[1:], x, side="right"))


def test_chain_matches_oracle(oracle):
    x = np.random.default_rng(3).random(10_000)
    for g in (1.2, 1.0):
        assert np.array_equal(quantize_chain(x, g), oracle.quantize_after_gamma(x, g))
