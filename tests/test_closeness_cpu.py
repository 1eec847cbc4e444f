"""CPU: the comparison helpers the GPU tests use for results that depend on the order of floating-point atomics
(tests/closeness.py) accept what they document and reject what the tests rely on them to reject."""
import numpy as np
import pytest

from closeness import assert_tables_match, sums_close


def test_sums_close_scales_with_the_largest_entry():
    want = np.array([1.0, 1e-3, 3e-17])          # the last entry: a near-complete cancellation
    assert sums_close(want * (1 + 5e-13), want, 1e-12)
    assert sums_close(want + np.array([0, 0, 5e-14]), want, 1e-12)        # off by 1e3 x itself, 5e-14 of the largest
    assert not sums_close(want + np.array([0, 1e-9, 0]), want, 1e-12)     # a real difference in a mid-sized entry
    assert not sums_close(want * (1 + 1e-9), want, 1e-12)


def test_tables_match_accepts_one_branch_flip_and_rejects_a_missing_contribution():
    rng = np.random.default_rng(0)
    want = rng.standard_normal(200_000) * 1e-2
    noise = rng.standard_normal(want.size) * 1e-8
    assert_tables_match(want + noise, want, 2e-5)
    flipped = want + noise
    flipped[rng.choice(want.size, 600, replace=False)] += 3e-3          # 0.3 % of the entries, a fraction of lr away
    assert_tables_match(flipped, want, 2e-5)
    too_many = want + noise
    too_many[rng.choice(want.size, 4000, replace=False)] += 3e-3        # 2 %: not one flipped sign any more
    with pytest.raises(AssertionError):
        assert_tables_match(too_many, want, 2e-5)
    too_far = want + noise
    too_far[7] += 0.2                                                    # further than a few Adam steps can carry an entry
    with pytest.raises(AssertionError):
        assert_tables_match(too_far, want, 2e-5)
    # a rank's contribution missing from a third of the rows
    with pytest.raises(AssertionError):
        assert_tables_match(np.where(np.arange(want.size) % 3 == 0, want * 0.5, want), want, 2e-5)
