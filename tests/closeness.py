"""Comparison helpers shared by the GPU tests for results that depend on the ORDER of floating-point atomics.

Two runs of the same kernels on the same data differ in the order their fp32 (tables) or fp64 (MLP) partial sums meet.  That
moves a sum by one rounding of its summands -- and two things amplify it beyond a plain tolerance:
  * an entry that is a near-complete cancellation carries the rounding relative to its summands, not to itself;
  * Adam (update = lr * m / (sqrt(v) + 1e-15)) turns the SIGN of such a near-zero gradient component into a full lr-sized
    step, so after a few steps one or two of ~10^5 updated table entries can sit ~lr away from their twin (observed about
    once in ten runs of tests/cpp/sharded_train_check.cpp).
"""
import numpy as np


def sums_close(got, want, rtol):
    """Entry-wise `rtol`, plus 1e-13 of the largest entry for the near-cancelled ones."""
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    return bool(np.all(np.abs(got - want) <= rtol * np.abs(want) + 1e-13 * np.abs(want).max()))


def assert_tables_match(got, want, atol, rtol=0.0, stragglers=5, cap=5e-2):
    """Within atol + rtol*|want| everywhere except at most `stragglers` entries, and those within `cap` (a few lr)."""
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    d = np.abs(got - want)
    off = int((d > atol + rtol * np.abs(want)).sum())
    assert off <= stragglers, (off, float(d.max()))
    assert off == 0 or float(d.max()) <= cap, float(d.max())
