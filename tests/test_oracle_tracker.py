"""Pins for the tracker-loop oracle (O17-O18) -- CPU only:
hand-worked parent masks and closed-form weighted means."""
import math

import numpy as np
import pytest


def test_next_parents_hand_example(orc):
    # two kept hypotheses over T = 4 old tracks; pairs 0..5; births at columns 6, 7
    pair_of = np.array([[0, -1, 2, 5], [1, 3, -1, -1]], np.int32)
    mask, lw = orc.next_parents([0.75, 0.25], pair_of, 4, 6, 2, 6, 1)
    assert mask[0, 0] == (1 << 0) | (1 << 2) | (1 << 5) | (1 << 6) | (1 << 7)
    assert mask[1, 0] == (1 << 1) | (1 << 3) | (1 << 6) | (1 << 7)
    np.testing.assert_allclose(lw, [math.log(0.75), math.log(0.25)], rtol=1e-15)
    # pairs past the capacity are dropped (not in the new set); births across a word boundary
    mask, lw = orc.next_parents([1.0], np.array([[31, 40]], np.int32), 2, 35, 3, 35, 2)
    assert mask[0, 0] == 1 << 31 and mask[0, 1] == (1 << 3) | (1 << 4) | (1 << 5)
    assert lw[0] == 0.0
    mask, lw = orc.next_parents([], np.zeros((0, 3), np.int32), 3, 4, 1, 4, 1)
    assert mask.shape == (0, 1)


def test_map_estimate_closed_forms(orc):
    x = np.array([[0.0, 1.0, 2.0, 3.0], [10.0, 10.0, 10.0, 10.0]], np.float32)
    y = np.array([[4.0, 4.0, 0.0, 0.0], [-1.0, 1.0, -1.0, 1.0]], np.float32)
    w = np.array([[0.5, 0.25, 0.25, 0.0], [1.0, 1.0, 1.0, 1.0]], np.float32)
    est = orc.map_estimate(1, np.array([1, -1, 0], np.int32), x, y, w)
    np.testing.assert_allclose(est[0], [10.0, 0.0, 1.0])                  # uniform: arithmetic mean
    assert np.isnan(est[1, 0]) and est[1, 2] == 0.0
    np.testing.assert_allclose(est[2], [0.75, 3.0, 1.0], rtol=1e-15)     # 0.25 + 0.5; 2 + 1
    # scale invariance of the weights and permutation invariance of the particles
    est2 = orc.map_estimate(1, np.array([0], np.int32), x[:1, ::-1], y[:1, ::-1], 1e-20 * w[:1, ::-1])
    np.testing.assert_allclose(est2[0], est[2], rtol=1e-12)
    # no kept hypothesis: nothing estimated
    assert np.all(orc.map_estimate(0, np.array([0, 1], np.int32), x, y, w)[:, 2] == 0)
