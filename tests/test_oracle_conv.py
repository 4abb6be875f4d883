"""Pins for the oracle's direct convolution (O7) and error metrics: closed forms,
special cases, brute force and a library routine (torch conv2d in
fp64, i.e. the DNN definition of a 3x3 stride-1 correlation layer)."""
import random
from fractions import Fraction as Fr

import numpy as np
import pytest
import torch

from oracle import conv as CV
from oracle import metrics as MT


def test_direct_vs_library_fp64():
    rng = np.random.default_rng(0)
    for (N, C, K, H, W, pad) in [(2, 3, 4, 9, 7, 1), (1, 5, 2, 6, 6, 0), (3, 8, 8, 16, 16, 1)]:
        x = rng.standard_normal((N, C, H, W))
        w = rng.standard_normal((K, C, 3, 3))
        y = CV.direct_conv2d_f64(x, w, pad)
        ref = torch.nn.functional.conv2d(torch.from_numpy(x), torch.from_numpy(w), padding=pad).numpy()
        np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)


def test_direct_vs_bruteforce_exact():
    rng = random.Random(1)
    rq = lambda: Fr(rng.randint(-9, 9), rng.randint(1, 4))
    x = [[[[rq() for _ in range(5)] for _ in range(4)] for _ in range(2)]]
    w = [[[[rq() for _ in range(3)] for _ in range(3)] for _ in range(2)] for _ in range(3)]
    ex = CV.direct_conv2d_exact(x, w, 1)
    y = CV.direct_conv2d_f64(np.array(x, dtype=float), np.array(w, dtype=float), 1)
    np.testing.assert_allclose(y, np.array(ex, dtype=float), rtol=1e-13, atol=1e-13)


def test_special_cases():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((1, 1, 6, 6))
    imp = np.zeros((1, 1, 3, 3))
    imp[0, 0, 0, 0] = 1                                   # S:296 impulse at (0,0): y_ij = x_ij
    assert np.array_equal(CV.direct_conv2d_f64(x, imp, 0), x[:, :, :4, :4])
    ones_x, ones_w = np.ones((1, 4, 5, 5)), np.ones((2, 4, 3, 3))
    y = CV.direct_conv2d_f64(ones_x, ones_w, 1)
    assert np.all(y[:, :, 1:-1, 1:-1] == 36.0)            # 9 C in the interior
    assert y[0, 0, 0, 0] == 16.0                          # corner: 4 taps x C
    assert not CV.direct_conv2d_f64(np.zeros((1, 2, 4, 4)), rng.standard_normal((1, 2, 3, 3)), 1).any()
    # separable kernel = 1D correlation along rows then columns
    h1, h2 = rng.standard_normal(3), rng.standard_normal(3)
    w = np.outer(h1, h2)[None, None]
    y = CV.direct_conv2d_f64(x, w, 0)[0, 0]
    rows = np.array([np.correlate(r, h2, "valid") for r in x[0, 0]])
    sep = np.array([np.correlate(c, h1, "valid") for c in rows.T]).T
    np.testing.assert_allclose(y, sep, rtol=1e-12, atol=1e-12)
    assert CV.direct_corr_1d([1, 1, 1], [1, 2, 3, 4]) == [6, 9]
    assert CV.direct_corr_1d([1, -2, 3], [4, 5, 6, 7]) == [12, 14]        # hand evaluation


def test_metrics_closed_forms():
    yref = np.zeros((1, 1, 2, 2))
    y = np.zeros((1, 1, 2, 2))
    y[0, 0, 0, 0], y[0, 0, 0, 1] = 3.0, 4.0               # S:393 3-4-5
    s = MT.stats8(y, yref, 2)
    assert s[0] == 7.0 and s[3] == 5.0 and s[6] == 1 and s[7] == 4
    assert s[4] == np.inf                                  # nonzero error on a zero reference
    yref = np.ones((1, 1, 3, 3))
    y = yref.copy()
    y[0, 0, 2, 2] = np.inf
    s = MT.stats8(y, yref, 2)                              # 2x2 tiles over 3x3, clipped
    assert s[5] == 1 and s[6] == 4 and s[7] == 9 and s[0] == np.inf
    s = MT.stats8(yref, yref, 2)
    assert s[0] == 0 and s[2] == 0 and s[1] == 9
    y = yref * 1.01
    sm = MT.summary(MT.stats8(y, yref, 3))
    assert sm["rel_l1"] == pytest.approx(0.01) and sm["mean_rel"] == pytest.approx(0.01)
