"""Pins for the prior-update oracle (oracle/prior.py, NEXT-2) and the library's host helpers
gc_gauss_taps / gc_kalman_step, no GPU: impulse response of the smoothing = the outer product
of the taps, constant masks in closed form, the recursion's steady state in closed form and the
weights SURVEY.md §8(c) reading c10 prints (P:428-436 with sigma_1 = 0.03, sigma_2 = 0.035 of
P:648)."""
import math

import numpy as np
import pytest

from oracle import prior


def test_impulse_response_is_outer_product_of_taps():
    taps = prior.gauss_taps(2.0, 5)
    m = np.zeros((21, 23), np.uint8)
    m[10, 11] = 1
    S = prior.smooth_sum(m, taps)
    g = np.array(taps[::-1] + taps[1:], np.int64)  # g_{-5..5}
    ref = np.zeros_like(S)
    ref[5:16, 6:17] = np.outer(g, g)
    np.testing.assert_array_equal(S, ref)


def test_constant_masks_closed_form():
    taps = prior.gauss_taps(1.5, 4)
    G = taps[0] + 2 * sum(taps[1:])
    q = np.full((9, 12), 40000, np.uint16)
    ones = prior.prior_update(np.ones((9, 12), np.uint8), q, 1000, taps, 0)
    zeros = prior.prior_update(np.zeros((9, 12), np.uint8), q, 1000, taps, 0)
    # f = 1: p = w + (1 - w) q / 65535; f = 0: p = (1 - w) q / 65535 (w = 1000/4096)
    assert np.all(ones == (1000 * G * G * 65535 + 3096 * 40000 * G * G + 2048 * G * G) // (4096 * G * G))
    assert np.all(zeros == (3096 * 40000 + 2048) // 4096)
    assert abs(int(ones[0, 0]) - round(65535 * (1000 / 4096 + (3096 / 4096) * 40000 / 65535))) <= 1


def test_edge_band_is_zero():
    taps = prior.gauss_taps(1.0, 2)
    out = prior.prior_update(np.ones((10, 10), np.uint8), np.full((10, 10), 65535, np.uint16), 2048, taps, 3)
    assert out[:3].max() == 0 and out[:, :3].max() == 0 and out[-3:].max() == 0 and out[:, -3:].max() == 0
    assert out[3:7, 3:7].min() == 65535


def test_kalman_recursion_as_printed():
    s1, s2 = 0.03 ** 2, 0.035 ** 2
    w1, v1 = prior.kalman_step(s1, s2, 0.0)
    assert abs(w1 - 0.423529) < 1e-6  # w_f(1) = 0.423529
    v = 0.0
    for _ in range(200):
        w, v = prior.kalman_step(s1, s2, v)
    vstar = (-s2 + math.sqrt(s2 * s2 + 4 * s1 * s2)) / 2  # steady state of v = s1 (s2 + v)/(s1 + s2 + v)
    assert abs(v - vstar) < 1e-15 and abs(v - 6.0308884908e-4) < 1e-12
    assert abs(prior.kalman_step(s1, s2, v)[0] - 0.329901) < 1e-6  # steady-state w_f


def test_library_host_helpers_match():
    gc = pytest.importorskip("paper_1008_0502_b200")
    for sigma, r in [(0.5, 0), (1.0, 3), (4.0, 16)]:
        assert gc.gc_gauss_taps(sigma, r) == prior.gauss_taps(sigma, r)
    v = 0.0
    for _ in range(5):
        wf, vn = gc.gc_kalman_step(0.03 ** 2, 0.035 ** 2, v)
        w_ref, v_ref = prior.kalman_step(0.03 ** 2, 0.035 ** 2, v)
        assert wf == prior.wf_q12(w_ref) and vn == v_ref
        v = vn
    with pytest.raises(gc.GcError):
        gc.gc_gauss_taps(0.0, 3)
    with pytest.raises(gc.GcError):
        gc.gc_gauss_taps(1.0, 17)
