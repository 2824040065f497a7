"""Synthetic input generator: shape of the inputs, and the paper-derived constants it uses."""
import math

import numpy as np
import pytest

import synth


def test_kalman_weights_first_frame():
    """Sec. 6 as printed with sigma1=0.03, sigma2=0.035, sigma_xi^2(0)=0:
    w_f = 9e-4/(9e-4+1.225e-3) = 0.423529..., w_q = 0.576470...."""
    wf, wq, v = synth.kalman_weights(1)
    assert abs(wf - 9e-4 / 2.125e-3) < 1e-12
    assert abs(wq - 1.225e-3 / 2.125e-3) < 1e-12
    assert v == 0.0


def test_kalman_fixed_point():
    """sigma_xi^2(t) -> positive root of v^2 + 1.225e-3 v - 1.1025e-6 = 0 = 6.0308885e-4
    (SURVEY.md appendix)."""
    s1, s2 = 0.03 ** 2, 0.035 ** 2
    root = (-s2 + math.sqrt(s2 * s2 + 4 * s1 * s2)) / 2
    _, _, v = synth.kalman_weights(400)
    assert abs(v - root) < 1e-12
    assert abs(root - 6.0308884908e-4) < 1e-12


@pytest.mark.parametrize("K", [4, 8])
def test_blob_caps_shape_and_range(K):
    cs, ct, nb = synth.gen_host("blob", synth.BASE_SEED + 1, 0, 2, 48, 64, K)
    off = synth.offgrid_mask(48, 64, K)
    assert cs.min() >= 0 and ct.min() >= 0 and cs.max() <= synth.CAP_MAX and ct.max() <= synth.CAP_MAX
    inn = nb[:, ~off]
    assert inn.min() >= 0 and inn.max() <= synth.CAP_MAX
    # n-links symmetric (the contrast term depends on |I_x - I_y| only)
    DY, DX = synth.DY, synth.DX
    for k in range(0, K, 2):
        for y in range(48):
            for x in range(64):
                y2, x2 = y + DY[k], x + DX[k]
                if 0 <= y2 < 48 and 0 <= x2 < 64:
                    assert nb[0, k, y, x] == nb[0, k ^ 1, y2, x2]
    # off-grid entries carry garbage (must be ignored downstream)
    assert np.any(nb[:, off] < 0) or np.any(nb[:, off] > synth.CAP_MAX)
    # a salient object exists: some pixels prefer label 1 (c(v,t) < c(s,v))
    assert (ct < cs).sum() > 20
    # frames differ over time (moving objects + noise)
    assert not np.array_equal(cs[0], cs[1])


def test_generator_deterministic():
    a = synth.gen_host("blob", 5, 2, 1, 30, 40, 4)
    b = synth.gen_host("blob", 5, 2, 1, 30, 40, 4)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_serpentine_walls():
    synth.set_serpentine_params(lane=6, big=1 << 20)
    cs, ct, nb = synth.gen_host("serpentine", 1, 0, 1, 27, 40, 4, garbage=False)
    synth.set_serpentine_params()
    # wall row 6 (between lane 0 and 1): closed except the gap at the right end
    assert np.all(nb[0, 2, 5, :40 - 6] == 0)  # S arcs from lane 0 into the wall are 0
    assert np.any(nb[0, 2, 5, 40 - 6:] > 0)
    assert cs[0, 0, :40].max() >= 1 << 20 and ct[0].max() >= 1 << 20
