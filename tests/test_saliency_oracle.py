"""Pins for the saliency oracle (oracle/saliency.py, NEXT-4), no GPU: SPEC's worked examples for
the normalisation N(.) (constant -> 0, an isolated peak kept, two equal peaks
suppressed), the trivial channel identities (grey frame -> no colour opponents, a
repeated frame -> no motion, a pure red pixel), closed forms of the pyramid, the up-sampling and
the centre-surround maps on constant inputs, the filter-bank symmetry, and SPEC's "white square
on black" example (the saliency argmax lies in the square, dilated)."""
import numpy as np

import paper_1008_0502_b200 as gc
from oracle import saliency as S


def test_normalize_spec_examples():
    assert not S.normalize(np.full((20, 30), 0.7, np.float32)).any()              # constant -> 0
    v = np.zeros((40, 40), np.float32)
    v[20, 20] = 5.0
    out = S.normalize(v)
    assert out[20, 20] == 1.0 and out.sum() == 1.0                                # single peak kept
    v[5, 5] = 5.0
    assert not S.normalize(v).any()                                               # two equal peaks: (1-1)^2 = 0
    v[5, 5] = 2.5
    out = S.normalize(v)
    assert abs(out[20, 20] - 0.25) < 1e-7                                         # mbar = 0.5 -> factor 0.25


def test_features_identities():
    grey = np.full((8, 8, 3), 120, np.uint8)
    I, RG, BY, M = S.features(grey)
    assert not RG.any() and not BY.any() and not M.any()
    assert not S.features(grey, grey)[3].any()
    red = np.zeros((1, 1, 3), np.uint8)
    red[..., 0] = 255
    I, RG, BY, _ = S.features(red)
    assert abs(I[0, 0] - 1 / 3) < 1e-7 and abs(RG[0, 0] - 3.0) < 1e-6        # (r - g) / I with I = 1/3
    dark = np.full((2, 2, 3), 20, np.uint8)
    assert not S.features(dark)[1].any()                                         # I < 0.1 -> opponents 0


def test_pyramid_and_upsampling_constant():
    c = np.full((37, 51), 0.375, np.float32)
    pyr = S.pyramid(c)
    assert [p.shape for p in pyr][:3] == [(37, 51), (19, 26), (10, 13)] and pyr[-1].shape == (1, 1)
    assert all(np.all(p == np.float32(0.375)) for p in pyr)                      # weights sum to 1 exactly
    assert np.all(S.bilinear(pyr[4], 10, 13) == np.float32(0.375))
    assert not np.abs(pyr[2] - S.bilinear(pyr[5], *pyr[2].shape)).any()           # centre-surround of a constant


def test_gabor_bank_symmetry_and_library_match():
    k = S.gabor_kernels()
    assert np.abs(k.sum(axis=(1, 2))).max() < 1e-6                               # zero mean
    np.testing.assert_allclose(k[2], k[0].T, atol=1e-7)                           # 90 degrees = transpose of 0
    np.testing.assert_allclose(k[3], k[1][:, ::-1], atol=1e-7)                    # 135 = mirror of 45
    assert np.array_equal(gc.gc_gabor_kernels(), k)                               # the library's host table


def test_square_on_black():
    img = np.zeros((256, 256, 3), np.uint8)
    img[40:72, 40:72] = 255
    sal = S.saliency(img)
    h4, w4 = sal.shape
    assert (h4, w4) == gc.gc_saliency_dims(256, 256) == (16, 16) and sal.max() == 1.0
    y, x = np.unravel_index(np.argmax(sal), sal.shape)
    # the square covers level-4 rows / cols 2.5..4.5; the argmax lies in that box dilated by 3
    assert 0 <= y <= 7 and 0 <= x <= 7
    assert sal[12:, 12:].max() < sal.max()
    assert not S.saliency(np.full((64, 64, 3), 99, np.uint8)).any()              # uniform grey -> 0
