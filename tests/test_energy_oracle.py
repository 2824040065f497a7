"""Pins for the energy -> capacity oracle (oracle/energy.py, NEXT-1) and for the library's
host-side GMM preparation (gc_gmm_prepare), no GPU.  Each pin is independent of the code it
checks: scipy's multivariate normal (a library density), closed forms, hand-computed values,
symmetry / monotonicity of the contrast term, and the cut-energy identity of P:358-359."""
import itertools

import numpy as np
import pytest
from scipy.special import logsumexp
from scipy.stats import multivariate_normal

import oracle
import synth
from oracle import energy

RNG = np.random.default_rng(2024)


def rand_gmm(M):
    w = RNG.random(M) + 0.1
    w = w / w.sum()
    mu = RNG.random((M, 3)) * 255
    A = RNG.normal(size=(M, 3, 3)) * 20
    S = np.einsum("mij,mkj->mik", A, A) + 30 * np.eye(3)
    return w, mu, S


def test_gmm_nll_matches_scipy_mixture():
    for M in (1, 2, 4):
        w, mu, S = rand_gmm(M)
        C = RNG.random((50, 3)) * 255
        ref = -logsumexp(np.stack([np.log(w[m]) + multivariate_normal(mu[m], S[m]).logpdf(C) for m in range(M)]), axis=0)
        np.testing.assert_allclose(energy.gmm_nll(C, w, mu, S), ref, rtol=1e-12, atol=1e-10)


def test_gmm_nll_closed_forms():
    # one component at its mean: -log N(mu; mu, S) = 1/2 log((2 pi)^3 det S)
    S = np.diag([4.0, 9.0, 16.0])
    v = energy.gmm_nll(np.array([1.0, 2.0, 3.0]), [1.0], [[1.0, 2.0, 3.0]], [S])
    assert abs(v - 0.5 * np.log((2 * np.pi) ** 3 * 576.0)) < 1e-12
    # diagonal covariance: sum of three 1-D normal NLLs
    C = np.array([4.0, -1.0, 7.0])
    ref = sum(0.5 * np.log(2 * np.pi * s2) + (c - m) ** 2 / (2 * s2) for c, m, s2 in zip(C, [1, 2, 3], [4, 9, 16]))
    assert abs(energy.gmm_nll(C, [1.0], [[1.0, 2.0, 3.0]], [S]) - ref) < 1e-12
    # two identical components with weights a, 1-a are one component
    assert abs(energy.gmm_nll(C, [0.3, 0.7], [[1, 2, 3], [1, 2, 3]], [S, S]) - ref) < 1e-12


def test_nlink_term_hand_values_and_shape():
    # dI = 0: lambda / dist + kappa
    assert abs(energy.nlink_value(0, 1.0, 10.0, 0.1, 0.05) - 10.05) < 1e-15
    assert abs(energy.nlink_value(0, np.sqrt(2.0), 10.0, 0.1, 0.05) - (10.0 / np.sqrt(2.0) + 0.05)) < 1e-15
    # dI = 25.5 (x = 0.1 = sigma): lambda e^{-1/2} + kappa
    assert abs(energy.nlink_value(25.5, 1.0, 10.0, 0.1, 0.05) - (10 * np.exp(-0.5) + 0.05)) < 1e-12
    v = energy.nlink_value(np.arange(256), 1.0, 10.0, 0.1, 0.05)
    # non-increasing towards kappa (strictly while the Gaussian term is resolvable in float64)
    assert np.all(np.diff(v) <= 0) and np.all(np.diff(v[:120]) < 0) and v[-1] >= 0.05


def test_quantize_rounding_and_clamp():
    np.testing.assert_array_equal(energy.quantize([0.0, 1 / 128 - 1e-9, 1 / 128, -5.0, 1e9], 64.0),
                                  [0, 0, 1, 0, (1 << 26) - 1])


def test_luma_integer_bt601():
    assert energy.luma(np.array([255, 255, 255], np.uint8)) == 255
    assert energy.luma(np.array([0, 0, 0], np.uint8)) == 0
    assert energy.luma(np.array([100, 50, 200], np.uint8)) == (77 * 100 + 150 * 50 + 29 * 200 + 128) >> 8


@pytest.mark.parametrize("K", [4, 8])
def test_caps_structure(K):
    """n-links symmetric (c_k(p) = c_opp(k)(p + d_k)), off-grid 0, t-links = the two label costs."""
    rgb, pr = synth.gen_energy_host(synth.BASE_SEED + 3, 5, 1, 37, 41)
    bg, ob = synth.energy_gmms()
    cs, ct, nb = energy.caps(rgb[0], pr[0], bg, ob, K)
    H, W = 37, 41
    for k in range(K):
        dy, dx = energy.DY[k], energy.DX[k]
        for y, x in itertools.product(range(H), range(W)):
            y2, x2 = y + dy, x + dx
            if 0 <= y2 < H and 0 <= x2 < W:
                assert nb[k, y, x] == nb[k ^ 1, y2, x2]
            else:
                assert nb[k, y, x] == 0
    p = np.clip(pr[0] / 65535.0, 1e-6, 1 - 1e-6)
    u0 = energy.gmm_nll(rgb[0].astype(float), *bg) - np.log(1 - p)
    np.testing.assert_array_equal(cs, np.floor(64 * u0 + 0.5).astype(np.int32))


def test_cut_of_energy_caps_is_the_energy():
    """with these caps, cut(S) is the quantised MRF energy of the labelling S (t-link
    of every pixel's label + contrast term of every label boundary, counted per directed arc
    leaving S as the graph of P:331-346 does); brute force on a 3x3 crop equals the minimum."""
    rgb, pr = synth.gen_energy_host(synth.BASE_SEED + 3, 0, 1, 3, 3)
    bg, ob = synth.energy_gmms()
    cs, ct, nb = energy.caps(rgb[0], pr[0], bg, ob, 4)
    best = None
    for bits in range(1 << 9):
        S = np.array([(bits >> i) & 1 for i in range(9)], np.uint8).reshape(3, 3)
        e = int(np.where(S == 1, ct, cs).sum())
        for k in range(4):
            for y, x in itertools.product(range(3), range(3)):
                y2, x2 = y + energy.DY[k], x + energy.DX[k]
                if 0 <= y2 < 3 and 0 <= x2 < 3 and S[y, x] == 1 and S[y2, x2] == 0:
                    e += int(nb[k, y, x])
        assert e == oracle.cut_value(cs, ct, nb, S)
        best = e if best is None else min(best, e)
    F, _ = oracle.brute(cs, ct, nb)
    assert F == best


def test_gmm_prepare_matches_definition():
    """The library's host helper: lognorm = log w - 1/2 log((2 pi)^3 det S), prec = S^-1."""
    gc = pytest.importorskip("paper_1008_0502_b200")
    for M in (1, 3):
        w, mu, S = rand_gmm(M)
        g = gc.gc_gmm_prepare(w, mu, S)
        assert g.M == M
        for m in range(M):
            assert abs(g.lognorm[m] - (np.log(w[m]) - 0.5 * np.log((2 * np.pi) ** 3 * np.linalg.det(S[m])))) < 1e-9
            P = np.linalg.inv(S[m])
            got = [g.prec[m][i] for i in range(6)]
            np.testing.assert_allclose(got, [P[0, 0], P[0, 1], P[0, 2], P[1, 1], P[1, 2], P[2, 2]], rtol=1e-10)
            np.testing.assert_allclose([g.mean[m][i] for i in range(3)], mu[m])
    with pytest.raises(gc.GcError):
        gc.gc_gmm_prepare([1.0], [[0, 0, 0]], [-np.eye(3)])
