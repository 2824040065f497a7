"""NEXT-2 on the GPU (gc_prior_update, §6): the smoothed previous mask fused with the
saliency prior by the Kalman-style weights, bit-exact against oracle/prior.py (exact integer
arithmetic on both sides), and the closed temporal loop mask(t-1) -> prior(t) -> energy solve
(NEXT-1) -> mask(t) against the oracle's loop."""
import numpy as np
import pytest

import oracle
import synth
from oracle import energy, prior

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    assert _t.cuda.is_available(), "GPU tests need a CUDA device"
    return _t


@pytest.fixture(scope="module")
def gc():
    import paper_1008_0502_b200 as _gc
    return _gc


@pytest.mark.parametrize("H,W,n,sigma,radius,band", [(48, 64, 3, 2.0, 6, 8), (37, 53, 2, 1.0, 0, 0),
                                                     (70, 130, 2, 5.0, 16, 3), (1, 1, 1, 1.0, 2, 0),
                                                     (240, 320, 4, 3.0, 9, 8), (1080, 1920, 1, 4.0, 12, 8)])
def test_prior_update_bit_exact(torch, gc, H, W, n, sigma, radius, band):
    rng = np.random.default_rng(H * 7 + W)
    mask = (rng.random((n, H, W)) < 0.3).astype(np.uint8)
    mask[:, H // 4:H // 2, W // 4:W // 2] = 1  # a blob
    q = rng.integers(0, 65536, size=(n, H, W)).astype(np.uint16)
    wf = rng.integers(0, 4097, size=n).astype(np.int32)
    g = gc.GridCut(neighborhood=4, max_h=max(H, 64), max_w=max(W, 64))
    params = gc.prior_params(sigma, radius, band)
    out = g.prior_update(torch.from_numpy(mask).cuda(), torch.from_numpy(q).cuda(), torch.from_numpy(wf).cuda(),
                         params).cpu().numpy()
    taps = prior.gauss_taps(sigma, radius)
    for i in range(n):
        np.testing.assert_array_equal(out[i], prior.prior_update(mask[i], q[i], int(wf[i]), taps, band))
    g.close()


def test_closed_loop_mask_prior_solve(torch, gc):
    """4 time steps of one sequence, QVGA, 8-neighbour: prior(t) = update(mask(t-1), q(t)) on the
    device, then gc_solve_energy with it; the oracle runs the same loop (oracle/prior.py,
    oracle/energy.py, Boykov-Kolmogorov).  Masks, F and priors agree at every step."""
    H, W, K, L = 240, 320, 8, 4
    rgb, q = synth.gen_energy_host(synth.BASE_SEED + 2, 0, L, H, W, seq_len=L)
    bg, ob = synth.energy_gmms()
    gm = torch.from_numpy(gc.gmm_table([(bg, ob)])).cuda()
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
    params = gc.prior_params(3.0, 9, 8)
    taps = prior.gauss_taps(3.0, 9)
    s1, s2, v = 0.03 ** 2, 0.035 ** 2, 0.0
    mask_g = None
    mask_o = None
    for t in range(L):
        if t == 0:
            pr_g = torch.from_numpy(q[0:1]).cuda()
            pr_o = q[0]
        else:
            wf, v_next = gc.gc_kalman_step(s1, s2, v)
            w_ref, v_ref = prior.kalman_step(s1, s2, v)
            assert wf == prior.wf_q12(w_ref) and v_next == v_ref
            v = v_next
            pr_g = g.prior_update(mask_g, torch.from_numpy(q[t:t + 1]).cuda(),
                                  torch.tensor([wf], dtype=torch.int32, device="cuda"), params)
            pr_o = prior.prior_update(mask_o, q[t], wf, taps, 8)
            np.testing.assert_array_equal(pr_g[0].cpu().numpy(), pr_o)
        F, mask_g = g.solve_energy(torch.from_numpy(rgb[t:t + 1]).cuda(), pr_g.contiguous(), gm)
        cs, ct, nb = energy.caps(rgb[t], pr_o, bg, ob, K)
        Fo, mask_o = oracle.solve(cs, ct, nb, "bk")
        assert int(F[0]) == Fo, t
        np.testing.assert_array_equal(mask_g[0].cpu().numpy(), mask_o)
    g.close()
