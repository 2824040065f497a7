"""NEXT-4 on the GPU (gc_saliency): the saliency map and its prior code equal the
float32 oracle (oracle/saliency.py) bit for bit -- float32 with the same operation order on both
sides, no fused multiply-add, exact reductions."""
import numpy as np
import pytest

import synth
from oracle import saliency as S

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


@pytest.mark.parametrize("H,W,n,motion", [(64, 96, 2, False), (100, 130, 2, True), (240, 320, 3, True),
                                          (256, 256, 1, False)])
def test_saliency_bit_exact(torch, gc, H, W, n, motion):
    rng = np.random.default_rng(H + W)
    rgb, _ = synth.gen_energy_host(synth.BASE_SEED + 2, 0, n + 1, H, W, seq_len=120)
    rgb = rgb.copy()
    rgb[..., 0] = np.clip(rgb[..., 0].astype(int) + rng.integers(-30, 30, size=rgb.shape[:-1]), 0, 255)  # colour
    img, prev = rgb[1:], rgb[:-1]
    g = gc.GridCut(neighborhood=4, max_h=max(H, 64), max_w=max(W, 64))
    dimg = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    dprev = torch.from_numpy(np.ascontiguousarray(prev)).cuda() if motion else None
    sal, q = g.saliency(dimg, dprev)
    sal, q = sal.cpu().numpy(), q.cpu().numpy()
    for i in range(n):
        ref = S.saliency(img[i], prev[i] if motion else None)
        assert np.array_equal(sal[i], ref), (i, float(np.abs(sal[i] - ref).max()))
        np.testing.assert_array_equal(q[i], S.prior_code(ref, H, W))
    g.close()


def test_saliency_to_prior_update_chain(torch, gc):
    """saliency -> prior code q -> prior update -> energy solve: the full GPU front end runs and
    its q input equals the oracle's."""
    H, W = 240, 320
    rgb, _ = synth.gen_energy_host(synth.BASE_SEED + 2, 0, 2, H, W, seq_len=120)
    g = gc.GridCut(neighborhood=8, max_h=H, max_w=W)
    img = torch.from_numpy(rgb).cuda()
    sal, q = g.saliency(img[1:].contiguous(), img[:1].contiguous())
    np.testing.assert_array_equal(q[0].cpu().numpy(), S.prior_code(S.saliency(rgb[1], rgb[0]), H, W))
    bg, ob = synth.energy_gmms()
    gm = torch.from_numpy(gc.gmm_table([(bg, ob)])).cuda()
    F, m = g.solve_energy(img[1:].contiguous(), q, gm)
    assert int(F[0]) > 0
    g.close()
