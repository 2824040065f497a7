"""NEXT-1 on the GPU (gc_solve_energy): the init pass builds the capacities from the energy of
PAPER.md §4 (RGB image, prior, colour GMMs -> t-links P:352-357; luma contrast -> n-links
P:342-346) and solves.  Checked against the CPU oracle: the caps it built (caps_out) equal
oracle/energy.py's, and F and mask equal Boykov-Kolmogorov's on the oracle's caps.

Both sides evaluate the costs in float64 with different exp/log implementations, so a
quantised cap may legitimately differ by 1 where the unrounded value lies within 1e-6 quanta
of a rounding boundary (reading c15); every other cap must be identical, and the
parity of F / mask is only asserted on frames whose caps are identical."""
import numpy as np
import pytest

import oracle
import synth
from certify import cut_cert
from oracle import energy

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


def oracle_caps(rgb, pr, K):
    bg, ob = synth.energy_gmms()
    out, raw = energy.caps(rgb, pr, bg, ob, K, raw=True)
    return out, raw


def compare_caps(gcaps, rgb, pr, K):
    """GPU caps [2+K,H,W] vs the oracle's; returns (oracle caps, identical?)."""
    (cs, ct, nb), (rs, rt, rn) = oracle_caps(rgb, pr, K)
    ref = np.concatenate([cs[None], ct[None], nb], axis=0)
    raw = np.concatenate([rs[None], rt[None], rn], axis=0)
    diff = gcaps != ref
    if diff.any():
        near = np.abs(raw[diff] - np.floor(raw[diff]) - 0.5) < 1e-6
        assert near.all() and np.all(np.abs(gcaps[diff].astype(np.int64) - ref[diff]) <= 1), \
            f"{int((~near).sum())} caps differ away from a rounding boundary"
        assert diff.sum() <= max(1, diff.size // 100000)
    return (cs, ct, nb), not diff.any()


def gmm_dev(torch, gc, n):
    bg, ob = synth.energy_gmms()
    return torch.from_numpy(gc.gmm_table([(bg, ob)] * n)).cuda()


@pytest.mark.parametrize("K,H,W,n", [(4, 48, 64, 3), (8, 48, 64, 2), (4, 37, 53, 2), (8, 70, 97, 2), (4, 240, 320, 4)])
def test_energy_caps_and_parity(torch, gc, K, H, W, n):
    rgb, pr = synth.gen_energy_host(synth.BASE_SEED + 3, 0, n, H, W)
    g = gc.GridCut(neighborhood=K, max_h=max(H, 64), max_w=max(W, 64))
    F, m, fs, cp = g.solve_energy(torch.from_numpy(rgb).cuda(), torch.from_numpy(pr).cuda(), gmm_dev(torch, gc, n),
                                  flow_state=True, caps=True)
    F, m, fs, cp = F.cpu().numpy(), m.cpu().numpy(), fs.cpu().numpy(), cp.cpu().numpy()
    for i in range(n):
        (cs, ct, nb), same = compare_caps(cp[i], rgb[i], pr[i], K)
        Fo, mo = oracle.solve(cs, ct, nb, "bk")
        # the solve is exact on the caps it built, whatever they are
        Fg, mg = oracle.solve(cp[i, 0], cp[i, 1], cp[i, 2:], "bk")
        assert int(F[i]) == Fg and np.array_equal(m[i], mg), i
        ok, Ff = cut_cert(cp[i, 0], cp[i, 1], cp[i, 2:], fs[i])
        assert ok and Ff == int(F[i])
        if same:
            assert int(F[i]) == Fo and np.array_equal(m[i], mo), i
    g.close()


def test_energy_equals_cap_solve_and_warm(torch, gc):
    """The energy solve equals gc_solve_batch on the caps it built, and a warm start from the
    previous frame's flows (Kohli-Torr) gives the same F and mask."""
    n, H, W, K = 4, 120, 160, 8
    rgb, pr = synth.gen_energy_host(synth.BASE_SEED + 2, 0, n + 1, H, W, seq_len=120)
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
    img, pri = torch.from_numpy(rgb).cuda(), torch.from_numpy(pr).cuda()
    gm = gmm_dev(torch, gc, n + 1)
    F, m, fs, cp = g.solve_energy(img, pri, gm, flow_state=True, caps=True)
    F2, m2 = g.solve(cp[:, 0].contiguous(), cp[:, 1].contiguous(), cp[:, 2:].contiguous())
    assert torch.equal(F, F2) and torch.equal(m, m2)
    gm1 = gm.view(n + 1, -1)[1:].contiguous().view(-1)
    Fw, mw = g.solve_energy(img[1:].contiguous(), pri[1:].contiguous(), gm1, warm_flow=fs[:n].contiguous())
    assert torch.equal(Fw, F[1:]) and torch.equal(mw, m[1:])
    g.close()


def test_energy_c4_frames(torch, gc):
    """C4 geometry (1920x1080, 8-neighbour) from energy inputs: 24 frames in one call (device
    refills); caps equal the oracle's and F / mask equal BK's on 4 frames, F == cut(mask) on
    all."""
    n, H, W, K = 24, 1080, 1920, 8
    img, pri = synth.gen_energy_torch(synth.BASE_SEED + 3, 0, n, H, W)
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
    F, m, cp = g.solve_energy(img, pri, gmm_dev(torch, gc, n), caps=True)
    torch.cuda.synchronize()
    from certify import cut_torch
    assert torch.equal(cut_torch(torch, cp[:, 0], cp[:, 1], cp[:, 2:], m), F)
    rgb, pr = img.cpu().numpy(), pri.cpu().numpy()
    for i in (0, 1, 13, 23):
        (cs, ct, nb), same = compare_caps(cp[i].cpu().numpy(), rgb[i], pr[i], K)
        assert same, i
        Fo, mo = oracle.solve(cs, ct, nb, "bk")
        assert int(F[i]) == Fo and np.array_equal(m[i].cpu().numpy(), mo), i
    g.close()


def test_energy_arg_errors(torch, gc):
    g = gc.GridCut(neighborhood=4, max_h=64, max_w=64)
    img = torch.zeros((1, 8, 8, 3), dtype=torch.uint8, device="cuda")
    pri = torch.zeros((1, 8, 8), dtype=torch.uint16, device="cuda")
    gm = gmm_dev(torch, gc, 1)
    with pytest.raises(gc.GcError) as ei:
        g.solve_energy(img, pri, gm, sigma=0.0)
    assert ei.value.status == 1
    with pytest.raises(gc.GcError):
        g.solve_energy(img, pri, gm, eps=0.7)
    g.close()
