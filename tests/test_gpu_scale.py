"""Parity at config scale (SURVEY.md §8(d) "every frame must match", north_star "bit-exact
... on every config"): whole BASELINE.json configs solved in the launch configuration the
bench uses -- one call, slots refilled on the device as frames finish -- and compared frame
by frame with the CPU oracle (Boykov-Kolmogorov, bit-exact F and mask), or, for the 4K
adversarial frames the oracle cannot finish, certified oracle-free (flow certificate +
host recomputation of the canonical cut).  Caps come from the CUDA twin of synth/ (tested
bit-identical to the host twin) and are copied to the host for the oracle."""
import os

import numpy as np
import pytest

import oracle
import synth
from certify import cut_cert, cut_torch, residual_closure_host

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def torch():
    import torch as _t
    assert _t.cuda.is_available(), "GPU tests need a CUDA device"
    return _t


@pytest.fixture(scope="module")
def gc():
    import paper_1008_0502_b200 as _gc
    return _gc


def oracle_compare(cs, ct, nb, F, mask, first=0, label=""):
    """Every frame of the device batch against BK on all host cores, in chunks; returns the
    number of frames checked.  Raises on the first mismatch with the frame index."""
    n = cs.shape[0]
    threads = len(os.sched_getaffinity(0))
    chunk = max(2 * threads, 8)
    Fh, mh = F.cpu().numpy(), mask.cpu().numpy()
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        Fo, mo = oracle.solve_batch(cs[a:b].cpu().numpy(), ct[a:b].cpu().numpy(), nb[a:b].cpu().numpy(), "bk",
                                    threads=threads)
        for i in range(b - a):
            f = a + i
            assert int(Fh[f]) == int(Fo[i]), f"{label} frame {first + f}: F gpu {int(Fh[f])} oracle {int(Fo[i])}"
            if not np.array_equal(mh[f], mo[i]):
                raise AssertionError(f"{label} frame {first + f}: {int((mh[f] != mo[i]).sum())} mask bytes differ")
    return n


def test_c4_bench_batch_every_frame_vs_oracle(torch, gc):
    """C4 exactly as bench.py runs it: 1024 frames of 1920x1080 8-neighbour caps in ONE
    gc_solve_batch call on a default context (24 slots; frames 24..1023 run in slots the
    device refilled after earlier frames, reusing their per-tile state).  Every frame's F and
    mask equal the oracle's; the device digest (gc_frame_digest) equals the digest of the
    oracle masks."""
    n = 1024
    cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 3, 0, n, 1080, 1920, 8)
    g = gc.GridCut(neighborhood=8, max_h=1080, max_w=1920)
    F, mask, st = g.solve(cs, ct, nb, stats=True)
    torch.cuda.synchronize()
    assert (st[:, 3] == 0).all()
    dg = g.digest(F, mask).cpu().numpy()
    checked = oracle_compare(cs, ct, nb, F, mask, label="C4")
    mh = mask.cpu().numpy()
    for f in range(0, n, 97):
        assert (int(dg[f, 1]), int(dg[f, 2])) == oracle.mask_digest(mh[f]), f
    print(f"C4: {checked} frames bit-exact vs BK (frames 0..{n - 1}; >= 1000 in device-refilled slots); "
          f"push tasks max {int(st[:, 0].max())}, relabels max {int(st[:, 1].max())}")
    g.close()
    del cs, ct, nb


def test_c2_all_300_frames_vs_oracle(torch, gc):
    """C2: the whole 300-frame QVGA clip in one call, every frame vs the oracle."""
    n = 300
    cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 1, 0, n, 240, 320, 4)
    g = gc.GridCut(neighborhood=4, max_h=240, max_w=320)
    F, mask = g.solve(cs, ct, nb)
    torch.cuda.synchronize()
    print(f"C2: {oracle_compare(cs, ct, nb, F, mask, label='C2')} frames bit-exact vs BK")
    g.close()


def test_c3_warm_sequences_every_frame(torch, gc):
    """C3 in the bench's warm schedule: 8 sequences x 120 VGA frames; the batch of time t is
    the 8 frames of that time step, warm-started from the flows the batch at t-1 exported.
    warm == cold == oracle on all 960 frames (F and mask)."""
    S, L, H, W = 8, 120, 480, 640
    cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 2, 0, S * L, H, W, 4, seq_len=L)
    order = torch.arange(S * L, device=cs.device).view(S, L).t().reshape(-1)  # [time][sequence]
    cs, ct, nb = cs[order].contiguous(), ct[order].contiguous(), nb[order].contiguous()
    g = gc.GridCut(neighborhood=4, max_h=H, max_w=W)
    Fw, mw, Fc, mc = [], [], [], []
    prev = None
    for t in range(L):
        sl = slice(t * S, (t + 1) * S)
        F1, m1, f1 = g.solve(cs[sl], ct[sl], nb[sl], warm_flow=prev, flow_state=True)
        prev = f1
        Fw.append(F1); mw.append(m1)
        F2, m2 = g.solve(cs[sl], ct[sl], nb[sl])
        Fc.append(F2); mc.append(m2)
    Fw, mw, Fc, mc = torch.cat(Fw), torch.cat(mw), torch.cat(Fc), torch.cat(mc)
    assert torch.equal(Fw, Fc) and torch.equal(mw, mc)
    print(f"C3: warm == cold on {S * L} frames; {oracle_compare(cs, ct, nb, Fw, mw, label='C3')} frames bit-exact vs BK")
    g.close()


def test_c3_sequence_pass_every_frame(torch, gc):
    """C3 through gc_solve_sequences, the bench's warm schedule: 8 sequences x 120 VGA frames in
    ONE device pass, frame t of a sequence warm-started from the flows frame t-1 exported.
    warm == cold (the same pass with warm=0) == oracle on all 960 frames."""
    S, L, H, W = 8, 120, 480, 640
    cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 2, 0, S * L, H, W, 4, seq_len=L)
    g = gc.GridCut(neighborhood=4, max_h=H, max_w=W)
    sh = lambda a: a.view((S, L) + tuple(a.shape[1:]))  # noqa: E731
    Fw, mw = g.solve_sequences(sh(cs), sh(ct), sh(nb), warm=True)
    Fc, mc = g.solve_sequences(sh(cs), sh(ct), sh(nb), warm=False)
    assert torch.equal(Fw, Fc) and torch.equal(mw, mc)
    n = oracle_compare(cs, ct, nb, Fw.reshape(-1), mw.reshape(S * L, H, W), label="C3 seq")
    print(f"C3 sequences: warm == cold == BK on {n} frames")
    g.close()


def test_c5_all_frames_certified(torch, gc):
    """C5 as bench.py --config c5 runs it: 8 frames of 3840x2160 serpentine caps (64-px lanes)
    in one call.  The oracle needs hours per frame, so every frame is certified without it
    (SURVEY.md §8(c)): the exported flow is arc-feasible and F(f) == F == cut(mask) (F is the
    maximum flow value, the mask a minimum cut), and the mask equals the residual closure of
    the excess nodes recomputed on the host with scipy's BFS (the canonical cut)."""
    n, H, W = 8, 2160, 3840
    synth.set_serpentine_params(lane=64, big=1 << 20)
    try:
        cs, ct, nb = synth.gen_torch("serpentine", synth.BASE_SEED + 4, 0, n, H, W, 4)
    finally:
        synth.set_serpentine_params()
    g = gc.GridCut(neighborhood=4, max_h=H, max_w=W)
    F, mask, fs = g.solve(cs, ct, nb, flow_state=True)
    torch.cuda.synchronize()
    cut = cut_torch(torch, cs, ct, nb, mask).cpu().numpy()
    for i in range(n):
        hc, ht, hn = cs[i].cpu().numpy(), ct[i].cpu().numpy(), nb[i].cpu().numpy()
        f = fs[i].cpu().numpy()
        Fg = int(F[i])
        assert int(cut[i]) == Fg, i
        ok, Ff = cut_cert(hc, ht, hn, f)
        assert ok and Ff == Fg, i
        np.testing.assert_array_equal(mask[i].cpu().numpy(), residual_closure_host(hc, ht, hn, f))
    print(f"C5: {n} 4K frames certified (flow certificate + canonical closure)")
    g.close()
