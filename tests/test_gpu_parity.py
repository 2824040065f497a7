"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit-exact in both
the flow value (int64) and the canonical mask (uint8) -- SURVEY.md §8(c)."""
import numpy as np
import pytest

import oracle
import synth
from certify import check_against_oracle, cut_cert, cut_torch, residual_closure_host

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


_SOLVERS = {}


def solver(gc, K, max_h=1080, max_w=1920, **kw):
    key = (K, max_h, max_w, tuple(sorted(kw.items())))
    if key not in _SOLVERS:
        _SOLVERS[key] = gc.GridCut(neighborhood=K, max_h=max_h, max_w=max_w, **kw)
    return _SOLVERS[key]


def to_dev(torch, *arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrs]


# ----------------------------------------------------------------------------- generator twin
@pytest.mark.parametrize("kind,H,W,K", [("blob", 48, 64, 4), ("blob", 240, 320, 8), ("serpentine", 100, 130, 4),
                                        ("random", 33, 47, 8)])
def test_generator_twins_bit_identical(torch, kind, H, W, K):
    a = synth.gen_host(kind, 99, 4, 3, H, W, K)
    b = synth.gen_torch(kind, 99, 4, 3, H, W, K)
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y.cpu().numpy())


# ----------------------------------------------------------------------------- small random
SIZES = [(1, 1), (1, 7), (5, 1), (2, 2), (3, 5), (8, 8), (13, 31), (31, 33), (32, 32), (33, 32), (32, 65),
         (47, 29), (64, 64), (70, 97)]


@pytest.mark.parametrize("K", [4, 8])
def test_random_grids_parity(torch, gc, K):
    rng = np.random.default_rng(500 + K)
    g = solver(gc, K, 128, 128)
    for (H, W) in SIZES:
        for tmax, nmax in [(3, 3), (20, 20), (1000, 50), (50, 1000)]:
            cs, ct, nb = synth.random_caps(rng, H, W, K, tmax=tmax, nmax=nmax, zero_frac=0.3, garbage=True, n=3)
            F, mask = g.solve(*to_dev(torch, cs, ct, nb))
            check_against_oracle(cs, ct, nb, F.cpu().numpy(), mask.cpu().numpy())


@pytest.mark.parametrize("K", [4, 8])
def test_extreme_caps(torch, gc, K):
    """CAP_MAX-edge capacities (int32 headroom of e and r) and all-zero frames."""
    rng = np.random.default_rng(77)
    g = solver(gc, K, 128, 128)
    H, W = 40, 50
    cs = rng.choice([0, gc.CAP_MAX, gc.CAP_MAX - 1, 1], size=(2, H, W)).astype(np.int32)
    ct = rng.choice([0, gc.CAP_MAX, 2], size=(2, H, W)).astype(np.int32)
    nb = rng.choice([0, gc.CAP_MAX, 5], size=(2, K, H, W)).astype(np.int32)
    cs[1] = 0; ct[1] = 0; nb[1] = 0
    F, mask = g.solve(*to_dev(torch, cs, ct, nb))
    check_against_oracle(cs, ct, nb, F.cpu().numpy(), mask.cpu().numpy())


# ----------------------------------------------------------------------------- configs
@pytest.mark.parametrize("K", [4, 8])
def test_c1_blob_64x48(torch, gc, K):
    cs, ct, nb = synth.gen_host("blob", synth.BASE_SEED + 0, 0, 1, 48, 64, K)
    g = solver(gc, K)
    F, mask, fs = g.solve(*to_dev(torch, cs, ct, nb), flow_state=True)
    F, mask, fs = F.cpu().numpy(), mask.cpu().numpy(), fs.cpu().numpy()
    check_against_oracle(cs, ct, nb, F, mask, "dinic")
    check_against_oracle(cs, ct, nb, F, mask, "bk")
    ok, Ff = cut_cert(cs[0], ct[0], nb[0], fs[0])
    assert ok and Ff == int(F[0]) == oracle.cut_value(cs[0], ct[0], nb[0], mask[0])


def test_c2_qvga_clip_sample(torch, gc):
    """C2 shape: 320x240 4-nbr blob frames, independent cold solves (40 of the 300)."""
    n = 40
    cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 1, 0, n, 240, 320, 4)
    g = solver(gc, 4)
    F, mask, st = g.solve(cs, ct, nb, stats=True)
    torch.cuda.synchronize()
    hc, ht, hn = synth.gen_host("blob", synth.BASE_SEED + 1, 0, n, 240, 320, 4)
    Fo, mo = oracle.solve_batch(hc, ht, hn, "bk")
    np.testing.assert_array_equal(F.cpu().numpy(), Fo)
    np.testing.assert_array_equal(mask.cpu().numpy(), mo)
    assert np.all(st.cpu().numpy()[:, 3] == 0)


def test_c3_vga_warm_start(torch, gc):
    """C3: 640x480 sequence; frame t>=1 warm-started from t-1's exported flows.
    warm == cold == oracle on every frame."""
    n = 6
    cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 2, 0, n, 480, 640, 4, seq_len=120)
    g = solver(gc, 4)
    Fc, mc, fc = g.solve(cs, ct, nb, flow_state=True)
    prev = fc[0:1]
    Fw, mw = [Fc[0:1]], [mc[0:1]]
    for t in range(1, n):
        F1, m1, f1 = g.solve(cs[t:t + 1], ct[t:t + 1], nb[t:t + 1], warm_flow=prev.contiguous(), flow_state=True)
        Fw.append(F1); mw.append(m1); prev = f1
    Fw, mw = torch.cat(Fw), torch.cat(mw)
    np.testing.assert_array_equal(Fw.cpu().numpy(), Fc.cpu().numpy())
    np.testing.assert_array_equal(mw.cpu().numpy(), mc.cpu().numpy())
    hc, ht, hn = synth.gen_host("blob", synth.BASE_SEED + 2, 0, n, 480, 640, 4, seq_len=120)
    Fo, mo = oracle.solve_batch(hc, ht, hn, "bk")
    np.testing.assert_array_equal(Fc.cpu().numpy(), Fo)
    np.testing.assert_array_equal(mc.cpu().numpy(), mo)


def test_warm_start_from_garbage_flow(torch, gc):
    """Any int32 warm flow is clamped, so the result equals the cold solve."""
    rng = np.random.default_rng(5)
    cs, ct, nb = synth.gen_host("blob", 3, 1, 2, 60, 70, 8)
    wf = rng.integers(-(1 << 31), (1 << 31) - 1, size=(2, 4, 60, 70), dtype=np.int64).astype(np.int32)
    g = solver(gc, 8)
    F, m = g.solve(*to_dev(torch, cs, ct, nb, wf)[:3], warm_flow=to_dev(torch, wf)[0])
    check_against_oracle(cs, ct, nb, F.cpu().numpy(), m.cpu().numpy())


def test_c4_1080p_8nbr_sample(torch, gc):
    """C4 shape: 1920x1080 8-neighbour frames (2 of the 1024), full-size parity."""
    n = 2
    cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 3, 0, n, 1080, 1920, 8)
    g = solver(gc, 8)
    F, mask, fs = g.solve(cs, ct, nb, flow_state=True)
    torch.cuda.synchronize()
    hc, ht, hn = synth.gen_host("blob", synth.BASE_SEED + 3, 0, n, 1080, 1920, 8)
    Fo, mo = oracle.solve_batch(hc, ht, hn, "bk")
    np.testing.assert_array_equal(F.cpu().numpy(), Fo)
    np.testing.assert_array_equal(mask.cpu().numpy(), mo)
    fsn = fs.cpu().numpy()
    for i in range(n):
        ok, Ff = cut_cert(hc[i], ht[i], hn[i], fsn[i])
        assert ok and Ff == Fo[i]


def test_serpentine_adversarial_small(torch, gc):
    """C5 shape at reduced size: long snaking augmenting paths."""
    synth.set_serpentine_params(lane=16, big=1 << 20)
    try:
        cs, ct, nb = synth.gen_host("serpentine", synth.BASE_SEED + 4, 0, 2, 256, 384, 4)
    finally:
        synth.set_serpentine_params()
    g = solver(gc, 4)
    F, mask = g.solve(*to_dev(torch, cs, ct, nb))
    check_against_oracle(cs, ct, nb, F.cpu().numpy(), mask.cpu().numpy(), "bk")


# ----------------------------------------------------------------------------- ABI behaviour
def test_host_entry_point_matches_device(torch, gc):
    cs, ct, nb = synth.gen_host("blob", 8, 0, 5, 120, 160, 4)
    g = solver(gc, 4)
    Fd, md = g.solve(*to_dev(torch, cs, ct, nb))
    Fh, mh = g.solve_host(cs, ct, nb)
    np.testing.assert_array_equal(Fh, Fd.cpu().numpy())
    np.testing.assert_array_equal(mh, md.cpu().numpy())
    assert g.launches() > 0


def test_host_entry_point_pipelined_chunks(torch, gc):
    """Host pointers over several chunks (max_batch=2, 7 frames: 4 chunks, ragged last): the H2D
    copy of chunk i+1 overlaps the solve of chunk i in two staging buffers. Cold and warm-started
    (next frames, warm_flow = the previous frames' exported flow) both equal the oracle."""
    n = 7
    cs, ct, nb = synth.gen_host("blob", 11, 0, n + 1, 96, 128, 4)
    g = solver(gc, 4, max_batch=2)
    F, m, fs, st = g.solve_host(cs[:n], ct[:n], nb[:n], flow_state=True, stats=True)
    check_against_oracle(cs[:n], ct[:n], nb[:n], F, m, "bk")
    assert (st[:, 3] == 0).all()
    c1, t1, n1 = (np.ascontiguousarray(a[1:]) for a in (cs, ct, nb))
    Fw, mw = g.solve_host(c1, t1, n1, warm_flow=fs)
    Fd, md = g.solve(*to_dev(torch, c1, t1, n1))
    np.testing.assert_array_equal(Fw, Fd.cpu().numpy())
    np.testing.assert_array_equal(mw, md.cpu().numpy())
    check_against_oracle(c1, t1, n1, Fw, mw, "bk", frames=[0, n - 1])


@pytest.mark.parametrize("H,W,K", [(37, 53, 4), (61, 45, 8), (100, 100, 4)])
def test_host_entry_point_one_frame_chunks_odd_geometry(torch, gc, H, W, K):
    """max_batch=1 (one frame per chunk, two staging buffers in turn) on geometries whose
    sub-buffers need alignment padding, warm start in and flow state out: every sub-buffer of
    a staging buffer lies inside it (the buffer size now comes from the same
    layout), so results equal the device path and the oracle on every frame."""
    n = 5
    cs, ct, nb = synth.gen_host("blob", 21 + K, 0, n + 1, H, W, K)
    g = solver(gc, K, 128, 128, max_batch=1)
    F, m, fs = g.solve_host(cs[:n], ct[:n], nb[:n], flow_state=True)
    check_against_oracle(cs[:n], ct[:n], nb[:n], F, m, "bk")
    for i in range(n):
        ok, Ff = cut_cert(cs[i], ct[i], nb[i], fs[i])
        assert ok and Ff == int(F[i]), i
    c1, t1, n1 = (np.ascontiguousarray(a[1:]) for a in (cs, ct, nb))
    Fw, mw, fw = g.solve_host(c1, t1, n1, warm_flow=fs, flow_state=True)
    check_against_oracle(c1, t1, n1, Fw, mw, "bk")
    for i in range(n):
        ok, Ff = cut_cert(c1[i], t1[i], n1[i], fw[i])
        assert ok and Ff == int(Fw[i]), i


def test_explicit_device_zero(torch, gc):
    """gc_config.device = 0 selects device 0 explicitly (it is not the "default" value)."""
    cs, ct, nb = synth.gen_host("blob", 4, 0, 2, 48, 64, 4)
    g = gc.GridCut(neighborhood=4, max_h=64, max_w=64, device=0)
    F, m = g.solve(*to_dev(torch, cs, ct, nb))
    check_against_oracle(cs, ct, nb, F.cpu().numpy(), m.cpu().numpy())
    g.close()


def test_frame_digest_matches_oracle_masks(torch, gc):
    """gc_frame_digest (the a6 statistics) on solved frames equals the digest of the oracle's
    masks recomputed in numpy from include/gc.h's definition."""
    cs, ct, nb = synth.gen_host("blob", 13, 0, 6, 70, 90, 8)
    g = solver(gc, 8, 128, 128)
    F, m = g.solve(*to_dev(torch, cs, ct, nb))
    dg = g.digest(F, m).cpu().numpy()
    Fo, mo = oracle.solve_batch(cs, ct, nb, "bk")
    for i in range(6):
        pop, h = oracle.mask_digest(mo[i])
        assert (int(dg[i, 0]), int(dg[i, 1]), int(dg[i, 2]), int(dg[i, 3])) == (int(Fo[i]), pop, h, 0), i


def test_range_error(torch, gc):
    cs, ct, nb = synth.gen_host("blob", 9, 0, 3, 40, 40, 4, garbage=True)
    cs[1, 5, 5] = -1
    nb[2, 0, 10, 10] = gc.CAP_MAX + 1
    g = solver(gc, 4)
    F, m = g.solve(*to_dev(torch, cs, ct, nb), allow=(2,))
    assert g.last_status == 2
    F = F.cpu().numpy()
    assert F[1] == -1 and F[2] == -1 and F[0] >= 0
    assert m.cpu().numpy()[1].sum() == 0
    check_against_oracle(cs, ct, nb, F, m.cpu().numpy(), frames=[0])


def test_arg_errors(torch, gc):
    g = solver(gc, 4, 64, 64)
    cs, ct, nb = to_dev(torch, *synth.gen_host("blob", 1, 0, 1, 70, 70, 4))
    with pytest.raises(gc.GcError) as ei:
        g.solve(cs, ct, nb)
    assert ei.value.status == 1
    b = gc.gc_batch(1, 10, 10, None, None, None, None, None, None, None, None)
    assert gc.gc_solve_batch(g.ctx, b, 0) == 1


def test_noconv(torch, gc):
    synth.set_serpentine_params(lane=4, big=1 << 20)
    try:
        cs, ct, nb = synth.gen_host("serpentine", 5, 0, 1, 128, 128, 4)
    finally:
        synth.set_serpentine_params()
    g = gc.GridCut(neighborhood=4, max_h=128, max_w=128, max_launches=3)
    F, m = g.solve(*to_dev(torch, cs, ct, nb), allow=(5,))
    assert g.last_status == 5 and int(F[0]) == -1
    g.close()


def test_same_layout_calls_after_abort(torch, gc):
    """Calls with the previous call's slot layout reuse its balanced border-flow counters
    (no zeroing); a call the watchdog stopped leaves them unbalanced, so the next call zeroes
    them again.  Every solved call stays bit-exact against the oracle."""
    synth.set_serpentine_params(lane=4, big=1 << 20)
    try:
        hard = synth.gen_host("serpentine", 5, 0, 1, 128, 128, 4)
    finally:
        synth.set_serpentine_params()
    g = gc.GridCut(neighborhood=4, max_h=128, max_w=128, max_batch=2, max_launches=3)
    for seed in (31, 32, 33):  # 3 calls, same layout (2 slots of 128 x 128, refilled)
        caps = synth.gen_host("blob", seed, 0, 5, 128, 128, 4)
        F, m = g.solve(*to_dev(torch, *caps))
        check_against_oracle(*caps, F.cpu().numpy(), m.cpu().numpy())
    hard2 = tuple(np.concatenate([h, h]) for h in hard)  # 2 frames: the same layout
    F, m = g.solve(*to_dev(torch, *hard2), allow=(5,))
    assert g.last_status == 5
    caps = synth.gen_host("blob", 34, 0, 5, 128, 128, 4)
    F, m = g.solve(*to_dev(torch, *caps))
    check_against_oracle(*caps, F.cpu().numpy(), m.cpu().numpy())
    g.close()


def test_two_contexts_interleaved(torch, gc):
    a = gc.GridCut(neighborhood=4, max_h=100, max_w=100)
    b = gc.GridCut(neighborhood=8, max_h=100, max_w=100)
    c4 = synth.gen_host("blob", 2, 0, 2, 90, 100, 4)
    c8 = synth.gen_host("blob", 2, 0, 2, 90, 100, 8)
    Fa, ma = a.solve(*to_dev(torch, *c4))
    Fb, mb = b.solve(*to_dev(torch, *c8))
    check_against_oracle(*c4, Fa.cpu().numpy(), ma.cpu().numpy())
    check_against_oracle(*c8, Fb.cpu().numpy(), mb.cpu().numpy())
    a.close(); b.close()


def test_c4_batch_flow_is_cut_of_mask(torch, gc):
    """C4 in the bench's launch configuration (many frames in flight, continuous batching):
    every frame's F equals the capacity of the cut its mask defines (max-flow = min-cut,
    checked on all 256 frames without the oracle), masks equal the oracle's on a stride,
    and a second solve returns the same F and masks (no race leaks into the results)."""
    n = 256
    cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 3, 0, n, 1080, 1920, 8)
    g = solver(gc, 8)
    F, mask = g.solve(cs, ct, nb)
    torch.cuda.synchronize()
    cut = cut_torch(torch, cs, ct, nb, mask)
    bad = torch.nonzero(cut != F).flatten().tolist()
    assert not bad, f"F != cut(mask) on frames {bad[:10]}"
    for _ in range(2):
        F2, mask2 = g.solve(cs, ct, nb)
        bad = torch.nonzero(cut_torch(torch, cs, ct, nb, mask2) != F2).flatten().tolist()
        assert not bad, f"F != cut(mask) on frames {bad[:10]} (repeat solve)"
        assert torch.equal(F, F2) and torch.equal(mask, mask2)
    hc, ht, hn = synth.gen_host("blob", synth.BASE_SEED + 3, 0, 3, 1080, 1920, 8)
    Fo, mo = oracle.solve_batch(hc, ht, hn, "bk")
    np.testing.assert_array_equal(F[:3].cpu().numpy(), Fo)
    np.testing.assert_array_equal(mask[:3].cpu().numpy(), mo)
    del cs, ct, nb


@pytest.mark.parametrize("kind,H,W,K,n,so", [("blob", 240, 320, 4, 300, 1), ("blob", 480, 640, 4, 120, 2),
                                             ("blob", 1080, 1920, 4, 32, 3)])
def test_batch_flow_is_cut_of_mask(torch, gc, kind, H, W, K, n, so):
    """C2 / C3 shapes (and a 4-neighbour 1080p batch): F == cut(mask) on every frame of the
    batch, identical results on a repeat solve, the oracle on the first frames."""
    cs, ct, nb = synth.gen_torch(kind, synth.BASE_SEED + so, 0, n, H, W, K)
    g = solver(gc, K)
    F, mask = g.solve(cs, ct, nb)
    torch.cuda.synchronize()
    bad = torch.nonzero(cut_torch(torch, cs, ct, nb, mask) != F).flatten().tolist()
    assert not bad, f"F != cut(mask) on frames {bad[:10]}"
    F2, mask2 = g.solve(cs, ct, nb)
    assert torch.equal(F, F2) and torch.equal(mask, mask2)
    m = 2
    hc, ht, hn = synth.gen_host(kind, synth.BASE_SEED + so, 0, m, H, W, K)
    Fo, mo = oracle.solve_batch(hc, ht, hn, "bk")
    np.testing.assert_array_equal(F[:m].cpu().numpy(), Fo)
    np.testing.assert_array_equal(mask[:m].cpu().numpy(), mo)


def test_host_watchdog_stops_the_kernel(torch, gc, monkeypatch):
    """The host wall-clock bound (GC_TIMEOUT_S) asks the persistent kernel to stop through the
    mapped host word: an adversarial frame that needs tens of seconds returns GC_ERR_NOCONV
    with F = -1 after ~0.3 s, and the next solve on a fresh context is correct (the GPU is
    left usable)."""
    synth.set_serpentine_params(lane=64, big=1 << 20)
    try:
        scs, sct, snb = synth.gen_torch("serpentine", synth.BASE_SEED + 4, 0, 1, 1080, 1920, 4)
    finally:
        synth.set_serpentine_params()
    monkeypatch.setenv("GC_TIMEOUT_S", "0.3")
    g = gc.GridCut(neighborhood=4, max_h=1080, max_w=1920)
    monkeypatch.delenv("GC_TIMEOUT_S")
    import time
    t0 = time.time()
    F, m = g.solve(scs, sct, snb, allow=(5,))
    assert time.time() - t0 < 10
    assert g.last_status == 5 and int(F[0]) == -1
    assert "timed out" in gc.gc_last_error(g.ctx)
    g.close()
    cs, ct, nb = synth.gen_host("blob", 11, 0, 8, 240, 320, 4)
    g2 = gc.GridCut(neighborhood=4, max_h=240, max_w=320)
    F2, m2 = g2.solve(*to_dev(torch, cs, ct, nb))
    check_against_oracle(cs, ct, nb, F2.cpu().numpy(), m2.cpu().numpy(), "bk", frames=[0, 7])
    g2.close()


def test_c5_4k_serpentine_certified(torch, gc):
    """C5 at its full size (3840x2160 serpentine, 64-px lanes, bimodal {1, 2^20} n-links):
    the CPU oracle needs hours on this frame, so the result is certified without it
    (SURVEY.md §8(c) "flow certificate"): the exported flow is arc-feasible, F(f) == F ==
    cut(mask) (so F is the maximum flow and the mask a minimum cut), and the mask equals the
    residual closure of the excess nodes recomputed on the host (the canonical cut)."""
    synth.set_serpentine_params(lane=64, big=1 << 20)
    try:
        hc, ht, hn = synth.gen_host("serpentine", synth.BASE_SEED + 4, 0, 1, 2160, 3840, 4)
    finally:
        synth.set_serpentine_params()
    g = gc.GridCut(neighborhood=4, max_h=2160, max_w=3840)
    cs, ct, nb = to_dev(torch, hc, ht, hn)
    F, mask, fs = g.solve(cs, ct, nb, flow_state=True)
    torch.cuda.synchronize()
    Fg = int(F[0])
    assert int(cut_torch(torch, cs, ct, nb, mask)[0]) == Fg
    ok, Ff = cut_cert(hc[0], ht[0], hn[0], fs[0].cpu().numpy())
    assert ok and Ff == Fg
    np.testing.assert_array_equal(mask[0].cpu().numpy(), residual_closure_host(hc[0], ht[0], hn[0], fs[0].cpu().numpy()))
    g.close()


def test_serpentine_lane64_parity(torch, gc):
    """C5's lane geometry (64-px lanes) at a size the oracle finishes in seconds: bit-exact
    F and mask against Boykov-Kolmogorov, two frames in flight."""
    synth.set_serpentine_params(lane=64, big=1 << 20)
    try:
        cs, ct, nb = synth.gen_host("serpentine", synth.BASE_SEED + 4, 0, 2, 256, 384, 4)
    finally:
        synth.set_serpentine_params()
    g = solver(gc, 4)
    F, mask = g.solve(*to_dev(torch, cs, ct, nb))
    check_against_oracle(cs, ct, nb, F.cpu().numpy(), mask.cpu().numpy(), "bk")


# ----------------------------------------------------------------------------- sequences
@pytest.mark.parametrize("K,S,L,H,W,mb", [(4, 3, 5, 96, 128, 0), (8, 5, 4, 70, 90, 2), (4, 2, 7, 33, 65, 1)])
def test_sequences_warm_equals_cold_equals_oracle(torch, gc, K, S, L, H, W, mb):
    """gc_solve_sequences: S sequences of L frames in one device pass; frame t warm-started
    from frame t-1's flows (warm=1) and the same schedule cold (warm=0) give the oracle's F and
    mask on every frame -- also with fewer slots than sequences (max_batch < S: a slot takes the
    next sequence when its sequence ends) and a garbage warm start for frame 0; the last
    frames' exported flows are certified (flow certificate)."""
    rng = np.random.default_rng(40 + K)
    cs, ct, nb = synth.gen_host("blob", 31 + K, 0, S * L, H, W, K, seq_len=L)
    cs, ct, nb = (a.reshape((S, L) + a.shape[1:]) for a in (cs, ct, nb))
    g = solver(gc, K, 128, 128, max_batch=mb) if mb else solver(gc, K, 128, 128)
    dcs, dct, dnb = to_dev(torch, cs, ct, nb)
    wf0 = rng.integers(-(1 << 31), (1 << 31) - 1, size=(S, K // 2, H, W), dtype=np.int64).astype(np.int32)
    Fw, mw, fsw, stw = g.solve_sequences(dcs, dct, dnb, warm=True, warm_flow=to_dev(torch, wf0)[0], flow_state=True,
                                         stats=True)
    Fc, mc = g.solve_sequences(dcs, dct, dnb, warm=False)
    assert torch.equal(Fw, Fc) and torch.equal(mw, mc)
    assert (stw[..., 3] == 0).all()
    F, m = Fw.cpu().numpy().reshape(-1), mw.cpu().numpy().reshape(S * L, H, W)
    check_against_oracle(cs.reshape((S * L,) + cs.shape[2:]), ct.reshape((S * L,) + ct.shape[2:]),
                         nb.reshape((S * L,) + nb.shape[2:]), F, m, "bk")
    fs = fsw.cpu().numpy()
    for j in range(S):
        ok, Ff = cut_cert(cs[j, L - 1], ct[j, L - 1], nb[j, L - 1], fs[j])
        assert ok and Ff == int(F[j * L + L - 1]), j


def test_sequences_arg_errors(torch, gc):
    g = solver(gc, 4, 64, 64)
    b = gc.gc_seq_batch(2, 0, 10, 10, None, None, None, None, None, None, None, None, 1)
    assert gc.gc_solve_sequences(g.ctx, b, 0) == 1
    b = gc.gc_seq_batch(2, 3, 10, 10, None, None, None, None, None, None, None, None, 1)
    assert gc.gc_solve_sequences(g.ctx, b, 0) == 1
