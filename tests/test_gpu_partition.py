"""NEXT-3: the band partition of each frame
(gc_set_partitions) -- an owner-computes domain decomposition of one frame over `parts` CTA
groups, emulated in one kernel on one device.  The bands only change WHO runs a tile's tasks,
so every result must stay bit-exact against the CPU oracle, for every part count, with frames
refilled into slots, with warm starts, and on a full-size 4K frame."""
import numpy as np
import pytest

import oracle
import synth
from certify import check_against_oracle, cut_cert

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


def to_dev(torch, *arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrs]


def test_bad_part_counts(gc):
    g = gc.GridCut(neighborhood=4, max_h=64, max_w=64)
    for bad in (0, -1, gc.PARTS_MAX + 1):
        with pytest.raises(gc.GcError):
            g.set_partitions(bad)
    g.set_partitions(gc.PARTS_MAX)
    g.set_partitions(1)
    g.close()


@pytest.mark.parametrize("K", [4, 8])
@pytest.mark.parametrize("parts", [2, 3, 8])
def test_random_grids_partitioned(torch, gc, K, parts):
    """Random caps (ties, zeros, off-grid garbage) on ragged sizes, including frames with
    fewer tile rows than bands (bands left empty)."""
    rng = np.random.default_rng(900 + 10 * K + parts)
    g = gc.GridCut(neighborhood=K, max_h=160, max_w=160)
    g.set_partitions(parts)
    for (H, W) in [(1, 7), (33, 32), (70, 97), (130, 45), (160, 160)]:
        for tmax, nmax in [(3, 3), (1000, 50), (50, 1000)]:
            cs, ct, nb = synth.random_caps(rng, H, W, K, tmax=tmax, nmax=nmax, zero_frac=0.3, garbage=True, n=3)
            F, mask = g.solve(*to_dev(torch, cs, ct, nb))
            check_against_oracle(cs, ct, nb, F.cpu().numpy(), mask.cpu().numpy())
    g.close()


@pytest.mark.parametrize("parts", [2, 4])
def test_refilled_slots_partitioned(torch, gc, parts):
    """More frames than slots (max_batch 3): every slot is refilled on the device while the
    bands' rings hold other frames' tasks."""
    H, W, K, n = 240, 320, 4, 11
    cs, ct, nb = synth.gen_host("blob", synth.BASE_SEED + 11, 0, n, H, W, K)
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W, max_batch=3)
    g.set_partitions(parts)
    F, mask = g.solve(*to_dev(torch, cs, ct, nb))
    check_against_oracle(cs, ct, nb, F.cpu().numpy(), mask.cpu().numpy(), algo="bk")
    g.close()


def test_serpentine_partitioned(torch, gc):
    """Long augmenting paths winding through every band (lane 16): flow crosses each band
    border many times."""
    synth.set_serpentine_params(lane=16, big=1 << 20)
    try:
        H, W, K = 200, 260, 4
        cs, ct, nb = synth.gen_host("serpentine", synth.BASE_SEED + 12, 0, 2, H, W, K)
        g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
        g.set_partitions(4)
        F, mask = g.solve(*to_dev(torch, cs, ct, nb))
        check_against_oracle(cs, ct, nb, F.cpu().numpy(), mask.cpu().numpy(), algo="bk")
        g.close()
    finally:
        synth.set_serpentine_params()


def test_warm_sequences_partitioned(torch, gc):
    """gc_solve_sequences with warm starts under a 3-band partition == the unpartitioned
    pass == the oracle (first and last frame of each sequence)."""
    H, W, K, S, L = 120, 160, 4, 2, 5
    cs, ct, nb = synth.gen_host("blob", synth.BASE_SEED + 13, 0, S * L, H, W, K, seq_len=L)
    d = [torch.from_numpy(a.reshape((S, L) + a.shape[1:])).cuda() for a in (cs, ct, nb)]
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
    F1, m1 = g.solve_sequences(*d, warm=True)
    g.set_partitions(3)
    F3, m3 = g.solve_sequences(*d, warm=True)
    assert np.array_equal(F1.cpu().numpy(), F3.cpu().numpy())
    assert np.array_equal(m1.cpu().numpy(), m3.cpu().numpy())
    Fh, mh = F3.cpu().numpy().reshape(-1), m3.cpu().numpy().reshape((S * L, H, W))
    check_against_oracle(cs, ct, nb, Fh, mh, algo="bk", frames=[0, L - 1, L, S * L - 1])
    g.close()


def test_4k_frame_partitioned_8(torch, gc):
    """One full-size 3840 x 2160 blob frame (8-neighbour) split into 8 bands: F and mask equal
    Boykov-Kolmogorov's, the exported flow certifies F, and the profiling counters saw
    requests cross band borders (none without the partition)."""
    H, W, K = 2160, 3840, 8
    cs, ct, nb = synth.gen_host("blob", synth.BASE_SEED + 14, 0, 1, H, W, K)
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
    dcs, dct, dnb = to_dev(torch, cs, ct, nb)
    g.set_profiling(True)
    gc.debug_counters(g.ctx, reset=True)
    F1, m1 = g.solve(dcs, dct, dnb)
    torch.cuda.synchronize()
    assert gc.debug_counters(g.ctx, reset=True)[19] == 0
    g.set_partitions(8)
    F8, m8, fs = g.solve(dcs, dct, dnb, flow_state=True)
    torch.cuda.synchronize()
    cross = gc.debug_counters(g.ctx, reset=True)[19]
    assert cross > 0
    assert int(F8[0]) == int(F1[0]) and np.array_equal(m8.cpu().numpy(), m1.cpu().numpy())
    check_against_oracle(cs, ct, nb, F8.cpu().numpy(), m8.cpu().numpy(), algo="bk")
    ok, Ff = cut_cert(cs[0], ct[0], nb[0], fs[0].cpu().numpy())
    assert ok and Ff == int(F8[0])
    g.close()
