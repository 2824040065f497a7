"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck): C1 (both
neighbourhoods), a few QVGA frames with warm start and flow export, a sequence pass, and two
1080p 8-neighbour frames; every result is checked against the oracle (tools/sanitize.sh)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1008_0502_b200 as gc  # noqa: E402
import synth  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"


def check(cs, ct, nb, F, m):
    for i in range(cs.shape[0]):
        Fo, mo = oracle.solve(cs[i], ct[i], nb[i], "bk")
        assert int(F[i]) == Fo and np.array_equal(m[i], mo), i


def dev(*a):
    return [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in a]


if which in ("all", "c1"):
    for K in (4, 8):
        cs, ct, nb = synth.gen_host("blob", synth.BASE_SEED, 0, 2, 48, 64, K)
        g = gc.GridCut(neighborhood=K, max_h=64, max_w=64)
        F, m = g.solve(*dev(cs, ct, nb))
        check(cs, ct, nb, F.cpu().numpy(), m.cpu().numpy())
        g.close()
    print("c1 ok", flush=True)
if which in ("all", "c2"):
    cs, ct, nb = synth.gen_host("blob", synth.BASE_SEED + 1, 0, 5, 240, 320, 4)
    g = gc.GridCut(neighborhood=4, max_h=240, max_w=320)
    F, m, fs = g.solve(*dev(cs, ct, nb), flow_state=True)
    check(cs, ct, nb, F.cpu().numpy(), m.cpu().numpy())
    c1, t1, n1 = (np.ascontiguousarray(a[1:]) for a in (cs, ct, nb))
    F2, m2 = g.solve(*dev(c1, t1, n1), warm_flow=fs[:4].contiguous())
    check(c1, t1, n1, F2.cpu().numpy(), m2.cpu().numpy())
    S, L = 2, 3
    sc, st_, sn = synth.gen_host("blob", synth.BASE_SEED + 2, 0, S * L, 120, 160, 4, seq_len=L)
    g2 = gc.GridCut(neighborhood=4, max_h=120, max_w=160)
    a, b, c = dev(sc, st_, sn)
    Fs, ms = g2.solve_sequences(a.view(S, L, 120, 160), b.view(S, L, 120, 160), c.view(S, L, 4, 120, 160), warm=True)
    check(sc, st_, sn, Fs.reshape(-1).cpu().numpy(), ms.reshape(S * L, 120, 160).cpu().numpy())
    print("c2 + sequences ok", flush=True)
if which in ("all", "c4"):
    cs, ct, nb = synth.gen_host("blob", synth.BASE_SEED + 3, 0, 2, 1080, 1920, 8)
    g = gc.GridCut(neighborhood=8, max_h=1080, max_w=1920)
    F, m = g.solve(*dev(cs, ct, nb))
    check(cs, ct, nb, F.cpu().numpy(), m.cpu().numpy())
    print("c4 ok", flush=True)
