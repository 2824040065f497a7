"""Quick performance probe (development aid): per-config solve time and kernel-class profile."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1008_0502_b200 as gc
import synth

cfgs = [("qvga", "blob", 240, 320, 4, 300), ("vga", "blob", 480, 640, 4, 32), ("1080p", "blob", 1080, 1920, 8, 16)]
if len(sys.argv) > 1:
    cfgs = [c for c in cfgs if c[0] in sys.argv[1:]]
for name, kind, H, W, K, n in cfgs:
    cs, ct, nb = synth.gen_torch(kind, synth.BASE_SEED + 1, 0, n, H, W, K)
    g = gc.GridCut(neighborhood=K, max_h=max(H, 1080), max_w=max(W, 1920))
    g.solve(cs, ct, nb)
    torch.cuda.synchronize()
    for prof in (False, True):
        g.set_profiling(prof)
        g.profile(reset=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        F, m, st = g.solve(cs, ct, nb, stats=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        px = n * H * W
        print(json.dumps({"cfg": name, "prof": prof, "ms": round(ms, 3), "ms_per_frame": round(ms / n, 4),
                          "Mpx_s": round(px / ms / 1e3, 1), "launches": g.launches(),
                          "stats0": st[0].tolist(), "stats_max": st.max(0).values.tolist(),
                          "profile": {k: (v[0], round(v[1], 3)) for k, v in g.profile().items()}}), flush=True)
    g.close()
