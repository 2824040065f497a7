"""Development probe: solve time and per-class profile for configs x chunk sizes x tunables.
usage: probe.py cfg[,cfg] chunk[,chunk] [rounds[,rounds]] [period[,period]]"""
import sys, os, json, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1008_0502_b200 as gc
import synth

ALL = {"qvga": ("blob", 240, 320, 4, 300), "vga": ("blob", 480, 640, 4, 120), "1080p": ("blob", 1080, 1920, 8, 64),
       "serp": ("serpentine", 1080, 1920, 4, 2), "4k": ("serpentine", 2160, 3840, 4, 2)}
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["qvga", "vga", "1080p"]
chunks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
rounds = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
periods = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [0]
for name in cfgs:
    kind, H, W, K, n = ALL[name]
    if kind == "serpentine":
        synth.set_serpentine_params(lane=64, big=1 << 20)
    cs, ct, nb = synth.gen_torch(kind, synth.BASE_SEED + 1, 0, n, H, W, K)
    ref = None
    for chunk, rd, per in itertools.product(chunks, rounds, periods):
        g = gc.GridCut(neighborhood=K, max_h=H, max_w=W, max_batch=chunk, rounds_per_launch=rd, relabel_period=per)
        F, m = g.solve(cs, ct, nb)
        torch.cuda.synchronize()
        if ref is None:
            ref = (F.clone(), m.clone())
        else:
            assert torch.equal(F, ref[0]) and torch.equal(m, ref[1]), "result changed with tunables!"
        best = 1e30
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); F, m, st = g.solve(cs, ct, nb, stats=True); e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        g.set_profiling(True); g.profile(reset=True)
        g.solve(cs, ct, nb); torch.cuda.synchronize()
        prof = g.profile(reset=True)
        px = n * H * W
        print(json.dumps({"cfg": name, "chunk": chunk, "rounds": rd, "period": per, "ms": round(best, 3),
                          "ms_per_frame": round(best / n, 4), "Mpx_s": round(px / best / 1e3, 1),
                          "launches": g.launches(), "st_max": st.max(0).values.tolist(),
                          "prof": {k: (v[0], round(v[1], 2), v[2]) for k, v in prof.items()}}), flush=True)
        g.close()
