"""Development aid: solve time for a config over a cartesian product of tuning knobs
(environment variables read by gc_create, plus rounds_per_launch as ROUNDS).
usage: sweep.py cfg frames "GC_VIS=1,4,64;GC_ALPHA=0.1,1" [seed_off]"""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1008_0502_b200 as gc
import synth

ALL = {"qvga": ("blob", 240, 320, 4), "vga": ("blob", 480, 640, 4), "1080p": ("blob", 1080, 1920, 8),
       "serp": ("serpentine", 1080, 1920, 4), "4k": ("serpentine", 2160, 3840, 4)}
name, n = sys.argv[1], int(sys.argv[2])
knobs = [kv.split("=") for kv in sys.argv[3].split(";")] if len(sys.argv) > 3 and sys.argv[3] else []
seed_off = int(sys.argv[4]) if len(sys.argv) > 4 else 3
kind, H, W, K = ALL[name]
if kind == "serpentine":
    synth.set_serpentine_params(lane=64, big=1 << 20)
cs, ct, nb = synth.gen_torch(kind, synth.BASE_SEED + seed_off, int(os.environ.get("T0", "0")), n, H, W, K)
ref = None
keys = [k for k, _ in knobs]
for vals in itertools.product(*[v.split(",") for _, v in knobs]):
    env = dict(zip(keys, vals))
    for k, v in env.items():
        os.environ[k] = v
    rounds = int(env.get("ROUNDS", "0"))
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W, rounds_per_launch=rounds)
    F, m, st = g.solve(cs, ct, nb, stats=True)
    torch.cuda.synchronize()
    if ref is None:
        ref = (F.clone(), m.clone())
    assert torch.equal(F, ref[0]) and torch.equal(m, ref[1]), f"result changed with {env}"
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.solve(cs, ct, nb); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    g.set_profiling(True); g.profile(reset=True); g.kernel_ms(reset=True)
    g.solve(cs, ct, nb); torch.cuda.synchronize()
    prof = g.profile(reset=True)
    dbg = gc.debug_counters(g.ctx, reset=True)
    stf = st.float()
    hard = torch.argsort(st[:, 0], descending=True)[:4].tolist()
    print(json.dumps({"cfg": name, "n": n, **env, "ms": round(best, 3), "Mpx_s": round(n * H * W / best / 1e3, 1),
                      "st_mean": [round(x, 1) for x in stf.mean(0).tolist()[:3]], "st_max": st.max(0).values.tolist()[:3],
                      "hard": hard, "cta_ms": {k: round(v[1], 2) for k, v in prof.items()},
                      "tasks": {k: v[2] for k, v in prof.items()},
                      "push_dbg": dict(zip(["real", "lower", "absorbed", "sent", "drained", "rounds", "act_end",
                                            "recv", "noprog", "cseed_tiles", "cseed_full", "clos_tasks", "clos_new"], dbg[:13]))}), flush=True)
    g.close()
    del g
    for k in env:
        os.environ.pop(k, None)
