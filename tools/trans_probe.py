"""Development: where the phase-transition time goes (profiling counters pdbg[9..14]: count,
head = slot words + BFS scan, decision, set bits, enqueue batches, tail) on the C3 sequence
pass (warm and cold), C2 and C4."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1008_0502_b200 as gc  # noqa: E402
import synth  # noqa: E402


def summarize(g, name, ms):
    dbg = gc.debug_counters(g.ctx, reset=True)
    prof = g.profile(reset=True)
    n = max(dbg[9], 1)
    out = {"case": name, "kernel_ms": ms, "transitions": dbg[9],
           "us_head": round(dbg[10] / n / 1e3, 2), "us_decide": round(dbg[11] / n / 1e3, 2),
           "us_bits": round(dbg[12] / n / 1e3, 2), "us_enqueue": round(dbg[13] / n / 1e3, 2),
           "us_tail": round(dbg[14] / n / 1e3, 2),
           "enq_us": [round(dbg[i] / n / 1e3, 2) for i in (15, 16, 17, 18)]}
    out["prof"] = {k: (v[0], round(v[1], 3)) for k, v in prof.items()}
    print(json.dumps(out), flush=True)


def seq_case(warm):
    H, W, K, S, L = 480, 640, 4, 8, 120
    cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + 2, 0, S * L, H, W, K, seq_len=L)
    cs, ct, nb = (a.view((S, L) + tuple(a.shape[1:])) for a in (cs, ct, nb))
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
    for _ in range(2):
        g.solve_sequences(cs, ct, nb, warm=warm)
    torch.cuda.synchronize()
    g.set_profiling(True)
    gc.debug_counters(g.ctx, reset=True)
    g.profile(reset=True)
    g.kernel_ms(reset=True)
    g.solve_sequences(cs, ct, nb, warm=warm)
    torch.cuda.synchronize()
    summarize(g, f"c3seq_{'warm' if warm else 'cold'}", round(g.kernel_ms(reset=True), 3))
    g.close()


def batch_case(name, H, W, K, n, off):
    cs, ct, nb = synth.gen_torch("blob", synth.BASE_SEED + off, 0, n, H, W, K)
    g = gc.GridCut(neighborhood=K, max_h=H, max_w=W)
    for _ in range(2):
        g.solve(cs, ct, nb)
    torch.cuda.synchronize()
    g.set_profiling(True)
    gc.debug_counters(g.ctx, reset=True)
    g.profile(reset=True)
    g.kernel_ms(reset=True)
    g.solve(cs, ct, nb)
    torch.cuda.synchronize()
    summarize(g, name, round(g.kernel_ms(reset=True), 3))
    g.close()


seq_case(True)
seq_case(False)
batch_case("c2", 240, 320, 4, 300, 1)
batch_case("c4", 1080, 1920, 8, 1024, 3)
