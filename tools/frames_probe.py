"""Per-frame solver statistics for a config (development aid)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1008_0502_b200 as gc
import synth
kind, H, W, K, n, seed, t0 = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), int(sys.argv[6]), int(sys.argv[7])
rounds = int(os.environ.get("ROUNDS", "0"))
cs, ct, nb = synth.gen_torch(kind, seed, t0, n, H, W, K)
g = gc.GridCut(neighborhood=K, max_h=H, max_w=W, rounds_per_launch=rounds)
F, m, st = g.solve(cs, ct, nb, stats=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.solve(cs, ct, nb); e1.record(); torch.cuda.synchronize()
print("ms", round(e0.elapsed_time(e1), 3), "launches", g.launches())
for i in range(n):
    print(i, "F", int(F[i]), "mask", int(m[i].sum()), "push_steps/relabels/sweeps", st[i, :3].tolist())
