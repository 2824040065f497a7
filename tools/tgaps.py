"""Development: per-CTA gaps between consecutive tasks in a trace (gpurun_out/trace_<tag>.npy)."""
import sys

import numpy as np

tr = np.load(f"gpurun_out/trace_{sys.argv[1]}.npy")
t0 = tr[:, 0].min()
st = (tr[:, 0] - t0) / 1e3
du = tr[:, 1] / 1e3
cta = ((tr[:, 2] >> np.uint64(32)) & np.uint64(0xffff)).astype(int)
md = (tr[:, 2] >> np.uint64(56)).astype(int)
fr = (tr[:, 2] & np.uint64(0xffffffff)).astype(int)
o = np.lexsort((st, cta))
st, du, cta, md = st[o], du[o], cta[o], md[o]
same = cta[1:] == cta[:-1]
gap = (st[1:] - (st[:-1] + du[:-1]))[same]
nxt = md[1:][same]
prv = md[:-1][same]
span = (st + du).max()
win = st[1:][same] < 0.85 * span
g = gap[win]
nct = cta.max() + 1
print("span", round(span, 1), "gap CTA-ms per CTA (first 85%)", round(g.sum() / 1e3 / nct, 3))
for lo, hi in [(0, 1), (1, 2), (2, 4), (4, 8), (8, 16), (16, 50), (50, 1e9)]:
    s = (g >= lo) & (g < hi)
    print(f"{lo:5}-{hi:5}: n={s.sum():7d} sum={g[s].sum() / 1e3 / nct:7.3f} ms/CTA")
names = {0: "init", 1: "seed", 2: "bfs", 3: "push", 4: "cseed", 5: "clos", 15: "trans"}
for m in names:
    s = nxt[win] == m
    if s.any():
        print(f"gap before {names[m]:6s} mean {g[s].mean():6.2f} p50 {np.median(g[s]):6.2f} n {s.sum()}")
