"""Top CUDA source lines of an ncu report by warp-stall samples, with the dominant reasons.
usage: ncu_lines.py report.ncu-rep [N]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr, lines = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        d = dict(zip(hdr[4:], r[4:]))
        try:
            smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            smp = 0
        reasons = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
        lines.append((smp, fname, int(r[0]), r[1].strip()[:70], reasons))
tot = sum(l[0] for l in lines) or 1
for smp, f, ln, src, rs in sorted(lines, key=lambda x: -x[0])[:N]:
    top = ",".join(f"{k[6:]}:{v}" for k, v in sorted(rs.items(), key=lambda x: -x[1])[:3])
    print(f"{smp / tot:6.3f} {f}:{ln:<5} {src:<70} {top}")
