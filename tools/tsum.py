"""Development: one-line summary of a bench log and a trace summary (gpurun_out/)."""
import json
import sys

tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_{tag}.log").read().strip().splitlines()[-1])
    print("bench", d["value"], "Mpx/s", d["ms_per_step"], "ms/step frac", d["roofline"]["frac"],
          "launch_ms", d["roofline"]["avg_launch_ms"], "e2e", (d.get("e2e") or {}).get("value"))
except Exception as e:
    print("bench ?", e)
try:
    t = json.loads(open(f"gpurun_out/trace_c4_{tag}.txt").readline())
    keys = ["span_us", "plain_kernel_ms"] + [k for k in t if k.startswith("cta_ms_") or k.startswith("n_") or k.startswith("mean_us")]
    print({k: t[k] for k in keys})
    print("latency", t["frame_latency_us"], "last", t["last_frames"][:2])
except Exception as e:
    print("trace ?", e)
