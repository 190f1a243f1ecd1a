"""Print the forward's per-role timeline of one CTA from gpurun_out/trace_cta<N>.json
(written by trace_c2.py): producer Q (1) / K (2) / V (3) loads, MMA S issue (10)
/ PV issue (11), epilogue S-ready (40) / P-stored (41), in cycles."""
import json
import sys

cta = sys.argv[1] if len(sys.argv) > 1 else "0"
ev = json.load(open(f"gpurun_out/trace_cta{cta}.json"))["fwd"]
names = {1: "Q", 2: "K", 3: "V", 10: "S-mma", 11: "PV-mma", 40: "ep-start", 41: "ep-done", 50: "ch-mask",
         51: "ch-sat", 52: "ch-gen", 54: "ch-band"}  # 5x: per-chunk end (-DJH_TRACE_CHUNKS=1)
last = {}
for c, r, code, arg in ev:
    d = c - last.get(r, c)
    last[r] = c
    print(f"{c:8d} r{r} {names.get(code, code):>8} {arg:5d}  (+{d})")
