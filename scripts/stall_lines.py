"""Aggregate ncu warp-stall samples per CUDA source line from a
`ncu -i X --page source --csv --print-source cuda,sass` dump."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else "attn_bwd.cu"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
hdr = None
fname = None
line = None
agg = defaultdict(lambda: defaultdict(float))
tot = defaultdict(float)
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] != "":
        line = int(r[0])
        continue
    d = dict(zip(hdr[2:], r[2:]))
    key = (fname.split("/")[-1], line)
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                agg[key][k] += float(v)
                tot[k] += float(v)
            except ValueError:
                pass
    try:
        agg[key]["samples"] += float(d["Warp Stall Sampling (All Samples)"])
        tot["samples"] += float(d["Warp Stall Sampling (All Samples)"])
    except (KeyError, ValueError):
        pass
print("total samples", tot["samples"], {k: int(v) for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]})
for key, d in sorted(agg.items(), key=lambda x: -x[1]["samples"])[:top]:
    st = sorted(((v, k) for k, v in d.items() if k != "samples"), reverse=True)[:4]
    print(f"{key[0]}:{key[1]:5d} {int(d['samples']):7d} " + " ".join(f"{k[6:]}={int(v)}" for v, k in st if v > 0))
