# time of the first (diagonal) half's phases on CTA 0 of the C2 backward
timeout 120 python scripts/trace_c2.py 0 > /dev/null 2>&1
python3 - <<'PY'
import json
t = json.load(open('gpurun_out/trace_cta0.json'))['bwd']
ev = [(c, code) for c, r, code, arg in t if r == 2]
first = lambda k: [c for c, code in ev if code == k][0]
print("diag half: P phase", first(22) - first(21), "dS phase", first(25) - first(24), "bwd span", t[-1][0])
PY
