# diagonal-half phase timings on CTA 0 for several JH_DBG experiment switches
for d in ${DBGS:-0}; do
  JH_DBG=$d timeout 120 python scripts/trace_c2.py 0 > /dev/null 2>&1
  python3 - $d <<'PY'
import json, sys
t = json.load(open('gpurun_out/trace_cta0.json'))['bwd']
ev = [(c, code) for c, r, code, arg in t if r == 2]
first = lambda k: [c for c, code in ev if code == k][0]
print("dbg", sys.argv[1], "diag half: P phase", first(22) - first(21), "dS phase", first(25) - first(24), "bwd span", t[-1][0])
PY
done
