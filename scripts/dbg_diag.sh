# general-chunk step timings (dK/dV kernel, CTA 0, warp 4 tracer) for several
# JH_DBG experiment switches
for d in ${DBGS:-0}; do
  JH_DBG=$d timeout 120 python scripts/trace_c2.py 0 > /dev/null 2>&1
  python3 - $d <<'PY'
import json, sys
t = json.load(open('gpurun_out/trace_cta0.json'))['bwd']
ev = [(c, code, arg) for c, r, code, arg in t if r == 2]
pl, sl, ps, ss = [], [], [], []
for (c0, k0, a0), (c1, k1, a1) in zip(ev, ev[1:]):
    if k0 == 30 and k1 == 31: pl.append(c1 - c0)
    if k0 == 31 and k1 in (30, 22): ps.append(c1 - c0)
    if k0 == 32 and k1 == 33: sl.append(c1 - c0)
    if k0 == 33 and k1 in (32, 25): ss.append(c1 - c0)
med = lambda x: sorted(x)[len(x) // 2] if x else -1
print(f"dbg {sys.argv[1]:>3}: P lookups {med(pl):5d} P rest {med(ps):5d} | dS compute {med(sl):5d} dS scatter {med(ss):5d}"
      f" | n={len(pl)} bwd span {t[-1][0]}")
PY
done
