# A/B of JH_DBG switches on the steady-state and C2 workloads (same library)
for d in ${DBGS:-0 8}; do
  echo "== JH_DBG=$d"
  JH_DBG=$d L=8192 B=4 timeout 120 python scripts/steady.py
  JH_DBG=$d timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-max-len 2>/dev/null | python3 -c "import json,sys; j=json.loads(sys.stdin.read()); print('C2 step', round(j['ms_per_step']*1e3,1), 'bwd', round(j['roofline']['ms_per_launch']*1e3,1), 'fwd', round(j['roofline']['fwd']['ms_per_launch']*1e3,1))"
done
