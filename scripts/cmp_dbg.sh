# A/B timing of JH_DBG experiment switches on the C2 bench (graph replay)
timeout 600 python -u -m pytest tests -m gpu -x -q --timeout 120 2>&1 | tail -1
for d in ${DBGS:-0 0}; do JH_DBG=$d timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-max-len 2>/dev/null | python3 -c "import json,sys; j=json.loads(sys.stdin.read()); print('dbg $d', j['ms_per_step'], j['roofline']['ms_per_launch'], j['roofline']['fwd']['ms_per_launch'])"; done
