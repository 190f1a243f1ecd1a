# A/B: the in-tree library vs build/alt/libjh_hstu.so on the steady-state and C2 workloads
run() { for d in ${DBGS:-0}; do JH_DBG=$d L=8192 B=4 timeout 120 python scripts/steady.py; done;
        timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-max-len 2>/dev/null | python3 -c "import json,sys; j=json.loads(sys.stdin.read()); print('C2', j['ms_per_step'], j['roofline']['ms_per_launch'], j['roofline']['fwd']['ms_per_launch'])"; }
echo "== A (in-tree)"; run
cp paper_2508_04711_b200/libjh_hstu.so /tmp/libA.so; cp build/alt/libjh_hstu.so paper_2508_04711_b200/libjh_hstu.so
echo "== B (build/alt)"; run
cp /tmp/libA.so paper_2508_04711_b200/libjh_hstu.so
