# A/B the in-tree library against build/alt1 and build/alt2 (C2 bench, twice each)
c2() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-max-len 2>/dev/null | python3 -c "import json,sys; j=json.loads(sys.stdin.read()); print('C2', round(j['ms_per_step']*1e3,1), 'bwd', round(j['roofline']['ms_per_launch']*1e3,1), 'fwd', round(j['roofline']['fwd']['ms_per_launch']*1e3,1))"; }
cp paper_2508_04711_b200/libjh_hstu.so /tmp/libA.so
for r in 1 2; do
  echo "== A"; cp /tmp/libA.so paper_2508_04711_b200/libjh_hstu.so; c2
  for v in alt1 alt2; do echo "== $v"; cp build/$v/libjh_hstu.so paper_2508_04711_b200/libjh_hstu.so; c2; done
done
cp /tmp/libA.so paper_2508_04711_b200/libjh_hstu.so
