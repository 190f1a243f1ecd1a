#!/bin/bash
# A/B the build/var_* libraries on C2 (kernel times + graph step); the in-tree library is restored
cp paper_2508_04711_b200/libjh_hstu.so /tmp/lib_intree.so
for d in ${VARS:-build/var_*}; do
  n=$(basename $d)
  cp $d/libjh_hstu.so paper_2508_04711_b200/libjh_hstu.so
  echo "== $n"
  timeout 300 python scripts/time_c2.py 2>&1 | head -3
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-max-len --no-stack --cp-sweep-gb 0 2>/dev/null | python3 -c "import json,sys; j=json.loads(sys.stdin.read()); print('C2 step', round(j['ms_per_step']*1e3,1), 'us  bwd', round(j['roofline']['ms_per_launch']*1e3,1), 'fwd', round(j['roofline']['fwd']['ms_per_launch']*1e3,1))"
done
cp /tmp/lib_intree.so paper_2508_04711_b200/libjh_hstu.so
