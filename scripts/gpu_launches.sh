# launch list of every kernel of the bench step (cold, serialised)
mkdir -p gpurun_out
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-max-len > gpurun_out/b.json 2>/dev/null; echo bench=$?
python3 -c "import json; j=json.load(open('gpurun_out/b.json')); print('step', j['ms_per_step'], 'bwd', j['roofline']['ms_per_launch'], 'fwd', j['roofline']['fwd']['ms_per_launch'])"
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-max-len --no-graph > gpurun_out/b2.json 2>/dev/null
python3 -c "import json; j=json.load(open('gpurun_out/b2.json')); print('nograph step', j['ms_per_step'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_all.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-max-len > /dev/null 2>&1; echo ncu=$?
python3 - <<'PY'
import csv,collections
lines=open('gpurun_out/launches_all.csv').read().splitlines()
i=[k for k,l in enumerate(lines) if l.startswith('"ID"')][0]
d=collections.defaultdict(list)
for r in csv.DictReader(lines[i:]):
    if r['Metric Name']=='gpu__time_duration.sum': d[r['Kernel Name'][:40]].append(float(r['Metric Value']))
for k,v in d.items(): print(f"{k:42s} {len(v):4d} {sum(v)/len(v):10.0f}")
PY
