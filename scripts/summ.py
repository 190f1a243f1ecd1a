"""Summarise gpurun_out/: kernel launch times, bench line, head of the trace."""
import csv, collections, json, sys
try:
    rows = [r for r in csv.reader(open('gpurun_out/launches.csv')) if len(r) > 10]
    hdr = rows[0]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
    d = collections.defaultdict(list)
    for r in rows[1:]: d[r[ki][:40]].append(float(r[vi].replace(',', '')))
    for k, v in d.items(): print(k, len(v), round(sum(v) / len(v)))
except Exception as e: print('no launches', e)
try:
    b = json.loads(open('gpurun_out/bench.json').read())
    print('value', b['value'], 'ms', b['ms_per_step'], 'bwd ms', b['roofline']['ms_per_launch'], 'fwd ms', b['roofline']['fwd']['ms_per_launch'], 'e2e', b['e2e']['value'])
except Exception as e: print('no bench', e)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 0
if n:
    t = json.load(open('gpurun_out/trace_cta0.json'))[sys.argv[2] if len(sys.argv) > 2 else 'bwd']
    prev = {}
    for c, r, code, arg in t[:n]:
        print(c, r, code, arg, c - prev.get(r, c)); prev[r] = c
