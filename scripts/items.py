"""Per-item timeline of the dK/dV kernel on CTA 0 (diagonal halves vs the rest)."""
import json
t = json.load(open('gpurun_out/trace_cta0.json'))['bwd']
mma = [(c, code, arg) for c, r, code, arg in t if r == 1]
items, cur = [], None
for c, code, arg in mma:
    if code == 11:
        cur = {'start': c, 'g': arg, 'p': [], 'ds': []}
    elif code == 12 and cur:
        cur['p'].append(c)
    elif code == 13 and cur:
        cur['ds'].append(c)
    elif code == 15 and cur:
        cur['end'] = c
        items.append(cur)
        cur = None
for it in items:
    n = len(it['p'])
    d = it['ds'][1] - it['start'] if n > 1 else it['end'] - it['start']
    rest = it['end'] - (it['ds'][1] if n > 1 else it['end'])
    print(f"item g={it['g']:4d} halves={n:2d} total={it['end'] - it['start']:6d} first2={d:6d} rest/half={rest / max(n - 2, 1):7.0f}")
print('span', t[-1][0])
