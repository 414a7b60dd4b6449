"""Summarise an ncu --metrics gpu__time_duration.sum launch list (dev tool)."""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0, ''])
for d in data:
    n = d['Kernel Name']
    fn = re.search(r'exs::(run_\w+)\(', n)
    inst = re.search(r'\(instance (\d+)\)', n)
    key = (fn.group(1) + '#' + inst.group(1)) if fn and inst else re.sub(r'<.*', '', n)[:60]
    agg[key][0] += 1; agg[key][1] += float(d['Metric Value']); agg[key][2] = d['Grid Size'] + '/' + d['Block Size']
tot = sum(v[1] for v in agg.values())
for k, (c, v, g) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v/1e6:9.3f} ms {100*v/tot:5.1f}% x{c:3d} {g:>24} {k}")
print('total ms', tot / 1e6, 'launches', len(data))
