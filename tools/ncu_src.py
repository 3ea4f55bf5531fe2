"""Per-SASS-line stall samples from `ncu --page source --csv` output:
python tools/ncu_src.py FILE.csv [first_line last_line]"""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3]) if len(sys.argv) > 3 else 10**9
ks = []
cur = None
for r in rows:
    if r and r[0] == 'Kernel Name':
        cur = {'name': r[1], 'rows': []}
        ks.append(cur)
        continue
    if r and r[0] == 'Address':
        cur['hdr'] = r
        continue
    if cur is not None and r:
        cur['rows'].append(r)
k = ks[0]
h = k['hdr']
idx = {n: i for i, n in enumerate(h)}
stall = [n for n in h if n.startswith('stall_') and 'Not Issued' not in n]
print(k['name'], 'total samples', sum(int(r[idx['# Samples']]) for r in k['rows']))
agg = collections.Counter()
tot = 0
for i, r in enumerate(k['rows']):
    if not (lo <= i <= hi):
        continue
    ns = int(r[idx['# Samples']])
    tot += ns
    s = {n: int(r[idx[n]]) for n in stall if int(r[idx[n]]) > 0}
    for n, v in s.items():
        agg[n] += v
    if len(sys.argv) > 2:
        top = sorted(s.items(), key=lambda x: -x[1])[:2]
        print(i, ns, r[idx['Instructions Executed']], r[idx['Source']].strip()[:64], top)
print('range samples', tot, agg.most_common(8))
