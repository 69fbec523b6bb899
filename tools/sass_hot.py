"""Aggregate ncu source-page SASS stall samples (barrier stalls excluded) by
code region: python tools/sass_hot.py <sass.csv> [block_bits]"""
import collections
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
bb = int(sys.argv[2]) if len(sys.argv) > 2 else 12
h = r[1]
col = {c: i for i, c in enumerate(h)}
reasons = [c for c in h if c.startswith('stall_') and '(Not' not in c and c != 'stall_barrier']
data = []
for x in r[2:]:
    try:
        a = int(x[col['Address']], 16)
    except ValueError:
        continue
    st = {c: int(x[col[c]] or 0) for c in reasons}
    data.append((a, st, int(x[col['Instructions Executed']] or 0), x[col['Source']]))
base = data[0][0]
tot = collections.Counter()
for a, st, e, s in data:
    tot.update(st)
T = sum(tot.values())
print('non-barrier samples', T, {k: round(100 * v / T, 1) for k, v in tot.most_common(9)})
B = collections.defaultdict(collections.Counter)
for a, st, e, s in data:
    B[(a - base) >> bb].update(st)
for k, c in sorted(B.items(), key=lambda t: -sum(t[1].values()))[:20]:
    v = sum(c.values())
    print(f'{hex(k << bb):>9} {100 * v / T:5.1f}%  ' + ' '.join(f'{n[6:]}={100 * m / v:.0f}' for n, m in c.most_common(4)))
