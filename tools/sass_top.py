"""Top SASS instructions by warp-stall samples from an ncu `--page source
--csv --print-source sass` export: python tools/sass_top.py <csv> [n]"""
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = r[1]
col = {c: i for i, c in enumerate(h)}
reasons = [c for c in h if c.startswith('stall_') and '(Not' not in c]
rows = []
for x in r[2:]:
    if x and x[0] == 'Kernel Name':
        break  # first kernel only
    if len(x) < len(h) or not x[col['Address']].startswith('0x'):
        continue
    st = {c: int(x[col[c]] or 0) for c in reasons}
    rows.append((sum(st.values()), x[col['Address']], x[col['Source']].strip(), st, int(x[col['Instructions Executed']] or 0)))
T = sum(t[0] for t in rows)
print('samples', T, 'instructions', len(rows))
for s, a, src, st, ex in sorted(rows, key=lambda t: -t[0])[:n]:
    top = sorted(st.items(), key=lambda t: -t[1])[:2]
    print(f'{100 * s / T:5.1f}% {a[-5:]} {src[:60]:60s} ex={ex:<8} ' + ' '.join(f'{k[6:]}={100 * v / max(s, 1):.0f}' for k, v in top))
