"""Top source lines by non-barrier warp-stall samples from an ncu
`--page source --csv --print-source cuda,sass` export."""
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = r[2]
col = {}
for i, c in enumerate(h):
    col.setdefault(c, i)
reasons = [c for c in h if c.startswith('stall_') and '(Not' not in c and c != 'stall_barrier']
lines = []
for x in r[3:]:
    if not x[0] or len(x) < len(h) or not x[0].isdigit():
        continue
    st = {c: int(x[col[c]] or 0) for c in reasons}
    lines.append((sum(st.values()), int(x[0]), x[1][:90], st))
T = sum(l[0] for l in lines)
print('non-barrier samples', T)
for s, ln, src, st in sorted(lines, reverse=True)[:n]:
    top = sorted(st.items(), key=lambda t: -t[1])[:3]
    print(f'{100 * s / T:5.1f}% L{ln:<5} {src:90s} ' + ' '.join(f'{k[6:]}={100 * v / max(s, 1):.0f}' for k, v in top))
