"""Top CUDA source lines by (non-barrier) warp-stall samples from an ncu
`--page source --csv --print-source cuda,sass` export:
python tools/src_lines.py <csv> [n] [--funcs]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
hdr = None
agg = collections.Counter()
ins = collections.Counter()
src = {}
func = None
fname = ''
fagg = collections.Counter()
reasons = collections.defaultdict(collections.Counter)
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].rsplit('/', 1)[-1]
        continue
    if r[0] == 'Function Name':
        func = r[1][:70]
        continue
    if r[0] == 'Line No':
        hdr = {c: i for i, c in enumerate(r)}
        st = [i for c, i in hdr.items() if c.startswith('stall_') and '(Not' not in c and c != 'stall_barrier']
        names = {i: c for c, i in hdr.items()}
        continue
    if hdr is None or not r[0].isdigit() or len(r) < len(hdr) or r[2] != '-':
        continue
    line = (fname, int(r[0]))
    s = sum(int(r[i] or 0) for i in st)
    agg[line] += s
    fagg[func] += s
    ins[line] += int(r[hdr['Instructions Executed']] or 0)
    src[line] = r[1].strip()
    for i in st:
        reasons[line][names[i][6:]] += int(r[i] or 0)
skip = [a for a in sys.argv[3:] if a.startswith('--skip=')]
if skip:
    for key in list(agg):
        if key[0].startswith(skip[0][7:]):
            del agg[key]
T = sum(agg.values())
print('non-barrier samples', T)
if '--funcs' in sys.argv:
    for f, v in fagg.most_common(15):
        print(f'{100 * v / T:5.1f}%  {f}')
for line, v in agg.most_common(n):
    top = ' '.join(f'{k}={100 * c / max(v, 1):.0f}' for k, c in reasons[line].most_common(3))
    print(f'{100 * v / T:5.1f}% {line[0][:10]}:{line[1]:<5} ins={ins[line]:<10} {src[line][:70]:70s} {top}')
