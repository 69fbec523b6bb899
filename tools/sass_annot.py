"""Annotated SASS of one device function: nvdisasm -c -gi text + ncu sass csv.
python tools/sass_annot.py <dis> <sass.csv> <function-substr> > out.txt
columns: offset, executed warp instructions, samples, top stall, instruction, innermost src line"""
import csv, re, sys
dis, sass, want = sys.argv[1:4]
ins = []; func = None; chain = []; pending = []; labels = {}
for l in open(dis):
    m = re.match(r"^(\$?_Z\S+|\$__\S+):\s*$", l)
    if m: func = m.group(1).split("$")[-1]; continue
    m = re.match(r"^(\.L_x_\d+):", l)
    if m: pending_label = m.group(1); labels[len(ins)] = pending_label; continue
    m = re.match(r'^\s*//## File "([^"]+)", line (\d+)', l)
    if m: pending.append((m.group(1).rsplit("/", 1)[-1], int(m.group(2)))); continue
    m = re.match(r"^\s+/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        if pending: chain = pending; pending = []
        ins.append((int(m.group(1), 16), func, tuple(chain), m.group(2).strip()))
rows = list(csv.reader(open(sass)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = {c: i for i, c in enumerate(rows[hi])}
st = [(c[6:], i) for c, i in hdr.items() if c.startswith("stall_") and "Not Issued" not in c]
dyn = [r for r in rows[hi + 1:] if r and r[0].startswith("0x")]
def num(x):
    try: return int(x)
    except ValueError: return 0
for k, ((off, fn, ch, text), r) in enumerate(zip(ins, dyn)):
    if want not in fn: continue
    if k in labels: print(labels[k] + ":")
    s = num(r[hdr["# Samples"]]); e = num(r[hdr["Instructions Executed"]])
    top = max(((num(r[i]), n) for n, i in st), default=(0, ""))
    mine = [c for c in ch if "serial" in c[0] or "polarsc" in c[0]]
    src = ":".join(map(str, mine[0])) if mine else ""
    cl = "<".join(str(c[1]) for c in mine[:4])
    print(f"{off:06x} ex={e:9d} s={s:5d} {top[1][:8] if s else '':8s} {text[:70]:70s} {cl}")
