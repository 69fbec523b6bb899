"""Stall samples grouped by the OUTERMOST source line of each instruction's inline chain
(the statement in the kernel body), with the top stall reason.
python tools/sass_outer.py <nvdisasm -c -gi of the kernel> <ncu sass csv> [top]"""
import collections, csv, re, sys
dis, sass = sys.argv[1:3]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
ins = []; func = None; chain = []; pending = []
for l in open(dis):
    m = re.match(r"^(\$?_Z\S+|\$__\S+):\s*$", l)
    if m: func = m.group(1).split("$")[-1]; continue
    m = re.match(r'^\s*//## File "([^"]+)", line (\d+)', l)
    if m: pending.append((m.group(1).rsplit("/", 1)[-1], int(m.group(2)))); continue
    m = re.match(r"^\s+/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        if pending: chain = pending; pending = []
        ins.append((func, tuple(chain), m.group(2).strip()))
rows = list(csv.reader(open(sass)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = {c: i for i, c in enumerate(rows[hi])}
st = [(c[6:], i) for c, i in hdr.items() if c.startswith("stall_") and "Not Issued" not in c]
dyn = [r for r in rows[hi + 1:] if r and r[0].startswith("0x")]
assert len(dyn) == len(ins), (len(dyn), len(ins))
num = lambda x: int(x) if x.isdigit() else 0
S = collections.Counter(); E = collections.Counter(); R = collections.defaultdict(collections.Counter); tot = 0
for (fn, ch, text), r in zip(ins, dyn):
    s = num(r[hdr["# Samples"]]); e = num(r[hdr["Instructions Executed"]])
    key = (fn[:40] if "sc_decode_kernel" not in fn else "kernel", ch[-1] if ch else ("?", 0))
    S[key] += s; E[key] += e; tot += s
    for n, i in st: R[key][n] += num(r[i])
src = {}
for f in ("paper_1204_5882_b200/csrc/polarsc.cu", "paper_1204_5882_b200/csrc/serial_q88.cuh"):
    try: src[f.rsplit("/", 1)[-1]] = open(f).read().splitlines()
    except OSError: pass
print("samples", tot)
for k, v in S.most_common(top):
    fn, (f, ln) = k
    text = src.get(f, [""] * (ln + 1))[ln - 1].strip()[:70] if ln and f in src and ln <= len(src[f]) else ""
    rs = ", ".join(f"{n} {100 * c / max(v, 1):.0f}%" for n, c in R[k].most_common(2))
    print(f"{100 * v / tot:5.1f}%  ex={E[k]:10d}  {fn}:{f}:{ln}  [{rs}]  {text}")
