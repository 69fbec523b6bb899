"""Join an ncu SASS source page with nvdisasm's inline line info.

python tools/sass_profile.py <nvdisasm -c -gi output> <ncu --page source --csv --print-source sass> [file-substr] [top]

Prints warp-stall samples and executed (warp-level) instructions per device
function, per stall reason, per innermost source line and per inline call
chain restricted to the files matching file-substr (default serial_q88).
"""
import collections
import csv
import re
import sys

dis, sass = sys.argv[1], sys.argv[2]
pos = [a for a in sys.argv[3:] if not a.startswith("--")]
sub = pos[0] if pos else "serial_q88"
top = int(pos[1]) if len(pos) > 1 else 40

# --- static side: per instruction (in order): function, inline chain [(file, line), ...] innermost first
ins = []
func = None
chain = []
pending = []
for l in open(dis):
    m = re.match(r"^(\$?_Z\S+|\$__\S+):\s*$", l)
    if m:
        func = m.group(1).split("$")[-1]
        continue
    m = re.match(r'^\s*//## File "([^"]+)", line (\d+)', l)
    if m:
        pending.append((m.group(1).rsplit("/", 1)[-1], int(m.group(2))))
        continue
    m = re.match(r"^\s+/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        if pending:
            chain = pending
            pending = []
        ins.append((int(m.group(1), 16), func, tuple(chain), m.group(2).strip()))
# --- dynamic side
rows = list(csv.reader(open(sass)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = {c: i for i, c in enumerate(rows[hi])}
stall_cols = [(c[6:], i) for c, i in hdr.items() if c.startswith("stall_") and "Not Issued" not in c]
dyn = [r for r in rows[hi + 1:] if r and r[0].startswith("0x")]
assert len(dyn) == len(ins), (len(dyn), len(ins))


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


by_func = collections.Counter()
ex_func = collections.Counter()
by_reason = collections.Counter()
by_line = collections.Counter()
ex_line = collections.Counter()
by_chain = collections.Counter()
ex_chain = collections.Counter()
by_op = collections.Counter()
tot = 0
tot_ex = 0
only = [a[7:] for a in sys.argv if a.startswith("--only=")]
skipf = [a[7:] for a in sys.argv if a.startswith("--skip=")]
for (off, fn, ch, text), r in zip(ins, dyn):
    if only and not any(o in fn for o in only):
        continue
    if any(o in fn for o in skipf):
        continue
    s = num(r[hdr["# Samples"]])
    e = num(r[hdr["Instructions Executed"]])
    tot += s
    tot_ex += e
    by_func[fn] += s
    ex_func[fn] += e
    for name, i in stall_cols:
        by_reason[name] += num(r[i])
    mine = [c for c in ch if sub in c[0]]
    key = mine[0] if mine else (ch[0] if ch else ("?", 0))
    by_line[key] += s
    ex_line[key] += e
    ck = tuple(c[1] for c in mine)
    by_chain[ck] += s
    ex_chain[ck] += e
    by_op[text.split()[0] if not text.startswith("@") else text.split()[1]] += s
print(f"samples {tot}  warp instructions executed {tot_ex}")
print("-- per function")
for k, v in by_func.most_common():
    print(f"{100 * v / tot:5.1f}%  ex={ex_func[k]:10d}  {k}")
print("-- per stall reason")
for k, v in by_reason.most_common(8):
    print(f"{100 * v / tot:5.1f}%  {k}")
print("-- per opcode (samples)")
for k, v in by_op.most_common(12):
    print(f"{100 * v / tot:5.1f}%  {k}")
print("-- per innermost line")
for k, v in by_line.most_common(top):
    print(f"{100 * v / tot:5.1f}%  ex={ex_line[k]:10d}  {k[0]}:{k[1]}")
print("-- per inline chain (lines, innermost first)")
for k, v in by_chain.most_common(top):
    print(f"{100 * v / tot:5.1f}%  ex={ex_chain[k]:10d}  {' < '.join(map(str, k))}")
