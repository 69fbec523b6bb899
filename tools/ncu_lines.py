"""Per-source-line warp-stall summary of an ncu --set full capture:
python tools/ncu_lines.py <source csv from `ncu -i X --page source --csv --print-source cuda,sass`> [lo hi]
Lines sorted by non-barrier samples; optional line range filter."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 10 ** 9)
hs = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
hdr = rows[hs[0]]
cols = {}
for i, h in enumerate(hdr):
    cols.setdefault(h, i)
bi, si, ie = cols["stall_barrier"], cols["# Samples"], cols["Instructions Executed"]
stalls = [(h, i) for h, i in cols.items() if h.startswith("stall_") and "Not Issued" not in h]
end = hs[1] - 2 if len(hs) > 1 else len(rows)
lines = []
for r in rows[hs[0] + 1:end]:
    if r and r[0].isdigit() and lo <= int(r[0]) <= hi:
        s, b = num(r[si]), num(r[bi])
        st = sorted(((h[6:], num(r[i])) for h, i in stalls if h != "stall_barrier"), key=lambda x: -x[1])[:3]
        lines.append((s - b, int(r[0]), b, num(r[ie]), st, r[1].strip()[:80]))
tot = sum(x[0] for x in lines)
print("non-barrier samples:", tot, " barrier samples:", sum(x[2] for x in lines))
for x in sorted(lines, reverse=True)[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    print(f"{x[1]:5d} nb={x[0]:7d} ({100 * x[0] / max(tot, 1):4.1f}%) bar={x[2]:7d} inst={x[3]:11d} {x[4]} | {x[5]}")
