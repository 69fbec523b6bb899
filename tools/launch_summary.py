"""Per-kernel summary of an ncu launch list (`--metrics gpu__time_duration.sum
--csv --log-file X`): python tools/launch_summary.py <csv> "<command line>" """
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
tot = collections.defaultdict(float)
cnt = collections.Counter()
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
for r in rows:
    k = r[4][:60]
    tot[k] += float(r[14].replace(",", "")) * scale.get(r[13], 1e-6)
    cnt[k] += 1
T = sum(tot.values())
print(f"ncu --metrics gpu__time_duration.sum --clock-control none: {sys.argv[2] if len(sys.argv) > 2 else ''}")
print("cold-cache serialised launches; shares, not absolutes, are comparable with the bench")
for k, v in sorted(tot.items(), key=lambda t: -t[1]):
    print(f"{k:60s} n={cnt[k]:3d} total={v:10.3f} ms  mean={v / cnt[k]:8.3f} ms  share={100 * v / T:5.1f}%")
