"""Summarise an `ncu --set full` raw CSV export (tools/profile_round.sh) into
the per-launch JSON that bench.py reads for roofline.traffic:
python tools/ncu_summary.py <raw.csv> <config> <fmode> <out.json>"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, units, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))


def num(k):
    return float(d[k].replace(",", ""))


scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
u = dict(zip(h, units))
rd = num("dram__bytes_read.sum") * scale[u["dram__bytes_read.sum"]]
wr = num("dram__bytes_write.sum") * scale[u["dram__bytes_write.sum"]]
dur = num("gpu__time_duration.sum") * {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "msecond": 1.0, "usecond": 1e-3}.get(
    u["gpu__time_duration.sum"], 1.0)
out = {
    "command": "ncu --set full --clock-control none --import-source on -k regex:sc_decode -s 1 -c 1 "
               f"python tools/prof_decode.py --config {sys.argv[2]} --fmode {sys.argv[3]}; tools/profile_round.sh",
    "kernel": d.get("Kernel Name", "sc_decode_kernel"),
    "config": sys.argv[2],
    "fmode": sys.argv[3],
    "dram__bytes_read.sum": int(rd),
    "dram__bytes_write.sum": int(wr),
    "traffic_bytes_per_launch": int(rd + wr),
    "gpu__time_duration_ms": dur,
    "registers_per_thread": int(num("launch__registers_per_thread")) if "launch__registers_per_thread" in d else None,
}
json.dump(out, open(sys.argv[4], "w"), indent=1)
print(json.dumps(out))
