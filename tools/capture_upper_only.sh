# ncu capture of the upper band in isolation (tools/upper_only.py, 256 frames, c3 shape):
# gpu__time_duration + dram bytes of the 4th sc_decode_kernel launch -> profiles/r02/ncu_upper_only.json
# (run under gpurun; bench.py's roofline.upper_band reads the JSON)
FM=${1:-fixed}
mkdir -p gpurun_out
timeout 300 python tools/upper_only.py 256 $FM > gpurun_out/upper_only_plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:sc_decode -s 3 -c 1 --csv --log-file gpurun_out/upper_only_ncu.csv \
    python tools/upper_only.py 256 $FM > gpurun_out/upper_only_ncu.log 2>&1
python - "$FM" <<'PY'
import csv, json, sys
rows = [r for r in csv.reader(open('gpurun_out/upper_only_ncu.csv')) if len(r) > 14]
h = rows[0]; ci = {c: i for i, c in enumerate(h)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3,
         "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
m = {r[ci['Metric Name']]: float(r[ci['Metric Value']].replace(',', '')) * scale.get(r[ci['Metric Unit']], 1)
     for r in rows[1:]}
plain = json.loads(open('gpurun_out/upper_only_plain.log').read().strip().splitlines()[-1])
out = {"command": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                  "--clock-control none -k regex:sc_decode -s 3 -c 1 python tools/upper_only.py 256 " + sys.argv[1],
       "kernel": rows[1][ci['Kernel Name']], "fmode": sys.argv[1], "frames": 256, "N": 1 << 20,
       "upper_levels": 7, "alg_bytes_per_launch": plain["alg_bytes_per_launch"],
       "gpu__time_duration_ms": m["gpu__time_duration.sum"],
       "dram__bytes_read.sum": int(m["dram__bytes_read.sum"]), "dram__bytes_write.sum": int(m["dram__bytes_write.sum"]),
       "traffic_bytes_per_launch": int(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]),
       "events_ms_per_decode_no_profiler": plain["ms_per_decode"]}
out["alg_GBps_ncu"] = round(out["alg_bytes_per_launch"] / out["gpu__time_duration_ms"] / 1e6, 1)
json.dump(out, open('gpurun_out/ncu_upper_only.json', 'w'), indent=1)
print(json.dumps(out))
PY
