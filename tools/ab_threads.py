"""A/B of threads per CTA on one config (PQ_OPT_THREADS): python tools/ab_threads.py c2"""
import sys, os, json, subprocess
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
for t in (256, 128, 0):
    out = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--no-cpu-baseline", "--steps", "5",
                          "--threads", str(t)], capture_output=True, text=True).stdout.strip().splitlines()[-1]
    d = json.loads(out)
    print(cfg, "threads", t, d["value"], d["config"].get("threads_per_cta"), d["config"]["subtree_log2"],
          d["roofline"].get("band_share"))
