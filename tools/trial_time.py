import sys, time
sys.path.insert(0, '.')
from paper_1204_5882_b200 import codes as K
from paper_1204_5882_b200.trials import run_trials
for key, T in (("c3", 1024), ("c2", 4096)):
    code, cfg = K.load_config(key), K.CONFIGS[key]
    r = run_trials(code, cfg.channel, T, 2012, representation="fixed", batch=256 if key == "c3" else 1024)
    print(key, T, "trials: fer", r.fer_measured, "decode-only Mbit/s", round(r.throughput_mbps, 1), "wall s", round(r.wall_time, 2),
          "=> wall Mbit/s", round(T * code.block_size / r.wall_time / 1e6, 1))
