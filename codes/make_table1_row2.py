"""Table-1 row-2 code of the paper (BSC p=0.02, N=2^20, frozen set for target FER
0.1 -- PAPER.md:170, acceptance 2 at SPEC.md:498), built with the
reference's own density evolution (subtree-parallel walk of make_codes.py, bit-
identical to construction.density_evolution) + select_frozen (construction.py:397),
cached as a PQCT file.  Runs only in the build container (imports /root/reference)."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_codes as M  # noqa: E402  (puts /root/reference/pkg/src on sys.path)
import numpy as np  # noqa: E402
from polarqkd import construction as C  # noqa: E402
from polarqkd.channel import Bsc  # noqa: E402

if __name__ == "__main__":
    ch, n = Bsc(0.02), 20
    M.CONFIGS["t1r2"] = dict(channel=("bsc", 0.02), n=n, rate=0.0)
    pe = M.build(["t1r2"], 6, int(os.environ.get("WORKERS", "7")))["t1r2"]
    os.makedirs(M.CACHE, exist_ok=True)
    np.save(os.path.join(M.CACHE, "bsc0.02_n20_pe.npy"), pe)
    res = C.ConstructionResult(n=n, channel=ch, pe=pe, quantization=C.DeGrid())
    code = C.select_frozen(res, 0.1)
    path = os.path.join(HERE, "t1r2.pqct")
    C.write_code_table(code, path)
    meta = {"t1r2": {"file": "t1r2.pqct", "channel": "bsc", "param": 0.02, "n": n, "target_fer": 0.1,
                     "rate": code.rate, "beta": C.efficiency(code, ch),
                     "union_bound": C.fer_upper_bound(code, res), "checksum": C.code_table_checksum(path)}}
    with open(os.path.join(HERE, "t1r2.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(meta)
