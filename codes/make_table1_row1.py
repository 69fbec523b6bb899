"""Table-1 row-1 code of the paper (BSC p=0.02, N=2^16, frozen set for target FER
0.1 -- PAPER.md:169), built with the reference's own
density_evolution + select_frozen (construction.py:313, :397) and cached as a
PQCT file.  Used by the SPEC's fixed-vs-float fidelity examples.
Runs only in the build container (imports /root/reference)."""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from polarqkd import construction as C  # noqa: E402
from polarqkd.channel import Bsc  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
res = C.density_evolution(Bsc(0.02), 16)
code = C.select_frozen(res, 0.1)
path = os.path.join(HERE, "t1r1.pqct")
C.write_code_table(code, path)
meta = {"t1r1": {"file": "t1r1.pqct", "channel": "bsc", "param": 0.02, "n": 16, "target_fer": 0.1,
                 "rate": code.rate, "beta": C.efficiency(code, Bsc(0.02)),
                 "union_bound": C.fer_upper_bound(code, res), "checksum": C.code_table_checksum(path)}}
with open(os.path.join(HERE, "t1r1.json"), "w") as fh:
    json.dump(meta, fh, indent=1)
print(meta)
