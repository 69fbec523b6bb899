"""Dump the node types of every width-32 sub-tree the SSC walk enters for a
config (decode order), 2W bytes each in sub-tree-local heap order (index 1 =
root, leaves W..2W-1): input of leaf_bench.cu."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_1204_5882_b200 import codes as K  # noqa: E402
from tree_stats import types, visited  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "c3"
out = sys.argv[2] if len(sys.argv) > 2 else f"/tmp/leaf_{key}.bin"
k = int(sys.argv[3]) if len(sys.argv) > 3 else 5  # sub-tree width 2^k
code = K.load_config(key)
ty = types(code.frozen_mask)
vis = visited(ty)
n = code.n
d32 = n - k
codes = {0: 0, 1: 1, 2: 2, 3: 3}  # tree_stats order = NT_MIXED, NT_RATE0, NT_RATE1, NT_REP
recs = []
for j in np.nonzero(vis[d32])[0]:
    t = np.zeros(2 << k, np.uint8)
    for e in range(k + 1):
        for q in range(1 << e):
            t[(1 << e) + q] = codes[int(ty[d32 + e][(j << e) + q])]
    recs.append(t)
arr = np.array(recs)
arr.tofile(out)
print(key, f"width-{1 << k} sub-trees entered:", len(recs), "mixed:", int((arr[:, 1] == 0).sum()), "->", out)
