"""SSC tree statistics of a frozen set: per width, how many nodes the decoder
visits and of which type (rate-0 / rate-1 / repetition / mixed)."""
import sys
import os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1204_5882_b200 import codes as K


def types(mask):
    N = mask.size
    n = N.bit_length() - 1
    fz = mask.astype(np.int64)
    levels = []
    last_info = (1 - fz).astype(bool)
    cnt = fz.copy()
    li = last_info.copy()
    levels.append((cnt.copy(), li.copy()))
    for d in range(n - 1, -1, -1):
        c = cnt.reshape(-1, 2).sum(1)
        l2 = li.reshape(-1, 2)[:, 1]
        cnt, li = c, l2
        levels.append((cnt.copy(), li.copy()))
    levels = levels[::-1]  # index by depth
    out = []
    for d, (c, l) in enumerate(levels):
        W = N >> d
        t = np.zeros(c.size, np.uint8)  # 0 mixed
        t[c == W] = 1
        t[c == 0] = 2
        t[(c == W - 1) & l & (W > 1)] = 3
        out.append(t)
    return out


def visited(ty):
    """nodes the SSC walk enters: root, and children of mixed nodes"""
    n = len(ty) - 1
    vis = [np.ones(1, bool)]
    for d in range(1, n + 1):
        par_mixed = ty[d - 1] == 0
        vis.append(np.repeat(par_mixed & vis[d - 1], 2))
    return vis


if __name__ == "__main__":
    for key in sys.argv[1:] or K.available_configs():
        code = K.load_config(key)
        ty = types(code.frozen_mask)
        vis = visited(ty)
        n = code.n
        print(f"== {key} N=2^{n}")
        tot_mixed = 0
        for d in range(n + 1):
            W = 1 << (n - d)
            v = vis[d]
            tt = ty[d][v]
            m = int((tt == 0).sum()); tot_mixed += m
            print(f"W=2^{n-d:2d} visited={v.sum():8d} mixed={m:8d} r0={(tt==1).sum():8d} r1={(tt==2).sum():8d} rep={(tt==3).sum():8d}")
        print("total mixed (internal) nodes:", tot_mixed)
