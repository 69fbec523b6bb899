"""Build the frozen sets of the five BASELINE.json configs with the REFERENCE's own
density evolution, then cache them as PQCT code tables (construction.py:464-480).

Runs only in the build container (it imports /root/reference); the GPU box and the
tests consume the committed `codes/*.pqct` + `codes/codes.json`, never this script.

Density evolution is the reference's (construction.py:313-391). The only change is
*who* walks the tree: each DE node depends only on its parent's density, so the
reference's DFS splits into independent subtrees. `_node_step` below re-states the
reference loop body (construction.py:362-389) verbatim in behaviour and calls the
reference's own `_GridOps` methods / `_fill_pruned_good`; subtrees are farmed out to
a process pool. `--check` proves bit-identity with the serial `density_evolution`.

Rate-K selection (BASELINE configs give a rate, not a target FER): information set =
the first K = round(rate*N) positions of the reference's ordering
`np.lexsort((np.arange(N), pe))` (construction.py:406).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from multiprocessing import get_context

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_NUM_THREADS", "1")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
import polarqkd  # noqa: E402
from polarqkd import construction as C  # noqa: E402
from polarqkd.channel import BiAwgn, Bsc  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CACHE = os.path.join(HERE, "_pe_cache")  # git-ignored full pe arrays

CONFIGS = {
    "c1": dict(channel=("bsc", 0.02), n=10, rate=0.80),
    "c2": dict(channel=("bsc", 0.03), n=16, rate=0.75),
    "c3": dict(channel=("bsc", 0.02), n=20, rate=0.83),
    "c4": dict(channel=("biawgn", 1.0), n=20, rate=0.45),
    "c5": dict(channel=("biawgn", 0.161), n=24, rate=0.09),
}

# defaults of density_evolution (construction.py:313-320)
PZ, PI, MF = 1e-9, 1e-3, 1e-30


def make_channel(spec):
    kind, p = spec
    return Bsc(p) if kind == "bsc" else BiAwgn(p)


def _node_step(ops, m, n, depth, offset, pe_out, pe_base):
    """One iteration of the reference DFS body (construction.py:362-389).

    Returns the children to push as [(m, depth, offset), ...] in pop order
    (f-child first), or [] when the node was resolved into pe_out.
    """
    d = n - depth
    if d == 0:
        pe_out[offset - pe_base] = min(0.5, ops.pe(m))
        return []
    z = ops.z_bound(m)
    if np.ldexp(z, d) <= PZ:
        C._fill_pruned_good(pe_out, offset - pe_base, d, z)
        return []
    mi_bound = ops.mutual_info_bound(m)
    if np.ldexp(mi_bound, d) <= PI:
        pe_out[offset - pe_base: offset - pe_base + (1 << d)] = 0.5
        return []
    mi = m[1:-1]
    tiny = (mi > 0.0) & (mi < MF)
    tiny[ops.center - 1] = False
    if tiny.any():
        m = m.copy()
        mi = m[1:-1]
        m[ops.center] += mi[tiny].sum()
        mi[tiny] = 0.0
    half = 1 << (d - 1)
    return [(ops.f_self(m), depth + 1, offset), (ops.g_self(m), depth + 1, offset + half)]


def _run_subtree(args):
    key, m, n, depth, offset = args
    ops = C._grid_ops(C.DeGrid())
    size = 1 << (n - depth)
    pe = np.empty(size)
    stack = [(m, depth, offset)]
    t0 = time.time()
    while stack:
        mm, dd, oo = stack.pop()
        kids = _node_step(ops, mm, n, dd, oo, pe, offset)
        for kid in reversed(kids):  # push g first so f pops first
            stack.append(kid)
    return key, offset, pe, time.time() - t0


def expand(ch, n, split_depth):
    """Walk the top of the tree in the parent process; returns (leaf tasks, pe parts)."""
    ops = C._grid_ops(C.DeGrid())
    base = C._base_density(ch, ops)
    frontier = [(base, 0, 0)]
    tasks, parts = [], []
    while frontier:
        m, depth, offset = frontier.pop()
        if depth >= split_depth or depth == n:
            tasks.append((m, depth, offset))
            continue
        d = n - depth
        pe = np.empty(1 << d)
        kids = _node_step(ops, m, n, depth, offset, pe, offset)
        if not kids:
            parts.append((offset, pe))
        frontier.extend(reversed(kids))
    return tasks, parts


def build(keys, split_depth, workers):
    tasks, pe_all = [], {}
    for key in keys:
        cfg = CONFIGS[key]
        n = cfg["n"]
        pe_all[key] = np.full(1 << n, np.nan)
        sd = min(split_depth, max(0, n - 8))
        t, parts = expand(make_channel(cfg["channel"]), n, sd)
        for off, pe in parts:
            pe_all[key][off: off + pe.size] = pe
        tasks += [(key, m, n, dep, off) for (m, dep, off) in t]
    tasks.sort(key=lambda t: -(t[2] - t[3]))  # biggest subtrees first
    print(f"{len(tasks)} subtree tasks", flush=True)
    ctx = get_context("fork")
    t0 = time.time()
    with ctx.Pool(workers) as pool:
        for i, (key, off, pe, dt) in enumerate(pool.imap_unordered(_run_subtree, tasks)):
            pe_all[key][off: off + pe.size] = pe
            print(f"[{time.time()-t0:8.1f}s] {i+1}/{len(tasks)} {key} off={off} {dt:.1f}s", flush=True)
    for key in keys:
        assert not np.isnan(pe_all[key]).any(), key
    return pe_all


def rate_k_code(key, pe):
    cfg = CONFIGS[key]
    n = cfg["n"]
    N = 1 << n
    K = int(round(cfg["rate"] * N))
    order = np.lexsort((np.arange(N), pe))
    mask = np.ones(N, dtype=np.uint8)
    mask[order[:K]] = 0
    ub = float(pe[order[:K]].sum())
    code = C.PolarCode(n=n, frozen_mask=mask, channel=make_channel(cfg["channel"]),
                       target_fer=min(ub, 1.0), quantization=C.DeGrid())
    return code, K, ub, order


def save(key, pe):
    os.makedirs(CACHE, exist_ok=True)
    np.save(os.path.join(CACHE, f"{key}_pe.npy"), pe)
    code, K, ub, order = rate_k_code(key, pe)
    path = os.path.join(HERE, f"{key}.pqct")
    C.write_code_table(code, path)
    meta_path = os.path.join(HERE, "codes.json")
    meta = json.load(open(meta_path)) if os.path.exists(meta_path) else {}
    import numba, scipy
    meta[key] = dict(
        file=f"{key}.pqct", channel=CONFIGS[key]["channel"][0], param=CONFIGS[key]["channel"][1],
        n=CONFIGS[key]["n"], rate=CONFIGS[key]["rate"], K=K, frozen=int(code.frozen_count),
        union_bound=ub, checksum=C.code_table_checksum(path),
        pe_sha256=hashlib.sha256(pe.tobytes()).hexdigest(),
        kth_pe=float(pe[order[K - 1]]), next_pe=float(pe[order[K]]) if K < pe.size else None,
        built_with=dict(polarqkd=polarqkd.__version__, numpy=np.__version__,
                        scipy=scipy.__version__, numba=numba.__version__,
                        de="construction.density_evolution defaults (2048 bins, +-30)"),
    )
    json.dump(meta, open(meta_path, "w"), indent=1, sort_keys=True)
    print(f"{key}: K={K} union bound={ub:.4g} -> {path}", flush=True)


def check(n=12):
    """Subtree-parallel DE == serial reference density_evolution, bit for bit."""
    for ch in (Bsc(0.02), BiAwgn(0.161)):
        ref = C.density_evolution(ch, n).pe
        CONFIGS["_chk"] = dict(channel=("bsc", ch.p) if isinstance(ch, Bsc) else ("biawgn", ch.snr),
                               n=n, rate=0.5)
        par = build(["_chk"], 3, 4)["_chk"]
        assert np.array_equal(ref, par), ch
        print("bit-identical:", ch, flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("keys", nargs="*", default=list(CONFIGS))
    ap.add_argument("--split", type=int, default=6)
    ap.add_argument("--workers", type=int, default=7)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    if a.check:
        check()
        sys.exit(0)
    pe_all = build(a.keys, a.split, a.workers)
    for k in a.keys:
        save(k, pe_all[k])
