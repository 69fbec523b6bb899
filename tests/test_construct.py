"""Code construction with density evolution on the GPU.

Pinned against the reference itself: tests/golden/de_ref.npz holds the
reference's density_evolution pe at small (channel, n) points and digests of
its grid tables (tests/golden/make_de_golden.py); codes/*.pqct hold the
frozen sets the reference's DE built for the BASELINE configs.  The GPU DE
differs from the reference only in floating-point summation order, so pe is
compared with a tolerance and the frozen sets must be identical."""
import hashlib
import os
import time

import numpy as np
import pytest

from conftest import golden
from paper_1204_5882_b200 import channel as C
from paper_1204_5882_b200 import codes as K
from paper_1204_5882_b200 import construct as D

POINTS = [("bsc002_n10", C.Bsc(0.02), 10), ("awgn1_n10", C.BiAwgn(1.0), 10),
          ("awgn0161_n12", C.BiAwgn(0.161), 12), ("bsc003_n12", C.Bsc(0.03), 12)]


def digest(a):
    return int.from_bytes(hashlib.blake2b(np.ascontiguousarray(a).tobytes(), digest_size=8).digest(), "little")


def test_grid_tables_bit_identical_to_reference():
    g = golden("de_ref.npz")
    t = D.grid_tables(D.DeGrid())
    assert digest(t.f_idx.astype(np.int32)) == int(g["f_idx_digest"])
    assert digest(t.f_whi.astype(np.float64)) == int(g["f_whi_digest"])
    assert digest(t.z_weights) == int(g["zw_digest"])
    assert digest(t.i_loss) == int(g["il_digest"])


@pytest.mark.parametrize("tag,ch,n", POINTS)
def test_base_density_matches_reference(tag, ch, n):
    g = golden("de_ref.npz")
    assert np.array_equal(D.base_density(ch, D.grid_tables(D.DeGrid())), g["base_" + tag])


def test_rate_rule_rebuilds_c1_from_reference_pe():
    g = golden("de_ref.npz")
    res = D.ConstructionResult(n=10, channel=C.Bsc(0.02), pe=g["pe_bsc002_n10"], quantization=D.DeGrid())
    code = D.select_rate(res, 0.80)
    assert np.array_equal(code.frozen_mask, K.load_config("c1").frozen_mask)


def test_argument_errors():
    with pytest.raises(ValueError):
        D.DeGrid(bins=100)
    with pytest.raises(ValueError):
        D.DeGrid(bins=1001)
    res = D.ConstructionResult(n=2, channel=C.Bsc(0.1), pe=np.array([0.4, 0.1, 0.2, 0.01]),
                               quantization=D.DeGrid())
    with pytest.raises(ValueError):
        D.select_frozen(res, 1.5)
    code = D.select_frozen(res, 0.12)  # 0.01 + 0.1 <= 0.12 < 0.31
    assert list(code.frozen_mask) == [1, 0, 1, 0]


def close_pe(got, ref):
    """Summation-order agreement, by pe band.  The reference convolves with an
    FFT (construction.py:231) whose round-off (~1e-17 absolute per slot, kept
    unless negative) dominates its densities' far tails, so pe of very good
    synthetic channels (< 1e-10, always information bits) is noise there; the
    GPU's direct convolution has none.  Measured: 1e-11 relative at pe >= 1e-2,
    1e-9 at 1e-4, 1e-7 at 1e-6, 6e-6 at 1e-8."""
    rel = np.abs(got - ref) / np.maximum(ref, 1e-300)
    return all(np.all(rel[ref >= lo] <= tol) for lo, tol in ((1e-2, 1e-9), (1e-4, 1e-8), (1e-6, 1e-6), (1e-8, 1e-4)))


@pytest.mark.gpu
@pytest.mark.parametrize("tag,ch,n", POINTS)
def test_gpu_density_evolution_matches_reference(cuda, tag, ch, n):
    g = golden("de_ref.npz")
    ref = g["pe_" + tag]
    res = D.density_evolution(ch, n)
    assert close_pe(res.pe, ref), tag
    # identical frozen sets under both selection rules, wherever the selection
    # boundary lies above the reference's FFT noise floor and is not a near-tie
    r0 = D.ConstructionResult(n=n, channel=ch, pe=ref, quantization=D.DeGrid())
    order = np.lexsort((np.arange(ref.size), ref))
    checked = 0
    for rate in (0.02, 0.05, 0.08, 0.1, 0.2, 0.3, 0.45, 0.5, 0.6, 0.7, 0.8, 0.9):
        k = int(round(rate * ref.size))
        if k == 0 or k >= ref.size:
            continue
        a, b = ref[order[k - 1]], ref[order[k]]
        if a < 1e-6 or (b - a) <= 1e-6 * b:
            continue
        checked += 1
        assert np.array_equal(D.select_rate(res, rate).frozen_mask, D.select_rate(r0, rate).frozen_mask), rate
    for fer in (1e-3, 0.01, 0.1, 0.3):
        assert np.array_equal(D.select_frozen(res, fer).frozen_mask, D.select_frozen(r0, fer).frozen_mask), fer
    assert checked >= 2


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["c2", "c3", "c4"])
def test_gpu_density_evolution_rebuilds_baseline_code(cuda, key):
    """The BASELINE configs' frozen sets (built by the reference's DE, hours on
    the CPU at n = 20) rebuilt on the GPU, identically.  (c5, N = 2^24 at rate
    0.09, is not in this list: its K-boundary pe ~2.2e-10 lies below the
    reference FFT's round-off floor, where the two constructions legitimately
    order channels differently -- see DESIGN.md.)"""
    cfg = K.CONFIGS[key]
    code = K.load_config(key)
    t0 = time.perf_counter()
    res = D.density_evolution(cfg.channel, code.n)
    dt = time.perf_counter() - t0
    got = D.select_rate(res, cfg.rate)
    assert np.array_equal(got.frozen_mask, code.frozen_mask), key
    print(f"{key}: GPU DE n={code.n} in {dt:.1f} s")
