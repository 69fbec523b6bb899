"""CPU oracle pinned against the SPEC's known answers, a brute-force SC, and
the reference's own boxplus (golden fixture).  No GPU."""
import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O


# ---- polar transform KATs and invariants
@pytest.mark.parametrize("u,x", [((0, 0, 0, 0), (0, 0, 0, 0)), ((0, 0, 0, 1), (1, 1, 1, 1)),
                                 ((1, 1, 1, 1), (0, 0, 0, 1))])
def test_transform_kat(u, x):
    assert tuple(O.polar_transform_bytes(u)) == x
    assert tuple(O.polar_transform_numpy(u)) == x


@pytest.mark.parametrize("n", [1, 2, 4, 8, 10, 16])
def test_transform_involution_and_two_restatements(n):
    rng = np.random.default_rng(n)
    for _ in range(20 if n == 16 else 200):
        u = rng.integers(0, 2, 1 << n, dtype=np.uint8)
        x = O.polar_transform_bytes(u)
        assert np.array_equal(O.polar_transform_bytes(x), u)
        if n <= 10:
            assert np.array_equal(x, O.polar_transform_numpy(u))


def test_transform_rejects_non_power_of_two():
    with pytest.raises(ValueError):
        O.polar_transform_bytes(np.zeros(6, np.uint8))


# ---- phi
def test_phi_kats():
    assert abs(O.phi(2.0) - 0.2723) < 1e-3
    assert abs(O.phi(O.phi(5.0)) - 5.0) < 1e-6
    tab = O.phi_table()
    assert abs(tab[512] / 256.0 - O.phi(2.0)) <= 2 ** -7  # table entry at x = 2.0
    with pytest.raises(ValueError):
        O.phi(0.0)


# ---- f pinned to the reference's own boxplus (construction.py:132-135)
def test_f64_matches_reference_boxplus():
    g = golden("boxplus_grid.npz")
    ours = O.fmag64(g["a"], g["b"])
    # the reference's stable form loses relative accuracy for tiny inputs
    # (cancellation of two log1p(~1) terms); compare absolutely there
    tol = 1e-12 + 1e-9 * np.abs(g["f"])
    assert np.all(np.abs(ours - g["f"]) <= np.maximum(tol, 4e-16))


def test_f32_mirror_accuracy():
    rng = np.random.default_rng(0)
    for lo, hi in [(1e-7, 1e-3), (1e-3, 1.0), (1.0, 40.0), (40.0, 1e3), (1e3, 1e8), (1e-7, 1e8)]:
        a = np.exp(rng.uniform(np.log(lo), np.log(hi), 200000)).astype(np.float32)
        b = np.exp(rng.uniform(np.log(lo), np.log(hi), 200000)).astype(np.float32)
        r32 = O.fmag32(a, b).astype(np.float64)
        r64 = O.fmag64(a.astype(np.float64), b.astype(np.float64))
        assert np.max(np.abs(r32 - r64) / r64) < 1e-6


def test_f_identities():
    # f(a, +inf) = a with +inf represented by the saturation value
    a = np.array([0.1, 1.0, 3.0, 7.0])
    assert np.allclose(O.fmag64(a, np.full(4, 30.0)), a, rtol=1e-12)
    assert np.all(O.fmag32(np.zeros(3, np.float32), np.float32([0, 2, 50])) == 0)


def _chain(m, k):
    t = m
    for _ in range(k):
        t = 0.427 * t * t if t < 1.0 else max(0.427, t - 0.6932)
    return t


def test_rate1_guard_bound_is_a_lower_bound():
    # the CUDA rate-1 shortcut chains b(t) <= |boxplus(t, t)|; check it here
    t = np.geomspace(1e-20, 1e4, 20000)
    b = np.where(t < 1.0, 0.427 * t * t, np.maximum(0.427, t - 0.6932))
    assert np.all(b <= O.fmag64(t, t) * (1 + 1e-12))


def test_rate1_tau_table_matches_its_derivation():
    """RATE1_TAU[k] (polarsc.cu) must make the k-fold bound chain reach 1e-30."""
    import os
    import re
    src = open(os.path.join(os.path.dirname(__file__), "..", "paper_1204_5882_b200", "csrc",
                            "polarsc.cu")).read()
    body = src[src.index("RATE1_TAU[26] = {"):]
    body = body[:body.index("}")]
    taus = [float(v) for v in re.findall(r"([0-9.e+-]+)f", body)]
    assert len(taus) == 26
    for k, tau in enumerate(taus):
        assert _chain(np.float32(tau).item(), k) >= 1e-30
        # and the threshold is not absurdly loose: 1% below it the chain fails
        assert _chain(tau * 0.99, k) < 1e-30 or tau < 1e-20


# ---- SC decoders: naive brute force vs C walk vs numpy recursion
MASKS3 = [np.array(m, np.uint8) for m in ([1, 1, 1, 0, 1, 0, 0, 0], [1, 0, 1, 0, 0, 0, 0, 0],
                                           [0] * 8, [1] * 8, [0, 1, 1, 0, 1, 0, 0, 1])]


@pytest.mark.parametrize("mi", range(len(MASKS3)))
def test_sc_all_256_patterns_n3(mi):
    """SPEC.md:248 / acceptance 6: exhaustive n=3, BSC 0.1, all 256 outputs."""
    mask = MASKS3[mi]
    c = np.log(9.0)
    rng = np.random.default_rng(mi)
    for pat in range(256):
        y = ((pat >> np.arange(8)) & 1).astype(np.uint8)
        llr = (1 - 2 * y.astype(np.float64)) * c
        fz = rng.integers(0, 2, 8).astype(np.uint8)
        u_naive, leaf = O.sc_decode_naive(mask, llr, fz)
        u64, x64, st = O.sc_decode(mask, llr, fz, 64, dump=True)
        u32, x32 = O.sc_decode(mask, llr.astype(np.float32), fz, 32)
        urec, xrec = O.sc_decode_recursive(mask, llr, fz)
        assert np.array_equal(u64, u_naive) and np.array_equal(u32, u_naive)
        assert np.array_equal(urec, u_naive)
        assert np.array_equal(x64, O.polar_transform_bytes(u64)) and np.array_equal(x64, xrec)
        assert np.allclose(st[3], leaf, rtol=1e-9, atol=1e-9)


def test_sc_naive_awgn_n4():
    rng = np.random.default_rng(5)
    for _ in range(40):
        mask = rng.integers(0, 2, 16).astype(np.uint8)
        llr = rng.normal(1.0, 2.0, 16)
        fz = rng.integers(0, 2, 16).astype(np.uint8)
        u_naive, leaf = O.sc_decode_naive(mask, llr, fz)
        u, _, st = O.sc_decode(mask, llr, fz, 64, dump=True)
        assert np.array_equal(u, u_naive)
        assert np.allclose(st[4], leaf, rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("n", [6, 9, 12])
def test_c_walk_matches_numpy_recursion(n):
    rng = np.random.default_rng(n)
    N = 1 << n
    for fmode in (O.F_EXACT, O.F_MINSUM):
        mask = (rng.random(N) < 0.5).astype(np.uint8)
        llr = rng.normal(0.8, 1.5, N)
        fz = rng.integers(0, 2, N).astype(np.uint8)
        u, x = O.sc_decode(mask, llr, fz, 64, fmode=fmode)
        ur, xr = O.sc_decode_recursive(mask, llr, fz, fmode=fmode)
        assert np.array_equal(u, ur) and np.array_equal(x, xr)


def test_noiseless_round_trip_n10():
    """all-+-30 LLRs of x, consistent frozen values -> u exactly."""
    rng = np.random.default_rng(3)
    mask = (rng.random(1024) < 0.3).astype(np.uint8)
    for _ in range(100):
        x = rng.integers(0, 2, 1024).astype(np.uint8)
        u = O.polar_transform_bytes(x)
        llr = (1.0 - 2.0 * x) * 30.0
        for prec in (64, 32):
            uh, xh = O.sc_decode(mask, llr, u, prec)
            assert np.array_equal(uh, u) and np.array_equal(xh, x)


def test_batch_driver_matches_single():
    rng = np.random.default_rng(9)
    N = 256
    mask = (rng.random(N) < 0.4).astype(np.uint8)
    llr = rng.normal(1.0, 1.5, (6, N)).astype(np.float32)
    fz = rng.integers(0, 2, (6, N)).astype(np.uint8)
    for prec in (32, 64):
        b = O.sc_decode_batch(mask, llr, fz, precision=prec, threads=3)
        for f in range(6):
            assert np.array_equal(b[f], O.sc_decode(mask, llr[f], fz[f], prec)[0])


def test_de_oracle_acceptance6():
    """Acceptance 6: reference DE pe at n=3 within 0.01 of genie-aided
    enumeration over all 2^8 BSC outputs (uses the oracle's naive SC)."""
    de = golden("de_small.npz")
    for p in (0.05, 0.1):
        c = np.log((1 - p) / p)
        pe = np.zeros(8)
        for pat in range(256):
            e = ((pat >> np.arange(8)) & 1)
            prob = np.prod(np.where(e == 1, p, 1 - p))
            llr = (1 - 2 * e.astype(float)) * c  # all-zero codeword sent
            # genie-aided: each bit-channel sees the true (zero) past
            _, leaf = O.sc_decode_naive(np.ones(8, np.uint8), llr, np.zeros(8, np.uint8))
            pe += prob * np.where(leaf < 0, 1.0, np.where(leaf == 0, 0.5, 0.0))
        assert np.max(np.abs(pe - de[f"pe_{p}"])) < 0.01


def test_fixed_batch_driver_matches_single_frame():
    """orc_sc_decode_batch(precision=16) = the fixed-point decoder on the
    quantised LLRs, frame by frame, whatever the thread count."""
    rng = np.random.default_rng(9)
    n, F = 9, 6
    N = 1 << n
    mask = (rng.random(N) < 0.4).astype(np.uint8)
    llr = rng.normal(0.7, 2.0, (F, N)).astype(np.float32)
    fz = rng.integers(0, 2, (F, N)).astype(np.uint8)
    ref = np.array([O.sc_decode_fixed(mask, O.quantize_q88(llr[f]), fz[f])[0] for f in range(F)])
    for t in (1, 3):
        assert np.array_equal(O.sc_decode_batch(mask, llr, fz, precision=16, threads=t), ref)


def test_fixed_f_is_table_boxplus_within_2_lsb():
    """The fixed-point f (read back through an n = 1 stage dump) is the exact
    boxplus to within 2 LSB (three roundings of at most 1/2 LSB each), sign =
    product of signs, |f| <= min(|a|, |b|); and the table is the spec'd form."""
    corr = O.corr_table_q88()
    k = np.arange(4097)
    assert np.array_equal(corr, np.rint(256 * np.log1p(np.exp(-k / 256.0))).astype(np.int16))
    rng = np.random.default_rng(31)
    mask = np.array([0, 0], np.uint8)
    for _ in range(3000):
        a, b = (int(v) for v in rng.integers(-4000, 4001, 2))
        _, _, st = O.sc_decode_fixed(mask, np.array([a, b], np.int16), np.zeros(2, np.uint8), dump=True)
        f = int(st[1, 0])
        assert abs(f) <= min(abs(a), abs(b))
        if a and b and f:
            assert (f < 0) == ((a < 0) != (b < 0))
        if a == 0 or b == 0:
            assert f == 0
            continue
        x, y = abs(a) / 256.0, abs(b) / 256.0
        exact = min(x, y) + np.log1p(np.exp(-(x + y))) - np.log1p(np.exp(-abs(x - y)))
        assert abs(abs(f) - 256 * exact) <= 2.0
