"""GPU parity: the CUDA decoder (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north star):
  * fp32 oracle mirror (same f, same operation order): decoded u, x and every
    stage LLR equal -- on ALL frames, SSC or plain;
  * f64 exact oracle: decoded bits bit-exact on every frame whose smallest
    |decision LLR| (information positions) is >= 1e-4; stage LLRs within
    |d| <= 1e-4 |ref| + 1e-6 on those frames;
  * FER within the binomial 3-sigma interval of the oracle's FER.
"""
import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O
from paper_1204_5882_b200 import channel as C
from paper_1204_5882_b200 import codes as K
from paper_1204_5882_b200.polar_core import (ScDecoder, pack_bits, polar_transform,
                                             polar_transform_words, sc_decode, unpack_bits)

pytestmark = pytest.mark.gpu


def to_dev(a, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def words_dev(bits, dev):
    return to_dev(pack_bits(bits).view(np.int32), dev)


def from_words(t, N):
    return unpack_bits(t.cpu().numpy().view(np.uint32), N)


def transform_rows(v):
    v = v.copy()
    W = v.shape[-1]
    h = 1
    while h < W:
        r = v.reshape(v.shape[:-1] + (W // (2 * h), 2, h))
        r[..., 0, :] ^= r[..., 1, :]
        h *= 2
    return v


def node_flips(mask, fz, n):
    """Sign-flip pattern of every node's LLRs in the coset-shifted domain:
    node (d, j) is flipped by T_W((v & mask)[jW:(j+1)W])."""
    s = (fz & mask).astype(np.uint8)
    N = 1 << n
    return np.stack([transform_rows(s.reshape(1 << d, N >> d)).ravel() for d in range(n + 1)])


def gpu_decode(dev, code, llr, fz, ssc=True, fmode="exact", want_x=True, subtree_log2=0):
    dec = ScDecoder(code, max_frames=max(1, llr.shape[0]), f_mode=fmode, ssc=ssc,
                    subtree_log2=subtree_log2)
    u, x = dec.decode(to_dev(llr.astype(np.float32), dev), words_dev(fz, dev), want_x=want_x)
    N = code.block_size
    return from_words(u, N), (from_words(x, N) if want_x else None)


def random_code(n, frac, rng, ch=C.BiAwgn(1.0)):
    mask = (rng.random(1 << n) < frac).astype(np.uint8)
    return K.PolarCode(n=n, frozen_mask=mask, channel=ch, target_fer=0.1)


def oracle_batch(code, llr, fz, prec, fmode=O.F_EXACT, threads=8):
    return O.sc_decode_batch(code.frozen_mask, llr.astype(np.float32), fz, precision=prec,
                             fmode=fmode, threads=min(threads, O.max_threads()), min_info=True)


# --------------------------------------------------------------------------
# polar transform (K4)

@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 8, 10, 14, 15, 16, 17, 18, 20])
def test_transform_bit_exact(cuda, n):
    rng = np.random.default_rng(n)
    F = 3 if n >= 18 else 8
    u = rng.integers(0, 2, (F, 1 << n), dtype=np.uint8)
    x = from_words(polar_transform_words(words_dev(u, cuda), n), 1 << n)
    for f in range(F):
        assert np.array_equal(x[f], O.polar_transform_bytes(u[f]))


def test_transform_large_and_inplace(cuda):
    n = 24
    rng = np.random.default_rng(24)
    u = rng.integers(0, 2, (2, 1 << n), dtype=np.uint8)
    w = words_dev(u, cuda)
    polar_transform_words(w, n, out=w)  # in place
    x = from_words(w, 1 << n)
    for f in range(2):
        assert np.array_equal(x[f], O.polar_transform_bytes(u[f]))
    assert np.array_equal(from_words(polar_transform_words(w, n), 1 << n), u)  # involution


def test_transform_spec_kats(cuda):
    assert tuple(polar_transform([0, 0, 0, 1])) == (1, 1, 1, 1)
    assert tuple(polar_transform([1, 1, 1, 1])) == (0, 0, 0, 1)
    assert tuple(polar_transform([0, 0, 0, 0])) == (0, 0, 0, 0)
    with pytest.raises(ValueError):
        polar_transform([1, 0, 1])


# --------------------------------------------------------------------------
# SC decode: exhaustive n = 3 (acceptance 6)

@pytest.mark.parametrize("mask", [[1, 1, 1, 0, 1, 0, 0, 0], [1, 0, 1, 0, 0, 0, 0, 0], [0] * 8,
                                  [1] * 8, [0, 1, 1, 0, 1, 0, 0, 1]])
@pytest.mark.parametrize("ssc", [True, False])
def test_all_256_patterns_n3(cuda, mask, ssc):
    mask = np.array(mask, np.uint8)
    code = K.PolarCode(n=3, frozen_mask=mask, channel=C.Bsc(0.1), target_fer=0.1)
    y = ((np.arange(256)[:, None] >> np.arange(8)) & 1).astype(np.uint8)
    llr = C.channel_llr(C.Bsc(0.1), y).astype(np.float32)
    fz = np.random.default_rng(1).integers(0, 2, (256, 8)).astype(np.uint8)
    u, x = gpu_decode(cuda, code, llr, fz, ssc=ssc)
    for f in range(256):
        un, _ = O.sc_decode_naive(mask, llr[f].astype(np.float64), fz[f])
        assert np.array_equal(u[f], un), f
        assert np.array_equal(x[f], O.polar_transform_bytes(un))


# --------------------------------------------------------------------------
# random codes, all sizes through every code path (warp sub-trees, shared
# sub-trees, HBM levels), SSC and plain, exact and min-sum

@pytest.mark.parametrize("n", [1, 2, 4, 5, 6, 7, 8, 10, 12, 14])
@pytest.mark.parametrize("frac", [0.0, 0.3, 0.7, 1.0])
def test_random_codes_vs_fp32_mirror(cuda, n, frac):
    rng = np.random.default_rng(100 * n + int(10 * frac))
    code = random_code(n, frac, rng)
    F = 16
    llr = rng.normal(0.7, 1.6, (F, 1 << n)).astype(np.float32)
    llr[:, rng.integers(0, 1 << n, 3)] = 0.0  # exact zeros exercise the tie rule / rate-1 guard
    fz = rng.integers(0, 2, (F, 1 << n)).astype(np.uint8)
    ref, _ = oracle_batch(code, llr, fz, 32)
    for ssc in (True, False):
        u, x = gpu_decode(cuda, code, llr, fz, ssc=ssc)
        assert np.array_equal(u, ref), f"ssc={ssc}"
        for f in range(F):
            assert np.array_equal(x[f], O.polar_transform_bytes(u[f]))


@pytest.mark.parametrize("n,log2s", [(12, 7), (13, 8), (16, 10), (16, 12)])
def test_forced_small_subtree_uses_hbm_levels(cuda, n, log2s):
    """Small S pushes many levels into the per-frame HBM/L2 scratch path."""
    rng = np.random.default_rng(n + log2s)
    code = random_code(n, 0.5, rng)
    F = 8
    llr = rng.normal(1.0, 2.0, (F, 1 << n)).astype(np.float32)
    fz = rng.integers(0, 2, (F, 1 << n)).astype(np.uint8)
    ref, _ = oracle_batch(code, llr, fz, 32)
    u, _ = gpu_decode(cuda, code, llr, fz, subtree_log2=log2s)
    assert np.array_equal(u, ref)


@pytest.mark.parametrize("n", [4, 8, 11])
def test_minsum_vs_mirror(cuda, n):
    rng = np.random.default_rng(7 + n)
    code = random_code(n, 0.5, rng)
    llr = rng.normal(0.5, 2.0, (12, 1 << n)).astype(np.float32)
    fz = rng.integers(0, 2, (12, 1 << n)).astype(np.uint8)
    ref, _ = oracle_batch(code, llr, fz, 32, fmode=O.F_MINSUM)
    for ssc in (True, False):
        u, _ = gpu_decode(cuda, code, llr, fz, ssc=ssc, fmode="min-sum")
        assert np.array_equal(u, ref)


# --------------------------------------------------------------------------
# stage LLRs

@pytest.mark.parametrize("n", [3, 6, 9, 12])
def test_stage_dump_vs_oracles(cuda, n):
    rng = np.random.default_rng(n)
    code = random_code(n, 0.45, rng)
    F = 6
    N = 1 << n
    llr = rng.normal(0.8, 1.8, (F, N)).astype(np.float32)
    fz = rng.integers(0, 2, (F, N)).astype(np.uint8)
    dec = ScDecoder(code, max_frames=F)
    u, x, dump = dec.decode_dump(to_dev(llr, cuda), words_dev(fz, cuda))
    dump = dump.cpu().numpy()
    u = from_words(u, N)
    for f in range(F):
        sign = 1.0 - 2.0 * node_flips(code.frozen_mask, fz[f], n)
        u32, _, st32 = O.sc_decode(code.frozen_mask, llr[f], fz[f], 32, dump=True)
        assert np.array_equal(u[f], u32)
        assert np.array_equal(dump[f] * sign, st32)  # every stage LLR, bit for bit (+-0 equal)
        u64, _, st64, lf64 = O.sc_decode(code.frozen_mask, llr[f].astype(np.float64), fz[f], 64,
                                         dump=True, leaf=True)
        if np.min(np.abs(lf64[code.frozen_mask == 0]), initial=np.inf) >= 1e-4:
            assert np.array_equal(u[f], u64)
            got = dump[f].astype(np.float64) * sign
            assert np.all(np.abs(got - st64) <= 1e-4 * np.abs(st64) + 1e-6)


# --------------------------------------------------------------------------
# the five BASELINE configs with the reference-constructed frozen sets

CFG_FRAMES = {"c1": 64, "c2": 32, "c3": 12, "c4": 12, "c5": 2}


def config_batch(key, frames):
    cfg = K.CONFIGS[key]
    code = K.load_config(key)
    N = code.block_size
    xs, ls = [], []
    for j in range(frames):
        x, y = C.frame(cfg.channel, cfg.seed, j, N)
        xs.append(x)
        ls.append(C.channel_llr(cfg.channel, y).astype(np.float32))
    x = np.array(xs)
    u = np.array([O.polar_transform_bytes(xi) for xi in xs])
    return cfg, code, x, u, np.array(ls)


@pytest.mark.parametrize("key", list(K.CONFIGS))
def test_config_parity(cuda, key):
    if key not in K.available_configs():
        pytest.skip(f"{key}.pqct not built")
    cfg, code, x, u_true, llr = config_batch(key, CFG_FRAMES[key])
    ref32, _ = oracle_batch(code, llr, u_true, 32)
    ref64, mi64 = oracle_batch(code, llr, u_true, 64)
    u, xh = gpu_decode(cuda, code, llr, u_true)
    assert np.array_equal(u, ref32)  # bit-exact vs the fp32 mirror on every frame
    clean = mi64 >= 1e-4
    assert np.array_equal(u[clean], ref64[clean])
    ok_gpu = np.all(u == u_true, axis=1)
    assert np.array_equal(ok_gpu, np.all(xh == x, axis=1))
    ok64 = np.all(ref64 == u_true, axis=1)
    F = len(ok_gpu)
    fer, fer64 = 1 - ok_gpu.mean(), 1 - ok64.mean()
    assert abs(fer - fer64) <= 3 * np.sqrt(max(fer64 * (1 - fer64), 1.0 / F) / F)
    if key == "c1":
        g = golden("c1_frames.npz")
        assert np.array_equal(llr[:16], g["llr"])  # inputs are the reference's own


def test_bsc_fused_front_end_matches_llr_path(cuda):
    key = "c1" if "c1" in K.available_configs() else None
    if key is None:
        pytest.skip("c1 not built")
    cfg, code, x, u_true, llr = config_batch(key, 64)
    y = np.array([C.frame(cfg.channel, cfg.seed, j, code.block_size)[1] for j in range(64)])
    dec = ScDecoder(code, max_frames=64)
    u1, x1 = dec.decode(to_dev(llr, cuda), words_dev(u_true, cuda), want_x=True)
    u2, x2 = dec.decode_bsc(words_dev(y, cuda), np.float32(cfg.channel.llr_magnitude),
                            words_dev(u_true, cuda), want_x=True)
    assert np.array_equal(u1.cpu().numpy(), u2.cpu().numpy())
    assert np.array_equal(x1.cpu().numpy(), x2.cpu().numpy())


# --------------------------------------------------------------------------
# SPEC examples and edge cases

def test_noiseless_round_trip_n10(cuda):
    """100 random x at n=10, all LLRs +-30 -> u_hat = T(x)."""
    rng = np.random.default_rng(10)
    code = random_code(10, 0.3, rng)
    x = rng.integers(0, 2, (100, 1024), dtype=np.uint8)
    u = np.array([O.polar_transform_bytes(xi) for xi in x])
    llr = ((1.0 - 2.0 * x) * 30.0).astype(np.float32)
    uh, xh = gpu_decode(cuda, code, llr, u)
    assert np.array_equal(uh, u) and np.array_equal(xh, x)


def test_spec_sc_decode_api_single_frame(cuda):
    rng = np.random.default_rng(4)
    code = random_code(8, 0.5, rng, ch=C.Bsc(0.05))
    x = rng.integers(0, 2, 256, dtype=np.uint8)
    y = C.transmit(C.Bsc(0.05), x, 3, 1)
    llr = C.channel_llr(C.Bsc(0.05), y)
    u = O.polar_transform_bytes(x)
    fv = u[code.frozen_indices()]
    got = sc_decode(code, llr, fv)
    ref, _ = O.sc_decode(code.frozen_mask, llr.astype(np.float32), u, 32)
    assert np.array_equal(got, ref)
    assert np.array_equal(got[code.frozen_indices()], fv)  # frozen positions carry the values
    with pytest.raises(ValueError):
        sc_decode(code, llr[:128], fv)
    with pytest.raises(ValueError):
        sc_decode(code, llr, fv[:-1])


def test_argument_errors(cuda):
    rng = np.random.default_rng(0)
    code = random_code(6, 0.5, rng)
    dec = ScDecoder(code, max_frames=2)
    import torch
    with pytest.raises(ValueError):
        dec.decode(torch.zeros((3, 64), device=cuda))  # > max_frames
    with pytest.raises(ValueError):
        dec.decode(torch.zeros((2, 32), device=cuda))  # wrong N
    u, _ = dec.decode(torch.zeros((0, 64), device=cuda))  # zero frames is a no-op
    assert u.shape[0] == 0


def test_ssc_equals_plain_on_large_random(cuda):
    rng = np.random.default_rng(77)
    code = random_code(16, 0.4, rng, ch=C.BiAwgn(1.0))
    llr = rng.normal(1.0, 2.0, (16, 1 << 16)).astype(np.float32)
    fz = rng.integers(0, 2, (16, 1 << 16)).astype(np.uint8)
    a, _ = gpu_decode(cuda, code, llr, fz, ssc=True)
    b, _ = gpu_decode(cuda, code, llr, fz, ssc=False)
    assert np.array_equal(a, b)


# --------------------------------------------------------------------------
# the f function itself, and the FAST (SFU) mode

def test_f_exact_is_the_mirror_and_fast_is_accurate(cuda):
    import torch
    from paper_1204_5882_b200.polar_core import f_device
    rng = np.random.default_rng(11)
    for lo, hi in [(1e-7, 1e-3), (1e-3, 1.0), (1.0, 8.0), (8.0, 40.0), (40.0, 1e3), (1e3, 1e8), (1e-7, 1e8)]:
        a = np.exp(rng.uniform(np.log(lo), np.log(hi), 200000)).astype(np.float32)
        b = np.exp(rng.uniform(np.log(lo), np.log(hi), 200000)).astype(np.float32)
        a *= np.where(rng.random(a.size) < 0.5, -1, 1).astype(np.float32)
        ta, tb = torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda)
        ex = f_device(ta, tb, "exact").cpu().numpy()
        mirror = O.fmag32(np.abs(a), np.abs(b)) * np.sign(a) * np.sign(b)
        assert np.array_equal(ex, mirror.astype(np.float32))
        ref = O.fmag64(np.abs(a).astype(np.float64), np.abs(b).astype(np.float64))
        fa = f_device(ta, tb, "fast").cpu().numpy().astype(np.float64)
        assert np.all(np.sign(fa) == np.sign(a) * np.sign(b))
        assert np.max(np.abs(np.abs(fa) - ref) / ref) < 2e-6, (lo, hi)


@pytest.mark.parametrize("key", ["c1", "c2", "c3", "c4"])
def test_config_parity_fast_f(cuda, key):
    """FAST f: bit-exact decisions vs the f64 oracle on every frame without a
    near-tie decision LLR; FER within the binomial interval."""
    if key not in K.available_configs():
        pytest.skip(f"{key}.pqct not built")
    cfg, code, x, u_true, llr = config_batch(key, CFG_FRAMES[key])
    ref64, mi64 = oracle_batch(code, llr, u_true, 64)
    u, xh = gpu_decode(cuda, code, llr, u_true, fmode="fast")
    clean = mi64 >= 1e-4
    assert np.array_equal(u[clean], ref64[clean])
    ok_gpu = np.all(u == u_true, axis=1)
    ok64 = np.all(ref64 == u_true, axis=1)
    F = len(ok_gpu)
    fer, fer64 = 1 - ok_gpu.mean(), 1 - ok64.mean()
    assert abs(fer - fer64) <= 3 * np.sqrt(max(fer64 * (1 - fer64), 1.0 / F) / F)


@pytest.mark.parametrize("n", [6, 10, 13])
def test_stage_llrs_fast_within_tolerance(cuda, n):
    """FAST f stage LLRs within 1e-4 relative (+1e-6) of the f64 oracle."""
    rng = np.random.default_rng(n + 100)
    code = random_code(n, 0.45, rng)
    F, N = 4, 1 << n
    llr = rng.normal(0.8, 1.8, (F, N)).astype(np.float32)
    fz = rng.integers(0, 2, (F, N)).astype(np.uint8)
    dec = ScDecoder(code, max_frames=F, f_mode="fast")
    u, _, dump = dec.decode_dump(to_dev(llr, cuda), words_dev(fz, cuda))
    dump = dump.cpu().numpy()
    u = from_words(u, N)
    for f in range(F):
        sign = 1.0 - 2.0 * node_flips(code.frozen_mask, fz[f], n)
        u64, _, st64, lf64 = O.sc_decode(code.frozen_mask, llr[f].astype(np.float64), fz[f], 64,
                                         dump=True, leaf=True)
        if np.min(np.abs(lf64[code.frozen_mask == 0]), initial=np.inf) >= 1e-4:
            assert np.array_equal(u[f], u64)
            got = dump[f].astype(np.float64) * sign
            assert np.all(np.abs(got - st64) <= 1e-4 * np.abs(st64) + 1e-6)


# --------------------------------------------------------------------------
# fixed point: SPEC.md's sc_decode_fixed (Q8.8, phi table) -- integer exact

def fix_f_numpy(a, b, corr):
    ma, mb = np.abs(a).astype(np.int64), np.abs(b).astype(np.int64)
    c = corr.astype(np.int64)
    m = np.minimum(ma, mb) + c[np.minimum(ma + mb, 4096)] - c[np.minimum(np.abs(ma - mb), 4096)]
    m = np.maximum(m, 0)
    return np.where((a < 0) != (b < 0), -m, m)


def test_fixed_f_matches_oracle_table(cuda):
    import torch
    from paper_1204_5882_b200.polar_core import f_device
    assert abs(O.phi_table_q88()[512] / 256.0 - O.phi(2.0)) <= 2 ** -7
    corr = O.corr_table_q88()
    rng = np.random.default_rng(21)
    a = rng.integers(-32767, 32768, 500000).astype(np.float32)
    b = np.where(rng.random(a.size) < 0.5, rng.integers(-600, 601, a.size),
                 rng.integers(-32767, 32768, a.size)).astype(np.float32)
    a[:2000] = rng.integers(-3000, 3001, 2000)
    b[:2000] = a[:2000] + rng.integers(-3, 4, 2000)
    got = f_device(torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda), "fixed").cpu().numpy()
    ref = fix_f_numpy(a.astype(np.int64), b.astype(np.int64), corr)
    assert np.array_equal(got.astype(np.int64), ref)


def fixed_oracle_batch(code, raw, fz):
    return np.array([O.sc_decode_fixed(code.frozen_mask, raw[f], fz[f])[0] for f in range(raw.shape[0])])


@pytest.mark.parametrize("n", [3, 4, 8, 12, 16])
@pytest.mark.parametrize("ssc", [True, False])
def test_fixed_random_codes_bit_exact(cuda, n, ssc):
    rng = np.random.default_rng(300 + n)
    code = random_code(n, 0.45, rng)
    F, N = (8 if n < 16 else 3), 1 << n
    llr = rng.normal(0.8, 1.8, (F, N)).astype(np.float32)
    llr[:, rng.integers(0, N, 3)] = 0.0
    fz = rng.integers(0, 2, (F, N)).astype(np.uint8)
    raw = O.quantize_q88(llr)
    ref = fixed_oracle_batch(code, raw, fz)
    u, _ = gpu_decode(cuda, code, llr, fz, ssc=ssc, fmode="fixed")
    assert np.array_equal(u, ref)


@pytest.mark.parametrize("n", [3, 7, 11])
def test_fixed_stage_dump_bit_exact(cuda, n):
    rng = np.random.default_rng(400 + n)
    code = random_code(n, 0.45, rng)
    F, N = 4, 1 << n
    llr = rng.normal(0.8, 1.8, (F, N)).astype(np.float32)
    fz = rng.integers(0, 2, (F, N)).astype(np.uint8)
    dec = ScDecoder(code, max_frames=F, f_mode="fixed")
    u, _, dump = dec.decode_dump(to_dev(llr, cuda), words_dev(fz, cuda))
    dump = dump.cpu().numpy()
    raw = O.quantize_q88(llr)
    for f in range(F):
        sign = 1 - 2 * node_flips(code.frozen_mask, fz[f], n).astype(np.int64)
        uo, _, st = O.sc_decode_fixed(code.frozen_mask, raw[f], fz[f], dump=True)
        assert np.array_equal(dump[f].astype(np.int64) * sign, st.astype(np.int64))


@pytest.mark.parametrize("key", list(K.CONFIGS))
def test_config_parity_fixed(cuda, key):
    if key not in K.available_configs():
        pytest.skip(f"{key}.pqct not built")
    frames = {"c1": 64, "c2": 16, "c3": 6, "c4": 6, "c5": 1}[key]
    cfg, code, x, u_true, llr = config_batch(key, frames)
    ref = fixed_oracle_batch(code, O.quantize_q88(llr), u_true)
    u, xh = gpu_decode(cuda, code, llr, u_true, fmode="fixed")
    assert np.array_equal(u, ref)
    assert np.array_equal(np.all(u == u_true, axis=1), np.all(xh == x, axis=1))


def test_fixed_bsc_front_end_matches(cuda):
    if "c1" not in K.available_configs():
        pytest.skip("c1 not built")
    cfg, code, x, u_true, llr = config_batch("c1", 64)
    y = np.array([C.frame(cfg.channel, cfg.seed, j, code.block_size)[1] for j in range(64)])
    dec = ScDecoder(code, max_frames=64, f_mode="fixed")
    u1, _ = dec.decode(to_dev(llr, cuda), words_dev(u_true, cuda))
    u2, _ = dec.decode_bsc(words_dev(y, cuda), np.float32(cfg.channel.llr_magnitude), words_dev(u_true, cuda))
    assert np.array_equal(u1.cpu().numpy(), u2.cpu().numpy())


def test_fixed_spec_examples(cuda):
    """noiseless exactness; on the Table-1 row-1 code (BSC 2%,
    N=2^16, FER-0.1 frozen set) 500 frames: >= 98% frame agreement with the
    float decoder and fixed FER <= 2x float FER."""
    from paper_1204_5882_b200.polar_core import sc_decode_fixed, quantize_q88
    rng = np.random.default_rng(12)
    code = random_code(10, 0.3, rng)
    x = rng.integers(0, 2, 1024).astype(np.uint8)
    u = O.polar_transform_bytes(x)
    got = sc_decode_fixed(code, quantize_q88((1.0 - 2.0 * x) * 30.0), u[code.frozen_indices()])
    assert np.array_equal(got, u)
    import os
    path = os.path.join(K.CODES_DIR, "t1r1.pqct")
    if not os.path.exists(path):
        pytest.skip("t1r1.pqct not built")
    code = K.read_code_table(path)
    ch, seed, F = C.Bsc(0.02), 4242, 500
    xs, ls = [], []
    for j in range(F):
        xj, yj = C.frame(ch, seed, j, code.block_size)
        xs.append(xj)
        ls.append(C.channel_llr(ch, yj).astype(np.float32))
    llr = np.array(ls)
    uu = np.array([O.polar_transform_bytes(xj) for xj in xs])
    u_fix, _ = gpu_decode(cuda, code, llr, uu, fmode="fixed")
    u_flt, _ = gpu_decode(cuda, code, llr, uu, fmode="exact")
    ok_fix, ok_flt = np.all(u_fix == uu, axis=1), np.all(u_flt == uu, axis=1)
    # frame-level agreement = the same outcome (verified / discarded) as the
    # float decoder; two failed decodes rarely fail identically bit for bit
    agree = np.mean(ok_fix == ok_flt)
    print(f"fixed FER {1 - ok_fix.mean():.4f} float FER {1 - ok_flt.mean():.4f} agreement {agree:.4f}")
    assert agree >= 0.98
    assert (1 - ok_fix.mean()) <= 2 * (1 - ok_flt.mean()) + 1e-12


@pytest.mark.parametrize("rep", ["float", "fixed"])
def test_run_trials_counts_match_oracle(cuda, rep):
    """trials.run_trials: the GPU's discarded-frame count
    equals the oracle's on the same seeded frames (c1, 96 trials, batch 40 so
    the last batch is ragged)."""
    from paper_1204_5882_b200.trials import run_trials
    if "c1" not in K.available_configs():
        pytest.skip("c1 not built")
    cfg = K.CONFIGS["c1"]
    code = K.load_config("c1")
    T, N, seed = 96, code.block_size, 77
    xs, llrs = [], []
    for j in range(T):
        x, y = C.frame(cfg.channel, seed, j, N)
        xs.append(x)
        llrs.append(C.channel_llr(cfg.channel, y))
    xs, llrs = np.array(xs), np.array(llrs, np.float32)
    u_true = transform_rows(xs)
    if rep == "fixed":
        u = fixed_oracle_batch(code, O.quantize_q88(llrs), u_true)
    else:
        u = np.array([O.sc_decode(code.frozen_mask, llrs[t], u_true[t], precision=32)[0] for t in range(T)])
    expect = int(np.sum(np.any(u != u_true, axis=1)))
    row = run_trials(code, cfg.channel, T, seed, representation=rep, batch=40, device=cuda)
    assert row.trials == T and row.n == code.n
    assert row.fer_measured == expect / T
    assert row.throughput_mbps > 0


# --------------------------------------------------------------------------
# thread-block clusters: K CTAs per frame share the upper band

def cluster_code(n, rng):
    """Left quarter frozen (a wide rate-0 node), next quarter random, right
    half information (a rate-1 node of width N/2 > S): exercises the
    cluster-sliced rate-0 zeroing, the cluster-wide rate-1 minimum and the
    sliced f/g/combine steps."""
    N = 1 << n
    mask = np.zeros(N, np.uint8)
    mask[: N // 4] = 1
    mask[N // 4: N // 2] = (rng.random(N // 4) < 0.5).astype(np.uint8)
    return K.PolarCode(n=n, frozen_mask=mask, channel=C.BiAwgn(1.0), target_fer=0.1)


@pytest.mark.parametrize("ncl", [2, 4, 8])
@pytest.mark.parametrize("fmode", ["exact", "fixed"])
def test_cluster_upper_band_bit_exact(cuda, ncl, fmode):
    from paper_1204_5882_b200 import _lib
    rng = np.random.default_rng(500 + ncl)
    n, F = 15, 3
    N = 1 << n
    for code in (cluster_code(n, rng), random_code(n, 0.4, rng)):
        # strong LLRs on frame 0 (rate-1 guard passes), weak ones elsewhere
        llr = rng.normal(1.0, 2.0, (F, N)).astype(np.float32)
        llr[0] = rng.normal(25.0, 2.0, N).astype(np.float32) * np.where(rng.random(N) < 0.2, -1, 1)
        fz = rng.integers(0, 2, (F, N)).astype(np.uint8)
        if fmode == "fixed":
            ref = fixed_oracle_batch(code, O.quantize_q88(llr), fz)
        else:
            ref, _ = oracle_batch(code, llr, fz, 32)
        dec = ScDecoder(code, max_frames=F, f_mode=fmode, subtree_log2=11)
        dec.set_option(_lib.PQ_OPT_CLUSTER, ncl)
        u, x = dec.decode(to_dev(llr, cuda), words_dev(fz, cuda), want_x=True)
        assert np.array_equal(from_words(u, N), ref)
        assert np.array_equal(from_words(x, N), transform_rows(from_words(u, N)))


def test_cluster_auto_c5_shape_matches_single_cta(cuda):
    """Auto cluster size on a few-frames N = 2^20 batch equals K = 1, bit for bit."""
    from paper_1204_5882_b200 import _lib
    if "c4" not in K.available_configs():
        pytest.skip("c4 not built")
    cfg, code, x, u_true, llr = config_batch("c4", 4)
    outs = []
    for ncl in (0, 1):
        dec = ScDecoder(code, max_frames=4, f_mode="fixed")
        dec.set_option(_lib.PQ_OPT_CLUSTER, ncl)
        u, _ = dec.decode(to_dev(llr, cuda), words_dev(u_true, cuda))
        outs.append(u.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("bsc", [True, False])
def test_pipelined_decoder_matches_direct(cuda, bsc):
    """pipeline.PipelinedDecoder: several host batches in flight on three streams
    give the same u-hat as one direct decode per batch."""
    import torch
    from paper_1204_5882_b200.pipeline import PipelinedDecoder
    if "c1" not in K.available_configs():
        pytest.skip("c1 not built")
    cfg, code, x, u_true, llr = config_batch("c1", 32)
    N = code.block_size
    dec = ScDecoder(code, max_frames=16, f_mode="fixed")
    mag = np.float32(cfg.channel.llr_magnitude) if bsc else None
    pipe = PipelinedDecoder(dec, 16, bsc_llr_mag=mag)
    batches = []
    for b in range(5):  # batches 0..4 over frames [0,16), [16,32), [0,16), ...
        sl = slice(16 * (b % 2), 16 * (b % 2) + 16)
        if bsc:
            y = np.array([C.frame(cfg.channel, cfg.seed, j, N)[1] for j in range(sl.start, sl.stop)])
            h_in = torch.from_numpy(pack_bits(y).view(np.int32).copy()).pin_memory()
        else:
            h_in = torch.from_numpy(np.ascontiguousarray(llr[sl])).pin_memory()
        h_fz = torch.from_numpy(pack_bits(u_true[sl]).view(np.int32).copy()).pin_memory()
        h_out = torch.empty((16, N // 32), dtype=torch.int32).pin_memory()
        pipe.submit(h_in, h_fz, h_out)
        batches.append((sl, h_out))
    pipe.synchronize()
    ref = ScDecoder(code, max_frames=32, f_mode="fixed")
    u_ref, _ = ref.decode(to_dev(llr, cuda), words_dev(u_true, cuda))
    u_ref = from_words(u_ref, N)
    for sl, h_out in batches:
        assert np.array_equal(unpack_bits(h_out.numpy().view(np.uint32), N), u_ref[sl])


def test_q88_input_matches_fp32_input(cuda):
    """pq_sc_decode_q88 (int16 Q8.8 codes) = the fixed decoder on fp32 LLRs that
    quantise to the same codes, on all five paths the channel reaches (root
    f/g steps through the TMA ring at n = 16, S = 2^11; a small block whose root
    is in the warp band)."""
    import torch
    rng = np.random.default_rng(77)
    for n, lg in ((16, 11), (9, 0), (14, 0)):
        code = random_code(n, 0.45, rng)
        N, F = 1 << n, 3
        llr = rng.normal(0.8, 2.5, (F, N)).astype(np.float32)
        fz = rng.integers(0, 2, (F, N)).astype(np.uint8)
        raw = O.quantize_q88(llr)
        ref = fixed_oracle_batch(code, raw, fz)
        dec = ScDecoder(code, max_frames=F, f_mode="fixed", subtree_log2=lg)
        u, _ = dec.decode_q88(torch.from_numpy(raw).to(cuda), words_dev(fz, cuda))
        assert np.array_equal(from_words(u, N), ref)
    with pytest.raises(ValueError):
        ScDecoder(code, max_frames=F, f_mode="exact").decode_q88(torch.from_numpy(raw).to(cuda))


# --------------------------------------------------------------------------
# the widest warp-band levels (warp_wide: W = 1024, 2048 taken by one warp)

def wide_node_code(n, rng):
    """Blocks of 2048 / 1024 leaves that are rate-0, repetition, rate-1 or
    mixed, so every node type reaches the 1024/2048 levels of the warp band."""
    N = 1 << n
    mask = np.zeros(N, np.uint8)
    kinds = ["r0", "rep", "r1", "mix", "r1", "rep", "mix", "r0"]
    for b in range(N // 1024):
        blk = mask[1024 * b: 1024 * (b + 1)]
        kind = kinds[b % len(kinds)]
        if kind == "r0":
            blk[:] = 1
        elif kind == "rep":
            blk[:-1] = 1
        elif kind == "mix":
            blk[:] = (rng.random(1024) < 0.5).astype(np.uint8)
    return K.PolarCode(n=n, frozen_mask=mask, channel=C.BiAwgn(1.0), target_fer=0.1)


@pytest.mark.parametrize("n,log2s", [(13, 0), (14, 11), (13, 12), (11, 0)])
@pytest.mark.parametrize("strength", [1.0, 6.0])
def test_warp_wide_levels_bit_exact(cuda, n, log2s, strength):
    """Rate-1 guards that pass (strong LLRs) and fail (weak ones), repetition
    sums and rate-0 children at widths 1024 / 2048, fp32 mirror and Q8.8."""
    import torch
    rng = np.random.default_rng(900 + n + log2s)
    code = wide_node_code(n, rng)
    F, N = 6, 1 << n
    llr = (rng.normal(strength, 2.0, (F, N))).astype(np.float32)
    fz = rng.integers(0, 2, (F, N)).astype(np.uint8)
    ref, _ = oracle_batch(code, llr, fz, 32)
    u, _ = gpu_decode(cuda, code, llr, fz, subtree_log2=log2s)
    assert np.array_equal(u, ref)
    raw = O.quantize_q88(llr)
    dec = ScDecoder(code, max_frames=F, f_mode="fixed", subtree_log2=log2s)
    u16, _ = dec.decode_q88(torch.from_numpy(raw).to(cuda), words_dev(fz, cuda))
    assert np.array_equal(from_words(u16, N), fixed_oracle_batch(code, raw, fz))
