"""bob_decode's verification step.

Hash = XXH64 seed-keyed.  The oracle restatement
(oracle/sc_oracle.c orc_xxh64) is pinned by published XXH64 test vectors;
the product's host (pq_xxh64) and device (pq_hash_frames / pq_verify_frames)
implementations must match it on every length class (stripes + 8/4/1-byte
tails, blocks shorter than one stripe); the batched device protocol must
agree frame by frame with the decoder's own outcome (u_hat == u) and with the
host bob_decode."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1204_5882_b200 import channel as C
from paper_1204_5882_b200 import codes as K
from paper_1204_5882_b200 import reconcile as R
from paper_1204_5882_b200.polar_core import block_hash_host, pack_bits, unpack_bits

# published XXH64 test vectors (xxHash project documentation / python-xxhash README)
KATS = [(b"", 0, 0xEF46DB3751D8E999), (b"a", 0, 0xD24EC4F1A98C6E5B), (b"abc", 0, 0x44BC2CF5AD770999),
        (b"Nobody inspects the spammish repetition", 0, 0xFBCEA83C8A378BF1)]


@pytest.mark.parametrize("data,seed,want", KATS)
def test_oracle_xxh64_known_answers(data, seed, want):
    assert O.xxh64(data, seed) == want


def test_host_xxh64_matches_oracle():
    rng = np.random.default_rng(7)
    for L in list(range(0, 70)) + [127, 128, 129, 1000, 4096 + 13]:
        data = rng.integers(0, 256, L, dtype=np.uint8).tobytes()
        seed = int(rng.integers(0, 2 ** 63)) * 2 + 1
        from paper_1204_5882_b200 import _lib
        assert int(_lib.load().pq_xxh64(data, len(data), seed)) == O.xxh64(data, seed), L


def test_block_hash_is_keyed_xxh64_of_packed_words():
    rng = np.random.default_rng(3)
    for n in (1, 3, 5, 6, 10):
        x = rng.integers(0, 2, 1 << n, dtype=np.uint8)
        for key in (0, 12345, 2 ** 64 - 1):
            h = R.block_hash(x, key)
            assert h == O.block_hash_words(pack_bits(x), key)
            assert h == block_hash_host(pack_bits(x), key)
        assert R.block_hash(x, 1) != R.block_hash(x, 2)


# ---------------------------------------------------------------- GPU
def _dev(a, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 3, 5, 6, 8, 10, 13, 16])
def test_device_hash_matches_oracle(cuda, n):
    from paper_1204_5882_b200.polar_core import hash_frames
    rng = np.random.default_rng(n)
    F = 37
    x = rng.integers(0, 2, (F, 1 << n), dtype=np.uint8)
    words = pack_bits(x)
    key = 0x1234_5678_9ABC_DEF1
    got = hash_frames(_dev(words.view(np.int32), cuda), n, key).cpu().numpy().view(np.uint64)
    want = [O.block_hash_words(words[f], key) for f in range(F)]
    assert [int(v) for v in got] == want


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["c1", "c2"])
def test_batched_disclose_decode_verify(cuda, key):
    import torch
    from paper_1204_5882_b200.polar_core import ScDecoder
    cfg = K.CONFIGS[key]
    if key not in K.available_configs():
        pytest.skip(f"{key} code table missing")
    code = K.load_config(key)
    N, F = code.block_size, (64 if key == "c1" else 24)
    frames = [C.frame(cfg.channel, cfg.seed, j, N) for j in range(F)]
    x = np.array([a for a, _ in frames])
    y = np.array([b for _, b in frames])
    llr = np.array([C.channel_llr(cfg.channel, yi) for yi in y]).astype(np.float32)
    session = 99
    xw = _dev(pack_bits(x).view(np.int32), cuda)
    frozen_u, hashes = R.alice_disclose_batch(code, xw, session)
    # Alice's hashes are the host hashes of x; her frozen words are u & mask
    assert [int(h) for h in hashes.cpu().numpy().view(np.uint64)] == [R.block_hash(xi, session) for xi in x]
    dec = ScDecoder(code, max_frames=F, f_mode="fixed")
    nd = torch.zeros(1, dtype=torch.int32, device=cuda)
    ver, x_hat = R.bob_decode_batch(dec, frozen_u, hashes, session, llr=_dev(llr, cuda), n_discarded=nd)
    ver = ver.cpu().numpy().astype(bool)
    xh = unpack_bits(x_hat.cpu().numpy().view(np.uint32), N)
    ok = np.all(xh == x, axis=1)
    assert np.array_equal(ver, ok)          # verdict = exact recovery (no hash collisions here)
    assert int(nd.item()) == int((~ok).sum())
    # the host bob_decode (SPEC signature) reaches the same verdict on a few frames
    for f in range(0, F, max(1, F // 4)):
        fv, h = R.alice_disclose(code, x[f], session)
        out, _ = R.bob_decode(code, y[f], cfg.channel, fv, h, session)
        assert (out == R.VERIFIED) == ok[f]
    # a flipped revealed value on a noiseless channel is discarded
    clean = np.where(x[:4] == 0, 30.0, -30.0).astype(np.float32)
    fu = frozen_u[:4].clone()
    fi = code.frozen_indices()
    if len(fi):
        i = int(fi[len(fi) // 2])
        fu[1, i >> 5] ^= (1 << (i & 31)) if (i & 31) < 31 else -(1 << 31)
    nd.zero_()
    ver, _ = R.bob_decode_batch(dec, fu, hashes[:4], session, llr=_dev(clean, cuda), n_discarded=nd)
    ver = ver.cpu().numpy().astype(bool)
    assert ver[0] and ver[2] and ver[3]
    if len(fi):
        assert not ver[1] and int(nd.item()) == 1
