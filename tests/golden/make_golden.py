"""Generate the golden fixtures in this directory from the REFERENCE itself.

Run only in the build container (imports /root/reference/pkg/src); the GPU
box and the test-suite read the committed .npz files and never the reference.

  channel_vectors.npz  -- make_rng / transmit / channel_llr outputs
                          (channel.py:66-150) for the package's restatement
  boxplus_grid.npz     -- the reference's exact boxplus magnitude
                          _boxplus_magnitude (construction.py:132-135) on a
                          log grid, to pin the oracle's and the GPU's f
  c1_frames.npz        -- config c1 frames 0..15 generated with the
                          reference's own make_rng/transmit/channel_llr
                          (x bits, y bits, fp32 channel LLRs)
  de_small.npz         -- reference density_evolution pe at n=3 (BSC 0.05,
                          0.1) for the SPEC acceptance-6 oracle check
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from polarqkd import channel as RC  # noqa: E402
from polarqkd import construction as RK  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    out = {}
    for seed, stream in ((0, None), (7, 3), (1003, 0), (1003, 1), (2**40 + 5, 17)):
        tag = f"{seed}_{stream}"
        r = RC.make_rng(seed, stream)
        out[f"ints_{tag}"] = r.integers(0, 2, 4096, dtype=np.uint8)
        out[f"unif_{tag}"] = r.random(64)
    bits = RC.make_rng(11, 0).integers(0, 2, 4096, dtype=np.uint8)
    out["bits"] = bits
    for p in (0.0, 0.02, 0.03, 0.1, 0.5):
        y = RC.transmit(RC.Bsc(p), bits, 5, 9)
        out[f"bsc_y_{p}"] = y
        out[f"bsc_llr_{p}"] = RC.channel_llr(RC.Bsc(p), y)
    for snr in (1.0, 0.161, 1e6):
        y = RC.transmit(RC.BiAwgn(snr), bits, 5, 9)
        out[f"awgn_y_{snr}"] = y
        out[f"awgn_llr_{snr}"] = RC.channel_llr(RC.BiAwgn(snr), y)
    np.savez_compressed(os.path.join(HERE, "channel_vectors.npz"), **out)

    g = np.concatenate([np.geomspace(1e-6, 60.0, 120), [0.5, 1.0, 2.0, 5.0, 29.99]])
    A, B = np.meshgrid(g, g, indexing="ij")
    np.savez_compressed(os.path.join(HERE, "boxplus_grid.npz"), a=A.ravel(), b=B.ravel(),
                        f=RK._boxplus_magnitude(A.ravel(), B.ravel()))

    # c1 frames, the bench's seed convention (frame j: bits from stream 2j,
    # noise from stream 2j+1), produced by the reference's functions
    seed, N, ch = 1001, 1024, RC.Bsc(0.02)
    xs, ys, ls = [], [], []
    for j in range(16):
        x = RC.make_rng(seed, 2 * j).integers(0, 2, N, dtype=np.uint8)
        y = RC.transmit(ch, x, seed, stream=2 * j + 1)
        xs.append(x); ys.append(y); ls.append(RC.channel_llr(ch, y).astype(np.float32))
    np.savez_compressed(os.path.join(HERE, "c1_frames.npz"), x=np.array(xs), y=np.array(ys),
                        llr=np.array(ls), seed=seed)

    de = {}
    for p in (0.05, 0.1):
        de[f"pe_{p}"] = RK.density_evolution(RC.Bsc(p), 3).pe
    np.savez_compressed(os.path.join(HERE, "de_small.npz"), **de)
    print("ok")


if __name__ == "__main__":
    main()
