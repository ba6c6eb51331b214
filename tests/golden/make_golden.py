"""Generates the golden fixtures in tests/golden/ from the FP64 oracle, after checking
each against the independent numpy/LAPACK restatement (oracle/np_ref.py).
Inputs are regenerated from the stored seeds with the reference-exact generators
(random_frame, generate_coprime_pair, encode_frame), rounded to FP32 like the device
inputs. Run: python tests/golden/make_golden.py"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import np_ref as N  # noqa: E402
from oracle import oracle as O  # noqa: E402

CASES = [
    # name, rows, cols, channels, t, latent stream seed, pair seed, search_min, search_max
    ("c1_256x256_t7", 256, 256, 1, 7, O.frame_seed(1, 0), O.frame_seed(2, 0), 3, 25),
    ("rt_64x64_t5", 64, 64, 1, 5, 137, 137, 3, 9),
    ("rgb_40x48_t3", 40, 48, 3, 3, 147, 147, 3, 7),
    ("odd_61x97_t9", 61, 97, 1, 9, 999, 998, 3, 25),
]


def inputs(rows, cols, ch, t, lseed, pseed):
    lat = O.random_frame(rows, cols, ch, lseed)
    pair = O.generate_coprime_pair(t, pseed)
    pub, prv = O.encode_frame(lat, pair.k1, pair.k2)
    return lat, pair, pub.astype(np.float32), prv.astype(np.float32)


def main():
    for name, rows, cols, ch, t, ls, ps, lo, hi in CASES:
        lat, pair, pub, prv = inputs(rows, cols, ch, t, ls, ps)
        d = O.decode_frame(pub.astype(np.float64), prv.astype(np.float64), cfg=O.make_cfg(lo, hi))
        ln, kn, tn = N.decode_frame(pub.astype(np.float64), prv.astype(np.float64), lo, hi)
        assert d.width_used == tn == t
        assert np.linalg.norm(d.kernel - kn) / np.linalg.norm(kn) <= 1e-9
        assert np.abs(d.latent - ln).max() <= 1e-7
        np.savez_compressed(os.path.join(HERE, name + ".npz"), rows=rows, cols=cols, channels=ch, t=t,
                            latent_seed=np.uint64(ls), pair_seed=np.uint64(ps), search_min=lo, search_max=hi,
                            kernel=d.kernel, latent=d.latent.astype(np.float32),
                            validation_residual=d.validation_residual, k1=pair.k1, k2=pair.k2,
                            pub_checksum=np.float64(pub.astype(np.float64).sum()))
        print(name, "ok")


if __name__ == "__main__":
    main()
