"""The committed golden fixtures (tests/golden/*.npz, made by make_golden.py) still match
the oracle on regenerated inputs (CPU)."""
import glob
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURES = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))


def load_case(oracle, path):
    g = np.load(path)
    rows, cols, ch, t = int(g["rows"]), int(g["cols"]), int(g["channels"]), int(g["t"])
    lat = oracle.random_frame(rows, cols, ch, int(g["latent_seed"]))
    pair = oracle.generate_coprime_pair(t, int(g["pair_seed"]))
    pub, prv = oracle.encode_frame(lat, pair.k1, pair.k2)
    return g, lat, pair, pub.astype(np.float32), prv.astype(np.float32)


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p) for p in FIXTURES])
def test_fixture_matches_oracle(oracle, path):
    g, lat, pair, pub, prv = load_case(oracle, path)
    assert np.array_equal(pair.k1, g["k1"]) and np.array_equal(pair.k2, g["k2"])
    assert pub.astype(np.float64).sum() == float(g["pub_checksum"])
    d = oracle.decode_frame(pub.astype(np.float64), prv.astype(np.float64),
                            cfg=oracle.make_cfg(int(g["search_min"]), int(g["search_max"])))
    assert d.width_used == int(g["t"])
    assert np.abs(d.kernel - g["kernel"]).max() <= 1e-12
    assert np.abs(d.latent.astype(np.float32) - g["latent"]).max() <= 1e-6
    assert oracle.psnr(lat, d.latent) >= 40.0
