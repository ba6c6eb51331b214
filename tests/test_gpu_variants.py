"""Opt-in deconvolution schedules (environment switches read once per process, so each runs
in a subprocess): the fused persistent A+B+C kernel (CBP_FUSED=1) and launch groups on side
streams (CBP_DEBLUR_STREAMS=3, CBP_GROUP_MB=28). Measured slower than the default three
whole-batch launches and kept as alternatives; they must give the same
latents: bit-identical to the default schedule (same tiles, same arithmetic) and within the
parity bar of the FP64 oracle."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from oracle import oracle as O
from paper_1203_4874_b200 import api
torch.cuda.set_device(0)
t = 11
pair = O.generate_coprime_pair(t, O.frame_seed(2, 7))
lat = api.synth_frames(4 * 3, 1080, 1920, seed=O.frame_seed(1, 7)).view(4, 3, 1080, 1920)
pub, _ = api.encode_frame(lat, pair.k1, pair.k2)
Mb, Nb = pub.shape[-2:]
ldp = (Nb + 3) // 4 * 4
x = torch.zeros((4, 3, Mb, ldp), dtype=torch.float32, device="cuda")[..., :Nb]
x.copy_(pub)
out = torch.full((4, 3, Mb, ldp), float("nan"), dtype=torch.float32, device="cuda")[..., :Nb]
api.spectral_deblur(x, pair.k1, 1e-8, out=out)
torch.cuda.synchronize()
got = out[..., :1080, :1920].cpu().numpy()
np.save(sys.argv[1], got)
ref = O.spectral_deblur(pub[3, 2].cpu().numpy().astype(np.float64), pair.k1, 1e-8)
err = float(np.abs(got[3, 2].astype(np.float64) - ref).max())
assert np.isfinite(got).all() and err <= 1e-4, err
print("ok", err)
"""


def _run(tmp_path, name, env):
    path = str(tmp_path / f"{name}.npy")
    script = tmp_path / f"{name}.py"
    script.write_text(SCRIPT.format(root=ROOT))
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, str(script), path], capture_output=True, text=True, timeout=600, env=e)
    assert r.returncode == 0, r.stdout + r.stderr
    import numpy as np
    return np.load(path)


def test_deblur_schedules_agree(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    base = _run(tmp_path, "default", {})
    fused = _run(tmp_path, "fused", {"CBP_FUSED": "1"})
    side = _run(tmp_path, "side", {"CBP_DEBLUR_STREAMS": "3", "CBP_GROUP_MB": "28"})
    assert (base == fused).all()
    assert (base == side).all()
