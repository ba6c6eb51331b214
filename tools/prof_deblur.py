"""Profiling driver: 1080p RGB spectral_deblur of PROF_FRAMES frames (default 29 = the 87
planes of one bench.py deconvolution launch, pitched rows as in bench.py) for ncu."""
import os
import sys
sys.path.insert(0, ".")
import torch
from paper_1203_4874_b200 import api
pair = api.generate_coprime_pair(11, api.frame_seed(2, 0))
F = int(os.environ.get("PROF_FRAMES", "29"))
lat = api.synth_frames(F * 3, 1080, 1920, seed=1).view(F, 3, 1080, 1920)
p, q = api.encode_frame(lat, pair.k1, pair.k2)
Mb, Nb = p.shape[-2:]
pub = torch.empty((F, 3, Mb, (Nb + 3) // 4 * 4), dtype=torch.float32, device="cuda")[..., :Nb]
pub.copy_(p)
out = torch.empty_like(pub)
for it in range(4):
    api.spectral_deblur(pub, pair.k1, 1e-8, out=out)
torch.cuda.synchronize()
print("ok")
