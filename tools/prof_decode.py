"""Profiling driver: decode_frame (kernel recovery + deconvolution + validation) of one
1080p RGB frame, repeated (for ncu)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_1203_4874_b200 import api
pair = api.generate_coprime_pair(11, api.frame_seed(2, 0))
lat = api.synth_frames(3, 1080, 1920, seed=1).view(1, 3, 1080, 1920)
pub, prv = api.encode_frame(lat, pair.k1, pair.k2)
out = torch.empty_like(pub)
slots = torch.zeros(api.SLOT_BYTES, dtype=torch.uint8, device="cuda")
cfg = api.make_cfg(9, 25, 1e-6, validate=True)
for it in range(3):
    api.decode_frames_async(pub, prv, cfg, out, slots)
torch.cuda.synchronize()
print("ok", api.read_slots(slots, 1)[0].status)
