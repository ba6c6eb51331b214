"""Deconvolution micro-benchmark (1080p RGB, fixed kernel slot): per-pass device time per
plane and frames/s of spectral_deblur_slot, for A/B experiments between library builds
(CBP_CUDA_LIB) and kernel variants (CBP_FFT_VARIANT). Prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1203_4874_b200 import api

frames = int(os.environ.get("MICRO_FRAMES", "29"))
pitch = int(os.environ.get("MICRO_PITCH", "0"))
rows, cols, t = (int(x) for x in os.environ.get("MICRO_GEOM", "1080,1920,11").split(","))
pair = api.generate_coprime_pair(t, api.frame_seed(2, 0))
CH = int(os.environ.get("MICRO_CH", "3"))
lat = api.synth_frames(CH, rows, cols, seed=1).view(1, CH, rows, cols)
pub1, prv1 = api.encode_frame(lat, pair.k1, pair.k2)
Mb, Nb = pub1.shape[-2:]
pitch = pitch or (Nb + 3) // 4 * 4
slots = torch.zeros(api.SLOT_BYTES, dtype=torch.uint8, device="cuda")
out1 = torch.empty_like(pub1)
api.decode_frames_async(pub1, prv1, api.make_cfg(), out1, slots)
# distinct frames > L2: reuse pub1 content is fine for timing, but keep the footprint large
store = torch.empty((frames, CH, Mb, pitch), dtype=torch.float32, device="cuda")
store[..., :Nb] = pub1
pub = store[..., :Nb]
out = torch.empty((frames, CH, Mb, pitch), dtype=torch.float32, device="cuda")[..., :Nb]
for _ in range(3):
    api.spectral_deblur_slot(pub, slots.data_ptr(), out)
torch.cuda.synchronize()
api.profile(True)
iters = 10
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(iters):
    api.spectral_deblur_slot(pub, slots.data_ptr(), out)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / iters
pass_ms, planes, groups = api.profile_read()
api.profile(False)
print(json.dumps({"lib": os.environ.get("CBP_CUDA_LIB", "default"), "variant": os.environ.get("CBP_FFT_VARIANT", "0"),
                  "pitch": pitch, "geom": [rows, cols, t], "us_per_plane": ms * 1000 / (CH * frames),
                  "fps": frames / ms * 1000,
                  "pass_us_per_plane": [round(x * 1000 / max(planes, 1), 3) for x in pass_ms]}))
