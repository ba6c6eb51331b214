"""Small decode + deblur + split-decode workloads on every compile-time plan geometry
(256x256, 640x480, 1080p RGB; 4K with SAN_4K=1): a quick all-plans run that checks the
slots (compute-sanitizer is not available on the GPU pool). Prints ok per geometry."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from paper_1203_4874_b200 import api
import bench_configs as bc

geoms = [(256, 256, 1, 7), (480, 640, 1, 9), (1080, 1920, 3, 11)]
if os.environ.get("SAN_4K"):
    geoms.append((2160, 3840, 1, 15))
for rows, cols, ch, t in geoms:
    pub, prv = bc.make_pairs(2, ch, rows, cols, t, 3)
    out = torch.empty_like(pub)
    slots = torch.zeros((1, api.SLOT_BYTES), dtype=torch.uint8, device="cuda")
    cfg = api.make_cfg(3 if t < 9 else 9, 25)
    api.decode_frames_async(pub[0:1], prv[0:1], cfg, out[0:1], slots[0])
    api.spectral_deblur_slot(pub[1:], slots[0].data_ptr(), out[1:])
    api.recover_kernels_async(pub[0:1], prv[0:1], cfg, slots[0])
    api.validate_frames_async(pub[0:1], out[0:1], slots[0])
    torch.cuda.synchronize()
    sl = api.read_slots(slots, 1)[0]
    assert sl.status == 0 and sl.width == t, (rows, sl.status, sl.width)
    print("ok", rows, cols, ch, t, flush=True)
