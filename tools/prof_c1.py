"""Profiling driver: config c1 (256x256 gray, t=7, search 3..25), decode_frame repeated
(for an ncu launch list of the latency chain)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from paper_1203_4874_b200 import api
import bench_configs as bc
pub, prv = bc.make_pairs(1, 1, 256, 256, 7, 1)
out = torch.empty_like(pub)
slots = torch.zeros((1, api.SLOT_BYTES), dtype=torch.uint8, device="cuda")
cfg = api.make_cfg(3, 25)
for _ in range(3):
    api.decode_frames_async(pub, prv, cfg, out, slots[0])
torch.cuda.synchronize()
print([(s.status, s.width) for s in api.read_slots(slots, 1)])
