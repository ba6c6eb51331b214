"""Profiling driver: config c4 (4K gray, t=15, per-frame recovery, estimated width), a batch
of B frames (PROF_C4_BATCH, default 4) decoded twice (for an ncu launch list)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from paper_1203_4874_b200 import api
import bench_configs as bc
B = int(os.environ.get("PROF_C4_BATCH", "4"))
pub, prv = bc.make_pairs(B, 1, 2160, 3840, 15, 7, shared_kernel=False)
out = torch.empty_like(pub)
slots = torch.zeros((B, api.SLOT_BYTES), dtype=torch.uint8, device="cuda")
for _ in range(2):
    api.decode_frames_async(pub, prv, api.make_cfg(9, 25), out, slots)
torch.cuda.synchronize()
print([(s.status, s.width) for s in api.read_slots(slots, B)])
