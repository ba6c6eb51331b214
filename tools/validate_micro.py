"""Validation-residual cost: decode_frames_async with validate on/off (1080p RGB frame, 4K
batch of 4), for A/B between library builds (CBP_CUDA_LIB). Profiling aid."""
# time decode_frames_async (validation on vs off) for one 1080p RGB frame and a 4-frame 4K batch
import sys, os, json
sys.path.insert(0, "."); sys.path.insert(0, "tools")
import torch
from paper_1203_4874_b200 import api
import bench_configs as bc
out = {"lib": os.environ.get("CBP_CUDA_LIB", "default")}
for (rows, cols, t, ch, B) in [(1080, 1920, 11, 3, 1), (2160, 3840, 15, 1, 4)]:
    pub, prv = bc.make_pairs(B, ch, rows, cols, t, 7, shared_kernel=False)
    o = torch.empty_like(pub)
    slots = torch.zeros((B, api.SLOT_BYTES), dtype=torch.uint8, device="cuda")
    for val in (True, False):
        cfg = api.make_cfg(9, 25, trust_hint=True, validate=val)
        ms = bc.timed(lambda: api.decode_frames_async(pub, prv, cfg, o, slots, hints=[t] * B), 10)
        out[f"{rows}p_val{int(val)}_ms"] = round(ms, 4)
    sl = api.read_slots(slots, B)
    out[f"{rows}p_resid"] = [s.residual for s in sl][:2]
print(json.dumps(out))
