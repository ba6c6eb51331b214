"""Kernel-internal phase timings of the recovery kernels (needs a library built with
-DCBP_PHASES, passed via CBP_CUDA_LIB). Profiling aid."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1203_4874_b200 import api, _native
R, Cc, CH, T = (int(x) for x in os.environ.get("PROBE", "1080,1920,3,11").split(","))
pair = api.generate_coprime_pair(T, api.frame_seed(2, 0))
lat = api.synth_frames(CH, R, Cc, seed=1).view(1, CH, R, Cc)
pub, prv = api.encode_frame(lat, pair.k1, pair.k2)
out = torch.empty_like(pub)
slots = torch.zeros(api.SLOT_BYTES, dtype=torch.uint8, device="cuda")
cfg = api.make_cfg(3 if T < 9 else 9, 25, 1e-6, validate=True)
for it in range(3):
    api.decode_frames_async(pub, prv, cfg, out, slots)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 64)()
_native.lib().cbp_debug_phases(buf)
ph = list(buf)
def d(a, b):
    return (ph[b] - ph[a]) / 1000.0 if ph[a] and ph[b] else None
print(json.dumps({
    "width_blocks_us": {"fill": d(0, 1), "eig": d(1, 2)},
    "solve_us": {"corr+gram": d(10, 11), "eig": d(11, 12), "refine": d(12, 13), "gap": d(13, 14)},
    "compose_us": {"complete": d(20, 21), "resolve_chol": d(21, 25), "resolve_invit": d(25, 22),
                   "resolve_refine": d(22, 23), "assemble": d(23, 24)},
    "compose_detail_us": {"refine_loop": d(22, 26), "after_refine": d(26, 23),
                           "div0": d(40, 41), "ifft0": d(41, 42), "realize0": d(42, 43),
                           "div1": d(44, 45), "ifft1": d(45, 46), "realize1": d(46, 47)},
    "eig_last_us": {"tridiag": d(30, 31), "ql": d(31, 32), "back": d(32, 33)}}))
