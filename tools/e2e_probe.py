"""e2e A/B aid: the bench's host-buffer run (cbp_decode_run_host over 3 epochs of 1080p RGB,
pinned host memory, recovery frame every 30) timed alone, plus the PCIe link calibration
(tools/pcie_probe.py). Prints one JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1203_4874_b200 import api

ROWS, COLS, CH, T, EPOCH, NE = 1080, 1920, 3, 11, 30, 3
Mb, Nb = ROWS + T - 1, COLS + T - 1
hpub = torch.empty((EPOCH * NE, CH, Mb, Nb), dtype=torch.float32).pin_memory()
hprv = torch.zeros_like(hpub).pin_memory()
rec = np.zeros(EPOCH * NE, np.int32)
for e in range(NE):
    pair = api.generate_coprime_pair(T, api.frame_seed(2, e))
    lat = api.synth_frames(EPOCH * CH, ROWS, COLS, seed=api.frame_seed(1, e)).view(EPOCH, CH, ROWS, COLS)
    p, q = api.encode_frame(lat, pair.k1, pair.k2)
    hpub[EPOCH * e:EPOCH * (e + 1)].copy_(p.cpu())
    hprv[EPOCH * e].copy_(q[0].cpu())
    rec[EPOCH * e] = 1
if os.environ.get("E2E_ONE_RECOVERY"):  # A/B: only the run's first frame recovers (no recovery stalls)
    rec[EPOCH:] = 0
hout = torch.empty_like(hpub).pin_memory()
cfg = api.make_cfg(9, 25, 1e-6, validate=True)
api.decode_run_host(hpub[:EPOCH], hprv[:EPOCH], rec[:EPOCH], cfg, out=hout[:EPOCH])
res = []
for _ in range(3):
    t0 = time.perf_counter()
    api.decode_run_host(hpub, hprv, rec, cfg, out=hout)
    res.append(EPOCH * NE / (time.perf_counter() - t0))
print(json.dumps({"e2e_fps": res, "env": {k: v for k, v in os.environ.items() if k.startswith("CBP_")}}))
