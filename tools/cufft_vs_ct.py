"""Vendor bar for the deconvolution (reference point, not the product path): the same 1080p RGB
Wiener deconvolution of 29 frames (87 planes, pitched rows as in bench.py) through planned
cuFFT R2C/C2R with callbacks (zero-padding load, filter-multiply store, crop store;
tools/cufft/cufft_baseline.cu, built by tools/cufft/build.sh) against cbp_spectral_deblur.
Prints one JSON line: us per plane of each and the max-abs difference of their latents."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_1203_4874_b200 import api  # noqa: E402

lib = C.CDLL(os.environ.get("CUFFT_BASELINE_LIB", os.path.join(HERE, "cufft", "libcufft_baseline.so")))
F, ROWS, COLS, T = int(os.environ.get("FRAMES", "29")), 1080, 1920, 11
pair = api.generate_coprime_pair(T, api.frame_seed(2, 0))
lat = api.synth_frames(F * 3, ROWS, COLS, seed=1).view(F, 3, ROWS, COLS)
p, _ = api.encode_frame(lat, pair.k1, pair.k2)
Mb, Nb = p.shape[-2:]
ld = (Nb + 3) // 4 * 4
pub = torch.zeros((F, 3, Mb, ld), dtype=torch.float32, device="cuda")[..., :Nb]
pub.copy_(p)
out_ct = torch.zeros((F, 3, Mb, ld), dtype=torch.float32, device="cuda")[..., :Nb]
out_cf = torch.zeros((F, 3, Mb, ld), dtype=torch.float32, device="cuda")[..., :Nb]  # pitched like out_ct
eps = 1e-8 * float(np.sum(pair.k1)) ** 2  # decoder.cpp:198-199 (nonnegative kernel: peak |K| = sum)
Gr, Gc = api.friendly_size(Mb), api.friendly_size(Nb)
kp = np.zeros((Gr, Gc))
kp[:T, :T] = pair.k1
K = np.fft.rfft2(kp)
H = (np.conj(K) / (np.abs(K) ** 2 + eps) / (Gr * Gc)).astype(np.complex64)
Hd = torch.from_numpy(H).cuda()

reps = 10
for _ in range(2):
    api.spectral_deblur(pub, pair.k1, eps, out=out_ct)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    api.spectral_deblur(pub, pair.k1, eps, out=out_ct)
e1.record()
torch.cuda.synchronize()
us_ct = e0.elapsed_time(e1) / reps * 1000 / (3 * F)

ms = C.c_float(0)
M, N = ROWS, COLS
rc = lib.cufft_deblur(C.c_void_p(pub.data_ptr()), C.c_longlong(Mb * ld), ld, Mb, Nb, C.c_void_p(Hd.data_ptr()), Gr, Gc,
                      C.c_void_p(out_cf.data_ptr()), C.c_longlong(Mb * ld), ld, M, N, 3 * F, reps, C.byref(ms))
torch.cuda.synchronize()
if rc:
    raise SystemExit(f"cufft_deblur failed: {rc}")
us_cf = ms.value * 1000 / (3 * F)
out_pl = torch.zeros((F, 3, Mb, ld), dtype=torch.float32, device="cuda")[..., :Nb]
rc = lib.cufft_deblur_plain(C.c_void_p(pub.data_ptr()), C.c_longlong(Mb * ld), ld, Mb, Nb, C.c_void_p(Hd.data_ptr()),
                            Gr, Gc, C.c_void_p(out_pl.data_ptr()), C.c_longlong(Mb * ld), ld, M, N, 3 * F, reps,
                            C.byref(ms))
torch.cuda.synchronize()
if rc:
    raise SystemExit(f"cufft_deblur_plain failed: {rc}")
us_pl = ms.value * 1000 / (3 * F)
diff = float((out_ct[..., :M, :N] - out_cf[..., :M, :N]).abs().max())
# FP64 numpy restatement of plane 0 (decoder.cpp:204-214): both must match it
x = np.zeros((Gr, Gc))
x[:Mb, :Nb] = pub[0, 0].cpu().numpy()
ref = np.fft.irfft2(np.fft.rfft2(x) * np.conj(K) / (np.abs(K) ** 2 + eps), s=(Gr, Gc))[:M, :N]
err_ct = float(np.abs(out_ct[0, 0, :M, :N].cpu().numpy() - ref).max())
err_cf = float(np.abs(out_cf[0, 0, :M, :N].cpu().numpy() - ref).max())
err_pl = float(np.abs(out_pl[0, 0, :M, :N].cpu().numpy() - ref).max())
print(json.dumps({"grid": [Gr, Gc], "planes": 3 * F, "cbp_us_per_plane": us_ct,
                  "cufft_callbacks_us_per_plane": us_cf, "cufft_plain_us_per_plane": us_pl,
                  "max_abs_diff_latents": diff, "plane0_max_abs_vs_fp64": {"cbp": err_ct, "cufft_callbacks": err_cf, "cufft_plain": err_pl},
                  "note": "cuFFT 11 planned R2C (load callback: zero padding; store callback: filter multiply) + "
                          "C2R (store callback: crop), batch of all planes; filter table precomputed (not timed) "
                          "for both: the cbp timing includes its own Wiener table kernels"}))
