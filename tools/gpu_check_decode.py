"""Ad-hoc GPU check: decode_frame and stage entries vs the FP64 oracle."""
import sys, time, traceback
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import oracle as O
from paper_1203_4874_b200 import api

def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))

def run(r, c, t, ch, smin, smax, hint, seed=137):
    lat = O.random_frame(r, c, ch, O.frame_seed(1, seed))
    pair = O.generate_coprime_pair(t, O.frame_seed(2, seed))
    pub, prv = O.encode_frame(lat, pair.k1, pair.k2)
    pub32 = pub.astype(np.float32); prv32 = prv.astype(np.float32)
    cfgo = O.make_cfg(smin, smax, trust_hint=hint)
    t0 = time.time()
    ref = O.decode_frame(pub32.astype(np.float64), prv32.astype(np.float64), hint=t, cfg=cfgo)
    tc = time.time() - t0
    cfg = api.make_cfg(smin, smax, trust_hint=hint)
    d = api.decode_frame(torch.from_numpy(pub32).cuda(), torch.from_numpy(prv32).cuda(), hint=t, cfg=cfg)
    torch.cuda.synchronize()
    lg = d.latent.cpu().numpy().astype(np.float64)
    print(f"{r}x{c} t={t} ch={ch} hint={hint}: width gpu={d.width_used} ref={ref.width_used} "
          f"kernel rel={rel(d.kernel_estimate, ref.kernel):.2e} vs-true={rel(d.kernel_estimate, pair.k1):.2e} "
          f"latent maxabs={np.abs(lg - ref.latent).max():.2e} psnr(gpu,ref)={O.psnr(ref.latent, lg):.1f} "
          f"psnr(gpu,truth)={O.psnr(lat, lg):.1f} resid gpu={d.validation_residual:.3e} ref={ref.validation_residual:.3e} "
          f"eps={d.epsilon_used:.3e}/{ref.epsilon_used:.3e} ms={[round(x,3) for x in vars(d.stage_timings).values()]} cpu={tc:.2f}s",
          flush=True)

for args in [(64, 64, 5, 1, 3, 9, False), (64, 64, 5, 1, 3, 9, True), (256, 256, 7, 1, 3, 25, False),
             (24, 24, 3, 3, 3, 7, False), (480, 640, 9, 1, 9, 25, False), (1080, 1920, 11, 3, 9, 25, False),
             (1080, 1920, 11, 3, 9, 25, True), (2160, 3840, 15, 1, 9, 25, True)]:
    try:
        run(*args)
    except Exception as e:
        traceback.print_exc()

# stage KATs
k1, k2, g = api.cofactor_null_solve([1, 3, 2], [3, 4, 1], 2)
print("cofactor KAT", k1, k2, g)
try:
    api.cofactor_null_solve([1, 2, 1], [1, 2, 1], 2)
    print("cofactor degenerate: NOT flagged")
except api.CbpError as e:
    print("cofactor degenerate flagged:", e.code, e)
lat = O.random_mat(12, 12, 5)
try:
    api.decode_frame(np.zeros((12, 12)), np.zeros((12, 12)), hint=3, cfg=api.make_cfg(3, 7, trust_hint=True))
except api.CbpError as e:
    print("zero scene:", e.code, e)
