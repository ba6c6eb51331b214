"""Ad-hoc GPU check: spectral_deblur vs the FP64 oracle (test infrastructure)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import oracle as O
from paper_1203_4874_b200 import api

for (r, c, t, ch) in [(16, 16, 3, 1), (24, 24, 3, 1), (64, 64, 5, 1), (61, 97, 7, 1), (480, 640, 9, 1), (1080, 1920, 11, 3)]:
    lat = O.random_frame(r, c, ch, O.frame_seed(1, r))
    pair = O.generate_coprime_pair(t, O.frame_seed(2, r))
    pub, prv = O.encode_frame(lat, pair.k1, pair.k2)
    pub32 = pub.astype(np.float32)
    t0 = time.time()
    ref = np.stack([O.spectral_deblur(pub32[k].astype(np.float64), pair.k1, 1e-8) for k in range(ch)])
    tcpu = time.time() - t0
    got = api.spectral_deblur(torch.from_numpy(pub32).cuda(), pair.k1, 1e-8)
    torch.cuda.synchronize()
    g = got.cpu().numpy().astype(np.float64)
    err = np.abs(g - ref).max()
    psnr_gt = O.psnr(lat, g) if True else 0
    print(f"{r}x{c} t={t} ch={ch}: max|gpu-oracle|={err:.3e} psnr(gpu,oracle)={O.psnr(ref, g):.1f} psnr(gpu,truth)={psnr_gt:.1f} cpu {tcpu:.3f}s", flush=True)
