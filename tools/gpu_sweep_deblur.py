import sys
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import oracle as O
from paper_1203_4874_b200 import api
cases = [(70, 50, 3, 1), (50, 142, 3, 1), (118, 60, 3, 1), (60, 1942, 3, 1), (1118, 60, 3, 1),
         (300, 300, 3, 1), (600, 60, 3, 1), (1090 - 2, 60, 3, 1), (60, 1930 - 2, 3, 1), (100, 100, 3, 3),
         (1078, 1918, 3, 1)]
for (r, c, t, ch) in cases:
    lat = O.random_frame(r, c, ch, 5)
    pair = O.generate_coprime_pair(t, 7)
    pub, _ = O.encode_frame(lat, pair.k1, pair.k2)
    pub32 = pub.astype(np.float32)
    ref = np.stack([O.spectral_deblur(pub32[k].astype(np.float64), pair.k1, 1e-8) for k in range(ch)])
    got = api.spectral_deblur(torch.from_numpy(pub32).cuda(), pair.k1, 1e-8).cpu().numpy()
    Gr, Gc = O.friendly_size(r + t - 1), O.friendly_size(c + t - 1)
    print(f"{r}x{c} ch={ch} grid {Gr}x{Gc} err={np.abs(got - ref).max():.3e}", flush=True)
