"""Quick c4 timing (4K gray, t=15, per-frame recovery): trusted hint and estimated width at
batches 4 and 16 (A/B driver for recovery-path changes)."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench_configs as bc

for B in (4, 16):
    for trust in (True, False):
        r = bc.c4(trust, B)
        print(json.dumps({k: r[k] for k in ("config", "batch", "frames_per_s", "ms_per_batch", "frames_recovered")}))
