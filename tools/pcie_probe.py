"""Host link calibration for the e2e number: pinned H2D alone, D2H alone, and both at once
on two streams (GB/s). Reference point only."""
import json, torch
n = 256 << 20  # floats (1 GiB)
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, dtype=torch.float32, device="cuda")
d_out = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); torch.cuda.synchronize(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1000
for _ in range(2):
    d_in.copy_(h_in, non_blocking=True); h_out.copy_(d_out, non_blocking=True)
gb = n * 4 / 1e9
t_h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
t_both = timed(both)
print(json.dumps({"h2d_GBs": gb / t_h2d, "d2h_GBs": gb / t_d2h, "bidir_each_GBs": gb / t_both}))
