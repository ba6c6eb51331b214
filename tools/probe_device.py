"""Device probe: properties plus L2-resident vs HBM copy bandwidth (design input)."""
import json, torch
p = torch.cuda.get_device_properties(0)
out = {"name": p.name, "sms": p.multi_processor_count, "l2_bytes": getattr(p, "L2_cache_size", None),
       "total_mem": p.total_memory}
def bw(nbytes, iters=50):
    a = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda").uniform_()
    b = torch.empty_like(a)
    for _ in range(5): b.copy_(a)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): b.copy_(a)
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) / iters * 1e-3
    return 2 * nbytes / t / 1e9
for mb in [4, 8, 16, 32, 48, 64, 96, 256, 1024]:
    out[f"copy_GBps_{mb}MB"] = round(bw(mb << 20), 1)
x = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
for _ in range(3): y = x @ x
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): y = x @ x
e.record(); torch.cuda.synchronize()
out["dgemm_tflops"] = round(2 * 4096**3 * 10 / (s.elapsed_time(e) * 1e-3) / 1e12, 2)
print(json.dumps(out))
open("gpurun_out/probe_device.json", "w").write(json.dumps(out, indent=1))
