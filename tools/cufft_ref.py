"""Reference point only: cuFFT (via torch.fft) time for the 1080p deconvolution grid.
Not used by the product path; it calibrates what the hand-written FFT should reach."""
import torch
dev = torch.device("cuda")
x = torch.randn(3, 1120, 1944, device=dev)
h = torch.randn(1120, 973, dtype=torch.complex64, device=dev)
def run():
    X = torch.fft.rfft2(x)
    X *= h
    return torch.fft.irfft2(X, s=(1120, 1944))
for _ in range(5): run()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(50): run()
e.record(); torch.cuda.synchronize()
print(f"cuFFT rfft2+mul+irfft2 per plane: {s.elapsed_time(e)/50/3*1000:.1f} us")
s.record()
for _ in range(50): torch.fft.rfft2(x)
e.record(); torch.cuda.synchronize()
print(f"cuFFT rfft2 per plane: {s.elapsed_time(e)/50/3*1000:.1f} us")
