"""cuFFT throughput probe (dev tool): a length-18432 transform batch against the
batched length-2048 / 9216 / 4608 transforms over the same data (torch.fft)."""
import torch, time
torch.backends.cuda.cufft_plan_cache.max_size = 16
def t(f, x, n=10):
    for _ in range(3): f(x)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): f(x)
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n
n1, B = 18432, 4609
xc = torch.randn(B, n1, dtype=torch.complex128, device='cuda')   # contiguous columns (current)
print('contiguous batch', B, 'x', n1, t(lambda x: torch.fft.fft(x, dim=1), xc), 'ms')
xr = torch.randn(n1, B, dtype=torch.complex128, device='cuda')   # strided (row-major band)
print('strided along dim0', t(lambda x: torch.fft.fft(x, dim=0), xr), 'ms')
x9 = torch.randn(B * 9, 2048, dtype=torch.complex128, device='cuda')
print('length-2048 batch', B*9, t(lambda x: torch.fft.fft(x, dim=1), x9), 'ms')
x2 = torch.randn(B, 9216, dtype=torch.complex128, device='cuda')
print('length-9216 batch', B, t(lambda x: torch.fft.fft(x, dim=1), x2), 'ms')
x3 = torch.randn(2*B, 9216, dtype=torch.complex128, device='cuda')
print('length-9216 batch', 2*B, t(lambda x: torch.fft.fft(x, dim=1), x3), 'ms')
x4 = torch.randn(B*4, 4608, dtype=torch.complex128, device='cuda')
print('length-4608 batch', 4*B, t(lambda x: torch.fft.fft(x, dim=1), x4), 'ms')
