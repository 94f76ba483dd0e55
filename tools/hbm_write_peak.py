"""Write-only HBM bandwidth on this B200 (context for the replay kernel's write-bound full mode):
torch fill_ / zero_ (cudaMemsetAsync) and a streaming-store copy of 2 GiB, CUDA events."""
import torch

n = 2 << 30
x = torch.empty(n // 8, dtype=torch.int64, device="cuda")
y = torch.empty_like(x)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, mult in (("fill_", lambda: x.fill_(7), 1), ("zero_", lambda: x.zero_(), 1), ("copy_", lambda: y.copy_(x), 2)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    print(f"{name}: {mult * n / (best * 1e-3) / 1e9:8.1f} GB/s ({best:.3f} ms for {mult} x 2 GiB)")
