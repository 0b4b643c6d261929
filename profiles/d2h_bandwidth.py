"""Device-to-host copy bandwidth into pinned memory (the e2e read-back path)."""
import torch, time
dev = torch.device("cuda", 0)
x = torch.empty(100 << 20, dtype=torch.uint8, device=dev)
h = torch.empty(100 << 20, dtype=torch.uint8).pin_memory()
for _ in range(3): h.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): h.copy_(x, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("D2H GB/s", round((100 << 20) / ms / 1e6, 1))
# chunks of 6.2 MB
c = 1920 * 1080 * 3
e0.record()
for i in range(16): h[i*c:(i+1)*c].copy_(x[i*c:(i+1)*c], non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("16 x 6.2MB D2H GB/s", round(16 * c / e0.elapsed_time(e1) / 1e6, 1))
