"""Plain read / copy bandwidth of this B200 through torch (sum and copy of 400 MB):
the practical streaming bound the selection passes are compared against."""
import torch
x = torch.rand(100_000_000, device="cuda")
for _ in range(3): y = x.sum()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): y = x.sum()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print("torch sum 400MB: %.1f us  %.2f TB/s" % (ms * 1e3, 0.4 / (ms * 1e-3) / 1e3))
z = torch.empty_like(x)
e0.record()
for _ in range(20): z.copy_(x)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print("torch copy 400MB: %.1f us  %.2f TB/s (r+w)" % (ms * 1e3, 0.8 / (ms * 1e-3) / 1e3))
