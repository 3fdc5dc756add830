import torch
s = torch.randint(0, 256, (1 << 28,), dtype=torch.uint8, device="cuda")
d = torch.empty(1 << 28, dtype=torch.bfloat16, device="cuda")
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
for _ in range(3): d.copy_(s)
e0.record()
for _ in range(10): d.copy_(s)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 10 * 1e-3
print(f"u8->bf16 copy: {3 * s.numel() / t / 1e9:.0f} GB/s (read+write)")
d2 = torch.empty_like(d)
e0.record()
for _ in range(10): d2.copy_(d)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 10 * 1e-3
print(f"bf16 copy: {4 * s.numel() / t / 1e9:.0f} GB/s (read+write)")
d.fill_(1.0)
e0.record()
for _ in range(10): d.fill_(2.0)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 10 * 1e-3
print(f"bf16 fill (write only): {2 * s.numel() / t / 1e9:.0f} GB/s")
