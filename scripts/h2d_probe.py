import time, torch, ctypes as C
x = torch.empty(1 << 28, dtype=torch.float32, pin_memory=True)  # 1 GiB
x.fill_(1.0)
y = torch.empty_like(x, device="cuda")
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize()
    print("pinned H2D GB/s", x.numel() * 4 / (time.perf_counter() - t) / 1e9)
z = torch.empty(1 << 28, dtype=torch.float32); z.fill_(1.0)
torch.cuda.synchronize(); t = time.perf_counter(); y.copy_(z); torch.cuda.synchronize()
print("pageable H2D GB/s", z.numel() * 4 / (time.perf_counter() - t) / 1e9)
print(torch.cuda.get_device_properties(0))
