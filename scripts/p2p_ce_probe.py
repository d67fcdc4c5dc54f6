"""Copy-engine peer bandwidth between two B200s (gpurun --gpus 2): one
direction and both at once, cudaMemcpyPeerAsync via torch, sizes like the
engine's reductions; and the same copy beside a HBM-bound kernel on the
destination (how much the copy slows the kernel and vice versa)."""
import time
import torch

def bw(fn, nbytes, it=10):
    fn(); torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    t = time.perf_counter()
    for _ in range(it):
        fn()
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    return nbytes * it / (time.perf_counter() - t) / 1e9

print("p2p", torch.cuda.can_device_access_peer(0, 1))
for mb in (64, 256, 1024):
    n = mb * (1 << 20) // 4
    a0 = torch.rand(n, device="cuda:0"); a1 = torch.rand(n, device="cuda:1")
    b0 = torch.empty(n, device="cuda:0"); b1 = torch.empty(n, device="cuda:1")
    s0 = torch.cuda.Stream(device=0); s1 = torch.cuda.Stream(device=1)
    def one():
        with torch.cuda.stream(s1):
            b1.copy_(a0, non_blocking=True)   # pull 0 -> 1 on device 1's stream
    def both():
        with torch.cuda.stream(s1):
            b1.copy_(a0, non_blocking=True)
        with torch.cuda.stream(s0):
            b0.copy_(a1, non_blocking=True)
    print(f"{mb} MB: one-way {bw(one, n * 4):.0f} GB/s, both ways {bw(both, 2 * n * 4) / 2:.0f} GB/s per direction", flush=True)
# beside a streaming kernel on device 1
n = 1024 * (1 << 20) // 4
a0 = torch.rand(n, device="cuda:0"); b1 = torch.empty(n, device="cuda:1")
x = torch.rand(4 * n, device="cuda:1"); y = torch.empty_like(x)
s1 = torch.cuda.Stream(device=1); k1 = torch.cuda.Stream(device=1)
def kern():
    with torch.cuda.stream(k1):
        y.copy_(x)
def copy():
    with torch.cuda.stream(s1):
        b1.copy_(a0, non_blocking=True)
def tm(fn, it=10):
    fn(); torch.cuda.synchronize(1); torch.cuda.synchronize(0)
    t = time.perf_counter()
    for _ in range(it): fn()
    torch.cuda.synchronize(1); torch.cuda.synchronize(0)
    return (time.perf_counter() - t) / it * 1e3
tk, tc = tm(kern), tm(copy)
tb = tm(lambda: (kern(), copy()))
print(f"kernel alone {tk:.2f} ms, copy alone {tc:.2f} ms, together {tb:.2f} ms", flush=True)
