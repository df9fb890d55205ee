"""Do H2D and D2H copies on two streams overlap (PCIe full duplex)?"""
import time
import torch

n = 1 << 28  # 1 GiB of float32
a = torch.empty(n, dtype=torch.float32).pin_memory()
b = torch.empty(n, dtype=torch.float32).pin_memory()
da = torch.empty(n, dtype=torch.float32, device="cuda")
db = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        da.copy_(a, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    with torch.cuda.stream(s2):
        b.copy_(db, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    with torch.cuda.stream(s1):
        da.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2):
        b.copy_(db, non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"H2D {4*n/(t1-t0)/1e9:.1f} GB/s  D2H {4*n/(t2-t1)/1e9:.1f} GB/s  both concurrently {(t3-t2)*1e3:.1f} ms "
          f"(sequential would be {(t2-t0)*1e3:.1f} ms)")
