import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1304_0878_b200 import btask as B
import workloads as W
elems = 1 << 30; T = 16384
f = W.sweep_factors(np.random.default_rng(1), 64)
for threads in (14,):
    rt = B.Runtime(device=0, host_threads=threads)
    addr, host = B.pinned_empty(elems * 4)
    host[:] = 1.5
    for step in range(3):
        t0 = time.perf_counter(); h = rt.register(addr, elems, 0); torch.cuda.synchronize(); t1 = time.perf_counter()
        subs = rt.partition(h, T); t2 = time.perf_counter()
        c = np.full(64*T, 1, np.int32); s = np.repeat(f, T); h0 = np.tile(np.array(subs, np.uint64), 64); t3 = time.perf_counter()
        rt.insert_batch(c, s, h0); t4 = time.perf_counter(); rt.wait(); t5 = time.perf_counter()
        rt.unpartition(h); t6 = time.perf_counter(); rt.unregister(h); t7 = time.perf_counter()
        print(f"threads={threads} register+sync {1e3*(t1-t0):.1f} partition {1e3*(t2-t1):.1f} arrays {1e3*(t3-t2):.1f} insert {1e3*(t4-t3):.1f} wait {1e3*(t5-t4):.1f} unpart {1e3*(t6-t5):.1f} unregister {1e3*(t7-t6):.1f} ms", flush=True)
    B.bt_free(addr); rt.close()
# raw copy bandwidth pinned
a = torch.empty(elems, dtype=torch.float32).pin_memory(); d = torch.empty(elems, dtype=torch.float32, device='cuda')
for _ in range(2):
    torch.cuda.synchronize(); t0=time.perf_counter(); d.copy_(a); torch.cuda.synchronize(); t1=time.perf_counter(); a.copy_(d); torch.cuda.synchronize(); t2=time.perf_counter()
    print(f"torch pinned H2D {4*elems/(t1-t0)/1e9:.1f} GB/s D2H {4*elems/(t2-t1)/1e9:.1f} GB/s")
