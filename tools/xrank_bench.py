"""Cross-rank read cost (bt_comm_init): two ranks (processes) ping-pong a buffer.

rank 0 owns X, rank 1 owns Y; each iteration submits COPY X->Y (runs on rank 1,
reads X from rank 0) and COPY Y->X (runs on rank 0, reads Y from rank 1): two
rendezvous per iteration.  Reports wall time per rendezvous for several sizes.
On one GPU the two ranks share the device (the copy is a device-local copy, not
NVLink); the host-side rendezvous latency is what this measures.

    python tools/xrank_bench.py [--iters 200]
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time
import uuid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(rank, name, sizes, iters, q):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    from paper_1304_0878_b200 import btask as B
    torch.cuda.set_device(0)
    rt = B.Runtime(rank=rank, nranks=2)
    rt.comm_init(name)
    out = []
    for n in sizes:
        x = torch.ones(n, dtype=torch.float32, device="cuda")
        y = torch.zeros(n, dtype=torch.float32, device="cuda")
        hx, hy = rt.register_tensor(x), rt.register_tensor(y)
        rt.set_rank(hx, 0)
        rt.set_rank(hy, 1)
        for it in range(iters + 10):
            if it == 10:
                rt.wait()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
            rt.copy(hx, hy)
            rt.copy(hy, hx)
        rt.wait()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out.append({"bytes": 4 * n, "us_per_rendezvous": dt / (2 * iters) * 1e6,
                    "GBps": 4 * n * 2 * iters / dt / 1e9})
        rt.unregister(hx)
        rt.unregister(hy)
    rt.close()
    q.put((rank, out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    args = ap.parse_args()
    sizes = [1024, 1 << 16, 1 << 20, 1 << 24]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = f"/bt-xbench-{os.getpid()}-{uuid.uuid4().hex[:6]}"
    ps = [ctx.Process(target=worker, args=(r, name, sizes, args.iters, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=30)
    for i, n in enumerate(sizes):
        r0, r1 = res[0][i], res[1][i]
        print(json.dumps({"case": "cross-rank ping-pong (2 ranks, one GPU)", "bytes": 4 * n,
                          "us_per_rendezvous": max(r0["us_per_rendezvous"], r1["us_per_rendezvous"]),
                          "GBps": min(r0["GBps"], r1["GBps"])}), flush=True)


if __name__ == "__main__":
    main()
