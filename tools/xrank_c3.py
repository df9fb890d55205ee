"""Cross-rank C3: a random DAG (12 buffers x 8K floats,
400 SCAL/AXPY/COPY tasks) with random owners over 2 ranks (processes), against
the same program on one rank.  Wall time per submit+wait (max over ranks) and
the number of rendezvous.  Both ranks share one GPU here (time-sliced
contexts), so this measures the protocol's latency, not NVLink.

    python tools/xrank_c3.py [--reps 20]   (BT_COMM_HOST=1: the host protocol)
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time
import uuid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(rank, nranks, name, reps, q):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import workloads as W
    from paper_1304_0878_b200 import btask as B
    from paper_1304_0878_b200.programs import Session
    from tests import xrank
    torch.cuda.set_device(0)
    p = W.c3_random_dag(nbuf=12, nx=1 << 13, ntasks=400, seed=4711)
    owners = xrank.owners_of(p, 2, 5) if nranks > 1 else [0] * len(p.buffers)
    tensors = [torch.from_numpy(b.copy()).cuda() for b in p.buffers]
    rt = B.Runtime(rank=rank, nranks=nranks)
    if nranks > 1:
        rt.comm_init(name)
    s = Session(rt, p, device_tensors=tensors)
    for b, own in enumerate(owners):
        rt.set_rank(s.roots[b], own)
    h0, h1 = s.handle_arrays()
    t = p.tasks
    c = np.ascontiguousarray(t["codelet"]).astype(np.int32)
    f = np.ascontiguousarray(t["scalar"]).astype(np.float32)
    walls, ins = [], []
    for r in range(reps + 3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rt.insert_batch(c, f, h0, h1)
        t1 = time.perf_counter()
        rt.wait()
        torch.cuda.synchronize()
        if r >= 3:
            walls.append(time.perf_counter() - t0)
            ins.append(t1 - t0)
    st = rt.stats()
    crossing = sum(1 for row in t if row["codelet"] != 1 and owners[row["b0"]] != owners[row["b1"]])
    s.finish()
    rt.close()
    q.put((rank, sorted(walls)[len(walls) // 2], st["epochs"] / (reps + 3), crossing, sorted(ins)[len(ins) // 2]))


def run(nranks, reps):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = f"/bt-xc3-{os.getpid()}-{uuid.uuid4().hex[:6]}"
    ps = [ctx.Process(target=worker, args=(r, nranks, name, reps, q)) for r in range(nranks)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=30)
    return max(r[1] for r in res), max(r[2] for r in res), res[0][3], max(r[4] for r in res)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    one, ep1, _, ins1 = run(1, args.reps)
    two, ep2, cross, ins2 = run(2, args.reps)
    print(json.dumps({"case": "C3 12 x 8K floats, 400 tasks", "protocol": "host" if os.environ.get("BT_COMM_HOST")
                      else ("device (flag kernels)" if os.environ.get("BT_COMM_FLAG_KERNELS") else "device"),
                      "ranks": "processes sharing one GPU (time-sliced contexts)",
                      "host_insert_ms_one": ins1 * 1e3, "host_insert_ms_two": ins2 * 1e3,
                      "one_rank_ms": one * 1e3, "two_ranks_ms": two * 1e3, "ratio": two / one,
                      "crossing_tasks": cross, "epochs_per_run_one": ep1, "epochs_per_run_two": ep2}), flush=True)


if __name__ == "__main__":
    main()
