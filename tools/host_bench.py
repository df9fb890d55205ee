"""Host dependency-builder throughput: bt_insert_task_batch of the C5 / C4
task streams for several builder thread counts (GPU runtime if available,
else a host-only runtime, which also records the task->item map).

    python tools/host_bench.py [--threads 1,2,4,8,16]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from paper_1304_0878_b200 import btask as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", default="1,2,4,8,16")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    try:
        import torch
        gpu = torch.cuda.is_available()
    except Exception:
        gpu = False
    out = []
    for fusion in (True, False):
        for T in [int(t) for t in args.threads.split(",")]:
            flags = (0 if fusion else B.BT_FLAG_NO_FUSION) | (0 if gpu else B.BT_FLAG_HOST_ONLY)
            rt = B.Runtime(flags=flags, host_threads=T)
            ntiles, sweeps = 16384, 64
            if gpu:
                t = torch.empty(ntiles * 64, dtype=torch.float32, device="cuda")
                h = rt.register_tensor(t)
            else:
                x = np.zeros(ntiles * 64, np.float32)
                h = rt.register_array(x)
            subs = rt.partition(h, ntiles)
            f = W.sweep_factors(np.random.default_rng(1), sweeps)
            c = np.full(sweeps * ntiles, 1, np.int32)
            s = np.repeat(f, ntiles)
            h0 = np.tile(np.array(subs, np.uint64), sweeps)
            ins, fin = [], []
            for rep in range(args.reps):
                t0 = time.perf_counter()
                rt.insert_batch(c, s, h0)
                t1 = time.perf_counter()
                if gpu:
                    rt.flush()
                else:
                    rt.dag_snapshot()
                t2 = time.perf_counter()
                if gpu:
                    rt.wait()
                ins.append((t1 - t0) * 1e3)
                fin.append((t2 - t1) * 1e3)
            st = rt.stats()
            rt.unpartition(h)
            rt.unregister(h)
            rt.close()
            row = {"fusion": fusion, "threads": T, "gpu_runtime": gpu, "tasks": int(c.shape[0]),
                   "insert_ms_min": min(ins[1:]), "insert_ms_med": float(np.median(ins[1:])),
                   "pack_launch_ms_min": min(fin[1:]), "items_per_epoch": st["items"] // max(1, st["epochs"] or
                                                                                          args.reps)}
            print(json.dumps(row), flush=True)
            out.append(row)
    return 0


if __name__ == "__main__":
    sys.exit(main())
