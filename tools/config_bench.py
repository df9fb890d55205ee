"""Throughput of every BASELINE config through the C ABI (device-resident data),
against its roofline.  One JSON line per case; used for profiles/.

    python tools/config_bench.py [--reps 5]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1304_0878_b200 import btask as B  # noqa: E402
from paper_1304_0878_b200.programs import Session  # noqa: E402

PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}
FMUL_PEAK = 148 * 128 * PEAKS.get("sm_max_mhz", 1965.0) * 1e6


def algorithmic(p):
    """Unfused algorithmic bytes and FP32 ops of the task stream."""
    t = p.tasks
    nbytes = flops = 0
    sizes = {}
    for b, buf in enumerate(p.buffers):
        nparts = p.nparts[b]
        sizes[b] = buf.shape[0] // nparts if nparts else buf.shape[0]
    for c, b0 in zip(t["codelet"], t["b0"]):
        n = sizes[int(b0)]
        if c == W.SCAL:
            nbytes += 8 * n
            flops += n
        elif c == W.AXPY:
            nbytes += 12 * n
            flops += 2 * n
        else:
            nbytes += 8 * n
    return nbytes, flops


def run(name, p, reps, **kw):
    tensors = [torch.from_numpy(b).cuda() for b in p.buffers]
    with B.Runtime(**kw) as rt:
        s = Session(rt, p, device_tensors=tensors)
        h0, h1 = s.handle_arrays()
        only_scal = bool(np.all(p.tasks["codelet"] == W.SCAL))
        # contiguous task columns made once (strided structured-array views
        # would be copied by the binding inside the timed region)
        t = {k: np.ascontiguousarray(p.tasks[k]) for k in ("codelet", "scalar")}
        t["codelet"] = t["codelet"].astype(np.int32)
        t["scalar"] = t["scalar"].astype(np.float32)
        h0 = np.ascontiguousarray(h0, np.uint64)
        h1 = np.ascontiguousarray(h1, np.uint64)
        times, dev = [], []
        for r in range(reps + 1):
            rt.stats_reset()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rt.insert_batch(t["codelet"], t["scalar"], h0, None if only_scal else h1)
            rt.wait()
            t1 = time.perf_counter()
            st = rt.stats()
            if r:
                times.append((t1 - t0) * 1e3)
                dev.append(st["device_span_ms"])
        s.finish()
    nbytes, flops = algorithmic(p)
    wall = float(np.median(times))
    span = float(np.median(dev))
    t_roof = max(nbytes / (PEAKS["hbm_gbs"] * 1e9), flops / FMUL_PEAK) * 1e3
    out = {"case": name, "tasks": p.ntasks, "wall_ms": wall, "device_span_ms": span,
           "tasks_per_s_wall": p.ntasks / (wall * 1e-3), "effective_task_GBps_device": nbytes / (span * 1e-3) / 1e9,
           "unfused_roofline_ms": t_roof, "items": st["items"], "edges": st["edges"], "epochs": st["epochs"],
           "grid": st["grid"]}
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    # C1 latency: one task, submit -> wait
    p = W.c1_single()
    run("C1 single vector_scal (1024 floats)", p, 20)
    p = W.c2_chain()
    run("C2 16-chain over 256 tiles, fused", p, args.reps)
    run("C2 16-chain over 256 tiles, unfused", p, args.reps, flags=B.BT_FLAG_NO_FUSION)
    p = W.c3_random_dag()
    run("C3 random DAG 10,000 tasks over 64 x 4 MiB", p, args.reps)
    p = W.c4_fine()
    run("C4 1,000,000 tasks on 4 KiB tiles, unfused", p, args.reps, flags=B.BT_FLAG_NO_FUSION)
    run("C4 fused", p, args.reps)


if __name__ == "__main__":
    main()
