"""Scheduler-overhead measurements, on one B200.

  (a) per-unit pop / release cost from in-kernel timestamps (BT_FLAG_TIMESTAMPS),
  (b) (T_device - T_roofline) / N for C4 unfused (1,000,000 tasks on 4 KiB tiles),
  (c) dependency latency: a 1-wide chain of 10,000 SCALs on one 4 KiB tile,
  (d) pure pop rate: C4b, 1,000,000 independent 4 KiB tiles x 1 task.
All through the C ABI with device-resident data; prints one JSON line per case.

    python tools/sched_overhead.py
"""
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

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def sm_clock_mhz():
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        return pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    except Exception:
        return 1965.0


def run_case(name, ntiles, tile, sweeps, flags, reps=5, trace=False):
    rt = B.Runtime(flags=flags | (B.BT_FLAG_TIMESTAMPS if trace else 0))
    x = torch.full((ntiles * tile,), 1.0, dtype=torch.float32, device="cuda")
    h = rt.register_tensor(x)
    subs = rt.partition(h, ntiles) if ntiles > 1 else [h]
    f = W.sweep_factors(np.random.default_rng(3), sweeps)
    c = np.full(ntiles * sweeps, 1, np.int32)
    s = np.repeat(f, ntiles)
    h0 = np.tile(np.asarray(subs, np.uint64), sweeps)
    dev, host, wall = [], [], []
    for r in range(reps + 1):
        rt.stats_reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rt.insert_batch(c, s, h0)
        rt.wait()
        t1 = time.perf_counter()
        st = rt.stats()
        if r:
            dev.append(st["device_ms"])
            host.append(st["host_build_ms"])
            wall.append((t1 - t0) * 1e3)
    tr = rt.trace() if trace else None
    if ntiles > 1:
        rt.unpartition(h)
    rt.unregister(h)
    rt.close()
    n = ntiles * sweeps
    t_dev = float(np.median(dev))
    t_roof = 8.0 * tile * n / (HBM * 1e9) * 1e3
    out = {"case": name, "tasks": n, "tile_bytes": 4 * tile, "device_ms": t_dev, "host_build_ms": float(np.median(host)),
           "wall_ms": float(np.median(wall)), "tasks_per_s_device": n / (t_dev * 1e-3),
           "hbm_roofline_ms": t_roof, "overhead_ns_per_task": (t_dev - t_roof) * 1e6 / n,
           "device_ns_per_task": t_dev * 1e6 / n, "items": st["items"], "edges": st["edges"], "grid": st["grid"]}
    if tr is not None:
        t, _ = tr
        mhz = sm_clock_mhz()
        ns = 1e3 / mhz
        out.update({"sm_mhz": mhz, "pop_ns_median": float(np.median(t[:, 1]) * ns),
                    "pop_ns_p99": float(np.percentile(t[:, 1], 99) * ns),
                    "body_span_ns_median": float(np.median(t[:, 2]) * ns),
                    "release_ns_median": float(np.median(t[:, 3]) * ns),
                    "release_ns_p99": float(np.percentile(t[:, 3], 99) * ns)})
    print(json.dumps(out), flush=True)
    return out


CASES = [
    ("C4 unfused (1M tasks, 4 KiB tiles, 64 sweeps)", 15625, 1024, 64, B.BT_FLAG_NO_FUSION, 5, False),
    ("C4 unfused, timestamps", 15625, 1024, 64, B.BT_FLAG_NO_FUSION, 2, True),
    ("C4 fused", 15625, 1024, 64, 0, 5, False),
    ("chain of 10,000 on one 4 KiB tile (dependency latency)", 1, 1024, 10000, B.BT_FLAG_NO_FUSION, 3, False),
    ("chain of 10,000, timestamps", 1, 1024, 10000, B.BT_FLAG_NO_FUSION, 3, True),
    ("C4b: 1M independent 4 KiB tiles x 1 task (pop rate)", 1 << 20, 1024, 1, 0, 5, False),
    ("C4b, timestamps", 1 << 20, 1024, 1, 0, 2, True),
]


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="", help="run only cases whose name starts with this (e.g. for ncu)")
    ap.add_argument("--reps", type=int, default=0, help="override the repetitions")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    for name, ntiles, tile, sweeps, flags, reps, trace in CASES:
        if args.case and not name.startswith(args.case):
            continue
        run_case(name, ntiles, tile, sweeps, flags, reps=args.reps or reps, trace=trace)


if __name__ == "__main__":
    main()
