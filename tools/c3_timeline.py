"""C3 occupancy timeline from per-unit trace records (BT_FLAG_TIMESTAMPS):
how many CTAs run a unit body over time, i.e. whether C3 is starved of ready
work (DAG-bound) or runs every CTA and is bound by the bodies.

    python tools/c3_timeline.py [sw|rw|auto]

(tracing turns the local continuations off: an approximation of the untraced run)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1304_0878_b200 import btask as B  # noqa: E402
import bench_configs as bc  # noqa: E402

p = W.c3_random_dag()
kern = sys.argv[1] if len(sys.argv) > 1 else "auto"
kf = {"sw": B.BT_FLAG_KERNEL_SW, "rw": B.BT_FLAG_KERNEL_RW, "auto": 0}[kern]
r, tr = bc._run(torch, B, p, 1, flags=B.BT_FLAG_TIMESTAMPS | kf)
t, item = tr
mhz = 1965.0
start = t[:, 0] + t[:, 1] * 1e3 / mhz            # body start (ns)
end = start + t[:, 2] * 1e3 / mhz                # body end
t0 = start.min()
ev = np.concatenate([np.stack([start - t0, np.ones_like(start)], 1), np.stack([end - t0, -np.ones_like(end)], 1)])
ev = ev[np.argsort(ev[:, 0], kind="stable")]
conc = np.cumsum(ev[:, 1])
dt = np.diff(ev[:, 0], append=ev[-1, 0])
total = ev[-1, 0]
hist = {}
for lo, hi in [(0, 100), (100, 200), (200, 300), (300, 400), (400, 445)]:
    sel = (conc >= lo) & (conc < hi)
    hist[f"{lo}-{hi}"] = float(dt[sel].sum() / total)
# concurrency over the run in 20 slices (is the start, the middle or the tail starved?)
edges = np.linspace(0, total, 21)
sl = []
for a0, a1 in zip(edges[:-1], edges[1:]):
    seg = (ev[:, 0] >= a0) & (ev[:, 0] < a1)
    sl.append(round(float((conc[seg] * dt[seg]).sum() / max(1.0, dt[seg].sum())), 1))
out = {"kernel": kern, "concurrency_by_twentieth": sl, "device_ms": r["device_span_ms"], "units": int(t.shape[0]), "span_ms": total / 1e6,
       "mean_concurrent_bodies": float((conc * dt).sum() / total), "time_fraction_by_concurrency": hist,
       "body_us_median": float(np.median(t[:, 2]) / mhz), "pop_us_median": float(np.median(t[:, 1]) / mhz),
       "release_us_median": float(np.median(t[:, 3]) / mhz)}
print(json.dumps(out), flush=True)
