"""Priority ready queue (upward-rank levels) against the FIFO on
C3 (64 x 4 MiB: HBM-bound) and C3s (64 x 16 KiB: dependency-latency bound),
device time through the C ABI.   python tools/prio_compare.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1304_0878_b200 import btask as B  # noqa: E402
import bench_configs as bc  # noqa: E402

for name, p, kw in (("C3", W.c3_random_dag(), {}),
                    ("C3s nx=4096", W.c3_random_dag(nx=4096), {}),
                    ("C3s nx=4096 sw", W.c3_random_dag(nx=4096), {"flags": B.BT_FLAG_KERNEL_SW}),
                    ("C3 nx=65536", W.c3_random_dag(nx=65536), {})):
    for mode, extra in (("priority", B.BT_FLAG_PRIORITY), ("fifo", 0)):
        kw2 = dict(kw, flags=kw.get("flags", 0) | extra)
        r, _ = bc._run(torch, B, p, 5, **kw2)
        print(json.dumps({"case": name, "queue": mode, "device_ms": r["device_span_ms"], "wall_ms": r["wall_ms"],
                          "items": r["items"], "edges": r["edges"]}), flush=True)
