"""Run config C2 fused (256 tiles x 16 chained sweeps, one direct launch of one
item group) a few times through the ABI with device-resident data (for ncu
captures of the direct kernel).  Measurement helper only."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import bench_configs as BC  # noqa: E402
import workloads as W  # noqa: E402
from paper_1304_0878_b200 import btask as B  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
r, _ = BC._run(torch, B, W.c2_chain(), reps, flush=BC._L2Flush(torch, 0))
print("C2 fused device_ms", round(r["device_span_ms"], 4), "launches", r["launches"], flush=True)
