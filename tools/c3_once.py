"""Run config C3 (random DAG, 10,000 tasks over 64 x 4 MiB) a few times through
the ABI with device-resident data (for ncu captures of its scheduler kernel)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1304_0878_b200 import btask as B  # noqa: E402
from paper_1304_0878_b200.programs import Session  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p = W.c3_random_dag()
tensors = [torch.from_numpy(b).cuda() for b in p.buffers]
with B.Runtime() as rt:
    s = Session(rt, p, device_tensors=tensors)
    h0, h1 = s.handle_arrays()
    t = p.tasks
    for r in range(reps):
        rt.stats_reset()
        rt.insert_batch(t["codelet"], t["scalar"], h0, h1)
        rt.wait()
        st = rt.stats()
        print(r, "device_ms", round(st["device_ms"], 3), "epochs", st["epochs"], "units", st["units"], flush=True)
    s.finish()
