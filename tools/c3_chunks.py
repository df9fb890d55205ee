"""C3 (random DAG, 64 x 4 MiB buffers) device time vs work-unit size and
scheduler variant:  python tools/c3_chunks.py [auto|sw|rw|wq ...]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import workloads as W
from paper_1304_0878_b200 import btask as B
from paper_1304_0878_b200.programs import Session

p = W.c3_random_dag()
tensors = [torch.from_numpy(b).cuda() for b in p.buffers]
KFLAG = {"auto": 0, "sw": B.BT_FLAG_KERNEL_SW, "rw": B.BT_FLAG_KERNEL_RW, "wq": B.BT_FLAG_KERNEL_WQ}
kernels = sys.argv[1:] or ["auto"]
for kern, cb in [(k, c) for k in kernels for c in [0, 16384, 32768, 65536, 131072, 262144]]:
    with B.Runtime(chunk_bytes=cb, flags=KFLAG[kern]) as rt:
        s = Session(rt, p, device_tensors=tensors)
        h0, h1 = s.handle_arrays()
        t = p.tasks
        dev = []
        for r in range(4):
            rt.stats_reset()
            rt.insert_batch(t["codelet"], t["scalar"], h0, h1)
            rt.wait()
            if r:
                dev.append(rt.stats()["device_span_ms"])
        s.finish()
    print(json.dumps({"kernel": kern, "chunk_bytes": cb, "device_ms": float(np.median(dev))}), flush=True)
