import sys, json, time
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as W
from paper_1304_0878_b200 import btask as B
from paper_1304_0878_b200.programs import Session
p = W.c2_chain()
for cb in [0, 16384, 32768, 65536, 131072, 262144]:
    tensors = [torch.from_numpy(b).cuda() for b in p.buffers]
    with B.Runtime(chunk_bytes=cb) as rt:
        s = Session(rt, p, device_tensors=tensors)
        h0, h1 = s.handle_arrays()
        t = p.tasks
        spans = []
        for r in range(8):
            rt.stats_reset(); torch.cuda.synchronize()
            rt.insert_batch(t["codelet"], t["scalar"], h0)
            rt.wait()
            st = rt.stats()
            if r >= 2: spans.append(st["device_span_ms"])
        s.finish()
    print(json.dumps({"chunk_bytes": cb, "span_ms": float(np.median(spans)), "units": st["units"], "grid": st["grid"]}), flush=True)
