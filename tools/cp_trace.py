"""Per-link timeline of a 200-long chain of 4 MiB tasks on the sw kernel from
BT_FLAG_TIMESTAMPS traces (task span, gaps, per-unit pop/body/release)."""
import sys, json
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as W
from paper_1304_0878_b200 import btask as B
from paper_1304_0878_b200.programs import Session
rng = np.random.default_rng(1)
x = W.unit_interval_floats(rng, 1 << 20)
f = W.sweep_factors(rng, 200)
p = W.sweep_program(x.shape[0], 1, f, x)
t = torch.from_numpy(p.buffers[0].copy()).cuda()
with B.Runtime(flags=B.BT_FLAG_NO_FUSION | B.BT_FLAG_KERNEL_SW | B.BT_FLAG_TIMESTAMPS) as rt:
    s = Session(rt, p, device_tensors=[t])
    h0, h1 = s.handle_arrays()
    for r in range(2):
        rt.insert_batch(p.tasks["codelet"], p.tasks["scalar"], h0)
        rt.wait()
    tr, item = rt.trace()
    s.finish()
ns = 1.0 / 1.965
g0 = tr[:, 0].astype(np.float64)
pop = tr[:, 1] * ns; body = tr[:, 2] * ns; rel = tr[:, 3] * ns
start = g0 + pop; end = start + body + rel
items = np.unique(item)
S = np.array([start[item == i].min() for i in items]); E = np.array([end[item == i].max() for i in items])
Bs = np.array([(start[item == i] + body[item == i]).max() for i in items])  # last body end
o = np.argsort(S); S, E, Bs = S[o], E[o], Bs[o]
print(json.dumps({"links": len(S), "task_span_us_med": float(np.median(E - S) / 1e3),
                  "first_to_last_body_end_us": float(np.median(Bs - S) / 1e3),
                  "gap_us_med": float(np.median(S[1:] - E[:-1]) / 1e3),
                  "link_us_med": float(np.median(S[1:] - S[:-1]) / 1e3),
                  "body_us_med": float(np.median(body) / 1e3), "pop_us_med": float(np.median(pop) / 1e3),
                  "release_us_med": float(np.median(rel) / 1e3)}))
