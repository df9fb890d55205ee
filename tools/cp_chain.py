"""Dependency latency of a DAG link with multi-unit tasks: a 632-long chain
(C3's critical-path length) of unfused SCALs on one 4 MiB buffer (64 units of
64 KiB per task), per scheduler variant."""
import sys, json
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as W
from paper_1304_0878_b200 import btask as B
from paper_1304_0878_b200.programs import Session
for ntiles_dummy in [1]:
    rng = np.random.default_rng(1)
    x = W.unit_interval_floats(rng, 1 << 20)
    f = W.sweep_factors(rng, 632)
    p = W.sweep_program(x.shape[0], 1, f, x, name="632-chain of 4 MiB SCALs")
    for kern, flag in [("sw", B.BT_FLAG_KERNEL_SW), ("rw", B.BT_FLAG_KERNEL_RW)]:
        t = torch.from_numpy(p.buffers[0].copy()).cuda()
        with B.Runtime(flags=B.BT_FLAG_NO_FUSION | flag) as rt:
            s = Session(rt, p, device_tensors=[t])
            h0, h1 = s.handle_arrays()
            ms = []
            for r in range(4):
                rt.stats_reset()
                rt.insert_batch(p.tasks["codelet"], p.tasks["scalar"], h0)
                rt.wait()
                if r: ms.append(rt.stats()["device_span_ms"])
            s.finish()
        print(json.dumps({"kernel": kern, "chain_ms": float(np.median(ms)), "us_per_link": float(np.median(ms)) * 1e3 / 632}), flush=True)
