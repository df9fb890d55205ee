"""A/B of scheduler changes: the DAG and chain configs most sensitive to the
release path, for the library BT_LIB_PATH names (default: the in-tree build).

    BT_LIB_PATH=$PWD/paper_1304_0878_b200/libbtask_old.so python tools/ab_sched.py
    python tools/ab_sched.py

Prints one JSON line: device span (ms) of C3 (4 MiB buffers), C3 on 16 KiB
buffers (auto = rw, forced sw), C3 on 256 KiB buffers, the 1-wide chain
(us per link), C4b (kernel and host build) and C4 unfused.  Run both builds
alternately on the same box (box-to-box variation exceeds most effects).
Measurement helper only: no oracle.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench_configs as BC  # noqa: E402
import workloads as W  # noqa: E402
from paper_1304_0878_b200 import btask as B  # noqa: E402


def main():
    out = {}
    for name, p, kw in (("C3", W.c3_random_dag(), {}), ("C3s", W.c3_random_dag(nx=4096), {}),
                        ("C3s sw", W.c3_random_dag(nx=4096), {"flags": B.BT_FLAG_KERNEL_SW}),
                        ("C3 64K", W.c3_random_dag(nx=65536), {})):
        r, _ = BC._run(torch, B, p, 5, **kw)
        out[name] = round(r["device_span_ms"], 3)
    x = np.ones(1024, np.float32)
    pch = W.sweep_program(1024, 1, W.sweep_factors(np.random.default_rng(3), 10000), x, name="chain")
    r, _ = BC._run(torch, B, pch, 5, flags=B.BT_FLAG_NO_FUSION)
    out["chain_us"] = round(r["device_span_ms"] * 1e3 / 10000, 4)
    nt = 1 << 20
    pb = W.sweep_program(nt * 1024, nt, np.array([0.5], np.float32), np.ones(nt * 1024, np.float32), name="C4b")
    r, _ = BC._run(torch, B, pb, 3)
    out["C4b"] = {k: round(r[k], 3) for k in ("device_span_ms", "kernel_ms", "host_build_ms")}
    del pb
    r, _ = BC._run(torch, B, W.c4_fine(), 7, flush=BC._L2Flush(torch, 0), flags=B.BT_FLAG_NO_FUSION)
    out["C4u"] = {k: round(r[k], 3) for k in ("device_span_ms", "kernel_ms", "host_build_ms", "wall_ms")}
    print(os.path.basename(B.LIB_PATH), json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
