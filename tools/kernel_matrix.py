"""Device time of DAG epochs per scheduler variant (auto / sw / rw / wq), to
fit the runtime's per-epoch kernel choice (runtime.cpp flush_epoch):

    python tools/kernel_matrix.py

Cases: C3-shaped random DAGs (10,000 tasks over 64 buffers) from 4 KiB to
4 MiB buffers; a 1-wide chain of 10,000 SCALs on one 4 KiB tile and on one
256 KiB vector (latency); C4-shaped tile-major fine DAG (not a pipelined run:
mixed codelets).  One JSON line per (case, kernel).  Measurement helper only.
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

KFLAG = {"auto": 0, "sw": B.BT_FLAG_KERNEL_SW, "rw": B.BT_FLAG_KERNEL_RW, "wq": B.BT_FLAG_KERNEL_WQ}


def k_chains(k: int, n: int, links: int):
    """k independent chains of `links` tasks, alternating SCAL x_i and
    AXPY(z_i -> x_i) (a DAG epoch, not a pipelined SCAL run), submitted
    round-robin over the chains."""
    rng = np.random.default_rng(k * 7 + n)
    bufs = [W.unit_interval_floats(rng, n) for _ in range(2 * k)]
    t = W._tasks(k * links)
    j = 0
    for step in range(links):
        for c in range(k):
            if step % 2 == 0:
                t[j] = (W.SCAL, np.float32(0.999), 2 * c, -1, -1, -1)
            else:
                t[j] = (W.AXPY, np.float32(1e-3), 2 * c + 1, -1, 2 * c, -1)
            j += 1
    return W.Program(bufs, [0] * (2 * k), t, name=f"{k} chains")


def cases():
    for nx in (1024, 4096, 16384, 65536, 262144, 1 << 20):
        yield f"C3 nx={nx}", W.c3_random_dag(nx=nx), 0
    rng = np.random.default_rng(3)
    for n in (1024, 65536):
        yield f"chain n={n}", W.sweep_program(n, 1, W.sweep_factors(rng, 10000), np.ones(n, np.float32)), \
            B.BT_FLAG_NO_FUSION
    p = W.c3_random_dag(nbuf=4096, nx=1024, ntasks=100000, seed=77)
    yield "C3 wide 4096 x 1024, 100k tasks", p, 0
    for k in (1, 2, 4, 8, 16, 32, 64, 256):
        for n in (1024, 65536):
            yield f"{k} chains n={n}", k_chains(k, n, 8192 // k if k < 256 else 64), 0
    yield "4096 chains n=1024 (wide)", k_chains(4096, 1024, 16), 0
    if os.environ.get("KM_RUNS"):   # pipelined SCAL runs (the first round's choice holds for the run)
        p = W.c4_fine()
        yield "C4 unfused", p, B.BT_FLAG_NO_FUSION
        yield "C4 fused", p, 0
        yield "C4 tile-major unfused", W.c4_fine(order="tile"), B.BT_FLAG_NO_FUSION
        nt = 1 << 20
        yield "C4b", W.sweep_program(nt * 1024, nt, np.array([0.5], np.float32), np.ones(nt * 1024, np.float32)), 0
        yield "C2 unfused", W.c2_chain(), B.BT_FLAG_NO_FUSION


def main():
    sel = [a for a in sys.argv[1:] if a in KFLAG] or list(KFLAG)
    only = os.environ.get("KM_ONLY")
    for name, p, flags in cases():
        if only and only not in name:
            continue
        for k in sel:
            r, _ = BC._run(torch, B, p, 3, flags=flags | KFLAG[k])
            print(json.dumps({"case": name, "kernel": k, "device_ms": round(r["device_span_ms"], 3),
                              "kernel_ms": round(r["kernel_ms"], 3), "items": r["items"], "edges": r["edges"],
                              "epochs": r["epochs"]}), flush=True)


if __name__ == "__main__":
    main()
