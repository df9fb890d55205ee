"""Write C3's work units as a job list (tools/chunk_probe.cu) and run the probe:
C3 without dependencies, in submission order and shuffled.

    python tools/chunk_probe.py
Measurement helper only (workloads' generator; no oracle, no product code).
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

JOB = np.dtype([("kind", "<u4"), ("x", "<u4"), ("y", "<u4"), ("chunk", "<u4"), ("a", "<f4")])


def jobs(order):
    p = W.c3_random_dag()
    t = p.tasks
    nchunk = p.buffers[0].shape[0] // 16384
    n = t.shape[0] * nchunk
    j = np.zeros(n, JOB)
    j["kind"] = np.repeat(t["codelet"], nchunk)
    j["x"] = np.repeat(t["b0"], nchunk)
    j["y"] = np.repeat(np.where(t["codelet"] == W.SCAL, t["b0"], t["b1"]), nchunk)
    j["chunk"] = np.tile(np.arange(nchunk, dtype=np.uint32), t.shape[0])
    j["a"] = np.repeat(t["scalar"], nchunk)
    if order == "shuffled":
        j = j[np.random.default_rng(5).permutation(n)]
    return len(p.buffers), j


def main():
    exe = os.path.join(ROOT, "tools", "chunk_probe")
    src = exe + ".cu"
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false", "-lineinfo",
                               src, "-o", exe])
    for order in (sys.argv[1:] or ["submission", "shuffled"]):
        nbuf, j = jobs(order)
        path = f"/tmp/c3_jobs_{order}.bin"
        with open(path, "wb") as f:
            f.write(np.array([nbuf, j.shape[0]], "<u4").tobytes())
            f.write(j.tobytes())
        subprocess.check_call([exe, path, "5"])


if __name__ == "__main__":
    main()
