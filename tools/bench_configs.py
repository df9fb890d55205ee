"""Secondary bench keys: every BASELINE config other than the headline C5, through
the C ABI with device-resident inputs (SURVEY.md 8(d) "Report" column).

    C1  submit -> wait latency of the paper's running example (one task)
    C2  16-chain over 256 tiles, fused and unfused (L2 flushed before each rep)
    C3  random DAG of 10,000 SCAL/AXPY/COPY tasks over 64 x 4 MiB buffers
    C4  1,000,000 tasks on 4 KiB tiles (unfused: scheduler-bound; fused),
        C4b (1M independent tiles), a 1-wide chain of 10,000 (dependency
        latency), and the in-kernel pop / release distribution from per-unit
        trace records (each unit writes its own record: no shared counter)

Called by bench.py (rank 0, N = 1) as ``run_all(dev)``; also runnable alone:
    python tools/bench_configs.py
Measurement helper only: no oracle, nothing of the method's arithmetic.
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}


def algorithmic(p):
    """Unfused algorithmic bytes and FP32 multiplies of a task stream."""
    t = p.tasks
    sizes = []
    for b, buf in enumerate(p.buffers):
        nparts = p.nparts[b]
        sizes.append(buf.shape[0] // nparts if nparts else buf.shape[0])
    n = np.asarray(sizes, np.int64)[t["b0"]]
    c = t["codelet"]
    nbytes = int(np.sum(np.where(c == 2, 12 * n, 8 * n)))
    fmul = int(np.sum(np.where(c == 3, 0, n)))
    return nbytes, fmul


class _L2Flush:
    """Evict the 126 MB L2 before a rep by READING a 512 MiB buffer: the L2 then
    holds clean lines (a written scratch would leave ~126 MB of dirty lines
    whose write-back the next kernel pays for)."""

    def __init__(self, torch, dev, nbytes=512 << 20):
        self.buf = torch.ones(nbytes // 4, dtype=torch.float32, device=dev)
        self.out = torch.empty((), dtype=torch.float32, device=dev)

    def __call__(self):
        import torch
        torch.sum(self.buf, dim=0, out=self.out)


def _run(torch, B, p, reps, flush=None, **kw):
    """Median wall (insert -> wait return) and device span over reps (+1 warm-up)."""
    from paper_1304_0878_b200.programs import Session
    tensors = [torch.from_numpy(b).cuda() for b in p.buffers]
    with B.Runtime(**kw) as rt:
        s = Session(rt, p, device_tensors=tensors)
        h0, h1 = s.handle_arrays()
        only_scal = bool(np.all(p.tasks["codelet"] == 1))
        c = np.ascontiguousarray(p.tasks["codelet"]).astype(np.int32)
        f = np.ascontiguousarray(p.tasks["scalar"]).astype(np.float32)
        h0 = np.ascontiguousarray(h0, np.uint64)
        h1 = np.ascontiguousarray(h1, np.uint64)
        wall, span, dev, host = [], [], [], []
        st = None
        for r in range(reps + 1):
            if flush:
                flush()
            torch.cuda.synchronize()
            rt.stats_reset()
            t0 = time.perf_counter()
            rt.insert_batch(c, f, h0, None if only_scal else h1)
            rt.wait()
            t1 = time.perf_counter()
            st = rt.stats()
            if r:
                wall.append((t1 - t0) * 1e3)
                span.append(st["device_span_ms"])
                dev.append(st["device_ms"])
                host.append(st["host_build_ms"])
        tr = rt.trace() if kw.get("flags", 0) & B.BT_FLAG_TIMESTAMPS else None
        s.finish()
    del tensors
    return {"wall_ms": float(np.median(wall)), "device_span_ms": float(np.median(span)),
            "kernel_ms": float(np.median(dev)), "host_build_ms": float(np.median(host)), "items": int(st["items"]),
            "edges": int(st["edges"]), "epochs": int(st["epochs"]), "launches": int(st["kernel_launches"]),
            "stream_resumes": int(st.get("stream_resumes", 0))}, tr


def run_all(dev: int = 0, quick: bool = False) -> dict:
    import torch
    import workloads as W
    from paper_1304_0878_b200 import btask as B
    torch.cuda.set_device(dev)
    peaks = _peaks()
    hbm = peaks["hbm_gbs"]
    props = torch.cuda.get_device_properties(dev)
    fmul_peak = props.multi_processor_count * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6
    flush = _L2Flush(torch, dev)
    reps = 3 if quick else 7
    out = {"note": "secondary keys (not the headline): device-resident inputs, through the C ABI; "
                   "wall = bt_insert_task_batch entry -> bt_task_wait_for_all return; device = CUDA events "
                   "around the epochs' launches; effective GB/s = unfused algorithmic task bytes / device time",
           "hbm_peak_GBps": hbm, "fmul_peak_T_per_s": fmul_peak / 1e12, "sms": props.multi_processor_count}

    # C1: the paper's running example, one SCAL of 1,024 floats
    p = W.c1_single()
    r, _ = _run(torch, B, p, 30 if not quick else 10)
    out["C1"] = {"workload": p.name, "submit_to_wait_us": r["wall_ms"] * 1e3, "device_us": r["device_span_ms"] * 1e3,
                 "launches": r["launches"], "bound": "launch latency (8 KiB of data)"}

    # C2: 16-chain over 256 tiles; 64 MiB fits the 126 MB L2 -> flushed before each rep
    p = W.c2_chain()
    nbytes, fmul = algorithmic(p)
    fused, _ = _run(torch, B, p, reps, flush=flush)
    unfused, _ = _run(torch, B, p, reps, flush=flush, flags=B.BT_FLAG_NO_FUSION)
    compulsory = 8.0 * p.buffers[0].shape[0]
    out["C2"] = {"workload": p.name, "l2": "512 MiB buffer read before each rep (clean L2)",
                 "fused": {"device_ms": fused["device_span_ms"], "wall_ms": fused["wall_ms"],
                           "compulsory_GBps": compulsory / (fused["device_span_ms"] * 1e-3) / 1e9,
                           "frac_of_measured_hbm": compulsory / (fused["device_span_ms"] * 1e-3) / 1e9 / hbm,
                           "effective_task_GBps": nbytes / (fused["device_span_ms"] * 1e-3) / 1e9,
                           "items": fused["items"], "launches": fused["launches"]},
                 "unfused": {"device_ms": unfused["device_span_ms"], "wall_ms": unfused["wall_ms"],
                             "effective_task_GBps": nbytes / (unfused["device_span_ms"] * 1e-3) / 1e9,
                             "frac_of_measured_hbm": nbytes / (unfused["device_span_ms"] * 1e-3) / 1e9 / hbm,
                             "items": unfused["items"], "edges": unfused["edges"]}}

    # C3: random DAG, 10,000 tasks over 64 x 4 MiB (256 MiB > L2)
    p = W.c3_random_dag()
    nbytes, fmul = algorithmic(p)
    r, _ = _run(torch, B, p, max(3, reps // 2))
    t_roof = max(nbytes / (hbm * 1e9), fmul / fmul_peak) * 1e3
    out["C3"] = {"workload": p.name, "device_ms": r["device_span_ms"], "wall_ms": r["wall_ms"],
                 "host_build_ms": r["host_build_ms"],
                 "tasks_per_s_device": p.ntasks / (r["device_span_ms"] * 1e-3),
                 "tasks_per_s_e2e": p.ntasks / (r["wall_ms"] * 1e-3),
                 "effective_task_GBps": nbytes / (r["device_span_ms"] * 1e-3) / 1e9,
                 "roofline_ms": t_roof, "roofline_frac": t_roof / r["device_span_ms"],
                 "items": r["items"], "edges": r["edges"]}
    del p

    # C4: 1M tasks on 4 KiB tiles (64 MB: L2-resident between reps unless flushed)
    p = W.c4_fine()
    nbytes, _ = algorithmic(p)
    t_roof = nbytes / (hbm * 1e9) * 1e3
    c4 = {"workload": p.name, "hbm_roofline_ms": t_roof, "l2": "512 MiB buffer read before each rep (clean L2)"}
    for name, flags in (("unfused", B.BT_FLAG_NO_FUSION), ("fused", 0)):
        r, _ = _run(torch, B, p, reps, flush=flush, flags=flags)
        c4[name] = {"device_ms": r["device_span_ms"], "wall_ms": r["wall_ms"], "host_build_ms": r["host_build_ms"],
                    "device_ns_per_task": r["device_span_ms"] * 1e6 / p.ntasks,
                    "tasks_per_s_device": p.ntasks / (r["device_span_ms"] * 1e-3),
                    "tasks_per_s_e2e": p.ntasks / (r["wall_ms"] * 1e-3),
                    "overhead_ns_per_task_vs_hbm": (r["device_span_ms"] - t_roof) * 1e6 / p.ntasks,
                    "items": r["items"], "epochs": r["epochs"]}
    # in-kernel pop / release per unit (C4 unfused, BT_FLAG_TIMESTAMPS; continuations off while tracing)
    r, tr = _run(torch, B, p, 1, flush=flush, flags=B.BT_FLAG_NO_FUSION | B.BT_FLAG_TIMESTAMPS)
    if tr is not None:
        t, _ = tr
        ns = 1e3 / peaks.get("sm_max_mhz", 1965.0)
        c4["trace"] = {"units": int(t.shape[0]), "clock_mhz_assumed": peaks.get("sm_max_mhz", 1965.0),
                       "pop_ns_median": float(np.median(t[:, 1]) * ns), "pop_ns_p99": float(np.percentile(t[:, 1], 99) * ns),
                       "body_ns_median": float(np.median(t[:, 2]) * ns),
                       "release_ns_median": float(np.median(t[:, 3]) * ns),
                       "release_ns_p99": float(np.percentile(t[:, 3], 99) * ns),
                       "traced_device_ms": r["device_span_ms"]}
    del p
    # dependency latency: a 1-wide chain of 10,000 SCALs on one 4 KiB tile
    x = np.ones(1024, np.float32)
    fch = W.sweep_factors(np.random.default_rng(3), 10000)
    pch = W.sweep_program(1024, 1, fch, x, name="1-wide chain of 10,000 on one 4 KiB tile")
    r, _ = _run(torch, B, pch, 3, flags=B.BT_FLAG_NO_FUSION)
    c4["chain_10000"] = {"device_ms": r["device_span_ms"], "us_per_link": r["device_span_ms"] * 1e3 / 10000}
    # C4b: 1M independent 4 KiB tiles x 1 task (pure pop rate; 4 GiB)
    if not quick:
        nt = 1 << 20
        xb = np.ones(nt * 1024, np.float32)
        pb = W.sweep_program(nt * 1024, nt, np.array([0.5], np.float32), xb, name="C4b")
        r, _ = _run(torch, B, pb, 3)
        tb = 8.0 * 1024 * nt / (hbm * 1e9) * 1e3
        c4["C4b_independent"] = {"device_ms": r["device_span_ms"], "device_ns_per_task": r["device_span_ms"] * 1e6 / nt,
                                 "hbm_roofline_ms": tb, "frac_of_measured_hbm": tb / r["device_span_ms"]}
        del xb, pb
    out["C4"] = c4
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    print(json.dumps(run_all(0, quick="--quick" in sys.argv)), flush=True)
