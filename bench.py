#!/usr/bin/env python
"""Benchmark of the task-stream hot path (BASELINE.json metric on config C5).

A step = one pass of the whole path over one batch of synthetic input:
submit the C5 task stream (64 chained vector_scal sweeps over 16,384 tiles of
a 4 GiB float32 vector; this rank's owner-computes share) through
bt_insert_task_batch -> dependency inference + chain fusion -> pack + upload
-> persistent scheduler kernel -> bt_task_wait_for_all.  Inputs are resident
in HBM before the timed region (registered once, device-homed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

Prints ONE JSON line on rank 0.  See DESIGN.md section "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "vector_scal effective HBM GB/s (frac of 8 TB/s) and tasks/s at 1/2/4/8 B200"
NOMINAL_HBM_GBPS = 8000.0
FP32_LANES_PER_SM = 128

C5 = dict(nx=1 << 30, ntiles=16384, sweeps=64)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def workload_name(cfg, world=1, scaling="weak"):
    base = (f"C5: {cfg['nx']} float32 ({cfg['nx'] * 4 / 2**30:.0f} GiB), {cfg['ntiles']} tiles x "
            f"{cfg['nx'] // cfg['ntiles']}, {cfg['sweeps']} chained vector_scal sweeps (sweep-major), "
            f"owner-computes tiles")
    if world == 1:
        return base
    if scaling == "weak":
        return base + f"; weak scaling: one such 4 GiB shard per GPU ({world} x 4 GiB in total)"
    return base + f"; strong scaling: the 4 GiB vector's tiles split over {world} GPUs"


class ClockSampler:
    """NVML clocks + throttle reasons sampled in a thread during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


def synth_tile_values(torch, n, seed, device):
    """x in [1,2): 23 random mantissa bits (same recipe as workloads.unit_interval_floats)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    bits = torch.randint(0, 1 << 23, (n,), dtype=torch.int32, device=device, generator=g) | 0x3F800000
    return bits.view(torch.float32)


def rank_tasks(np, handles, factors):
    """This rank's task stream, sweep-major: for s: for t in my tiles: SCAL(f_s; t)."""
    nt, ns = len(handles), len(factors)
    codelets = np.full(nt * ns, 1, np.int32)
    scalars = np.repeat(factors.astype(np.float32), nt)
    h0 = np.tile(np.asarray(handles, np.uint64), ns)
    return codelets, scalars, h0


def run_reference(args):
    """--impl reference: the sequential C oracle, timed on this host's cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    import oracle
    import workloads as W
    cfg = dict(C5)
    tile = cfg["nx"] // cfg["ntiles"]
    sample_tiles = args.ref_tiles
    rng = np.random.default_rng(W.SEED_BASE + 4)
    f = W.sweep_factors(rng, cfg["sweeps"])
    x = W.unit_interval_floats(np.random.default_rng(1), sample_tiles * tile)
    p = W.sweep_program(x.shape[0], sample_tiles, f, x)
    off0, len0, off1, len1 = oracle.model.resolve(p)
    t = p.tasks
    bufs = [x]

    def step():
        oracle.run_tasks(bufs, t["codelet"], t["scalar"], t["b0"], off0, len0, t["b1"], off1, len1)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    elems = sample_tiles * tile
    value = 8.0 * elems / dt / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "tasks_per_s": sample_tiles * cfg["sweeps"] / dt,
            "config": {"workload": workload_name(cfg, args.gpus, args.scaling),
                       "sample": f"{sample_tiles} of {cfg['ntiles']} tiles, "
                       f"all {cfg['sweeps']} sweeps, task-major"},
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": f"{sample_tiles} tiles x {tile} floats x {cfg['sweeps']} sweeps "
                                       f"({sample_tiles * cfg['sweeps']} tasks) per step"},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(np, seconds_target=12.0, threads=0):
    """The oracle as it stands on a bounded sample of C5: single-threaded pinned
    to one core (threads = 0, the oracle's definition: submission order), or its
    OpenMP variant (element-parallel inside each task) on `threads` cores."""
    import oracle
    import workloads as W
    tile = C5["nx"] // C5["ntiles"]
    rng = np.random.default_rng(W.SEED_BASE + 4)
    f = W.sweep_factors(rng, C5["sweeps"])
    ntile = 64 if threads <= 1 else 512
    x = W.unit_interval_floats(np.random.default_rng(2), ntile * tile)
    p = W.sweep_program(x.shape[0], ntile, f, x)
    off0, len0, off1, len1 = oracle.model.resolve(p)
    t = p.tasks
    old_aff = os.sched_getaffinity(0)
    core = min(old_aff)
    if threads <= 1:
        os.sched_setaffinity(0, {core})
    try:
        reps, t0 = 0, time.perf_counter()
        while True:
            oracle.run_tasks([x], t["codelet"], t["scalar"], t["b0"], off0, len0, t["b1"], off1, len1,
                             threads=threads if threads > 1 else 0)
            reps += 1
            if time.perf_counter() - t0 > seconds_target:
                break
        dt = time.perf_counter() - t0
    finally:
        os.sched_setaffinity(0, old_aff)
    cpu = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            cpu = next(l.split(":", 1)[1].strip() for l in fh if l.startswith("model name"))
    except Exception:
        pass
    how = (f"single-threaded pinned to core {core}" if threads <= 1 else
           f"OpenMP variant (oracle_run_omp: tasks in order, each task's elements split over {threads} threads)")
    return {"value": 8.0 * ntile * tile * reps / dt / 1e9, "unit": "GB/s", "cores": max(1, threads),
            "kind": "oracle" if threads <= 1 else "oracle_openmp",
            "sample": f"{reps} x ({ntile} tiles x {tile} floats x {C5['sweeps']} sweeps, task-major), "
                      f"{dt:.1f} s {how}",
            "host": {"cpu": cpu, "nproc": os.cpu_count()},
            "tasks_per_s": reps * ntile * C5["sweeps"] / dt}


def sm_count(torch, dev):
    """Streaming multiprocessors of this GPU, queried (148 on B200)."""
    return torch.cuda.get_device_properties(dev).multi_processor_count


def builder_threads(args):
    """Dependency-builder threads per rank: the node's cores shared among its
    ranks (one left per rank for the CUDA driver / caller), at least 2, at most 16."""
    if args.host_threads:
        return args.host_threads
    lw = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    cores = os.cpu_count() or 2
    return max(2, min(16, cores // lw - (2 if lw == 1 else 1)))


def timed_steps(torch, dev, stream, dist, rt, tasks, steps, warmup):
    """warmup untimed steps, then `steps` timed ones (barrier + synchronize on
    both sides, CUDA events on the runtime's stream).  A step = submit the
    batch (dependency inference, fusion, pack, upload, kernels) + wait."""
    codelets, scalars, h0 = tasks
    for _ in range(warmup):
        rt.insert_batch(codelets, scalars, h0)
        rt.wait()
    rt.stats_reset()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        rt.insert_batch(codelets, scalars, h0)
        rt.wait()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    return ev0.elapsed_time(ev1) / steps, rt.stats()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-fusion", action="store_true", help="unfused (scheduler-bound) variant")
    ap.add_argument("--no-stream", action="store_true",
                    help="one launch per pipelined round instead of one stream launch per step (comparison)")
    ap.add_argument("--sweeps", type=int, default=C5["sweeps"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--configs", type=int, default=1,
                    help="N = 1: also report the other BASELINE configs C1-C4 (secondary keys, tools/bench_configs.py)")
    ap.add_argument("--ref-tiles", type=int, default=64)
    ap.add_argument("--chunk-bytes", type=int, default=0, help="fixed work-unit size (0 = adaptive)")
    ap.add_argument("--host-threads", type=int, default=0)
    ap.add_argument("--rounds", type=int, default=0, help="pipelined rounds per SCAL run (0 = library default)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong",
                    help="N > 1: strong = ONE 4 GiB vector whose tiles are block-distributed over the ranks "
                         "(bt_data_distribute_block; every rank submits every task, each runs its own: default, "
                         "BASELINE configs[4]); weak = a full 4 GiB C5 per GPU")
    ap.add_argument("--secondary-scaling", type=int, default=1,
                    help="N > 1: also time the other scaling mode (secondary key)")
    ap.add_argument("--hbm-variant", type=int, default=1,
                    help="also time the HBM-bound 16-sweep variant on the same tiles (secondary key)")
    ap.add_argument("--streamed", type=int, default=1,
                    help="also time the K steps submitted back to back with one wait (diagnostic key)")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="diagnostic (N = 1): rank 0 of an N-rank strong-scaling job alone on this GPU "
                         "(its line is not a bench result)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # one rank per GPU; BT_BENCH_BACKEND=gloo lets a 1-GPU box run the N>1
    # code path (ranks share the GPU; their kernels never wait on each other)
    backend = os.environ.get("BT_BENCH_BACKEND", "nccl")
    local_dev = local % torch.cuda.device_count()
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def allreduce_max(vals, op="max"):
        t = torch.tensor(vals, dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        if dist:
            dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return t.tolist()

    from paper_1304_0878_b200 import btask as B
    import workloads as W

    cfg = dict(C5, sweeps=args.sweeps)
    T, S = cfg["ntiles"], cfg["sweeps"]
    tile = cfg["nx"] // T
    factors = W.sweep_factors(np.random.default_rng(W.SEED_BASE + 4), S)
    stream = torch.cuda.current_stream(dev)
    flags = (B.BT_FLAG_NO_FUSION if args.no_fusion else 0) | (B.BT_FLAG_NO_STREAM if args.no_stream else 0)
    threads = builder_threads(args)
    emulate = args.emulate_ranks if (args.emulate_ranks and world == 1) else 0

    def make_run(mode):
        """Runtime + registered, partitioned device-resident C5 input + this rank's task stream.
        strong: every rank registers the whole vector (a 4 GiB allocation per GPU, of which it
        writes its block of tiles), partitions it into T tiles, block-distributes them over the
        ranks (bt_data_distribute_block) and submits every task of the
        stream; the library's rank filter runs the local ones.  weak: a full C5 per rank."""
        nranks = (emulate or world) if mode == "strong" else 1
        myrank = 0 if mode == "weak" else rank
        rt = B.Runtime(device=local_dev, stream=stream.cuda_stream, rank=myrank, nranks=nranks, flags=flags,
                       chunk_bytes=args.chunk_bytes, host_threads=threads, pipeline_rounds=args.rounds)
        x = synth_tile_values(torch, cfg["nx"], 1000 + (rank if mode == "weak" else 0), dev)
        h = rt.register_tensor(x)
        subs = rt.partition(h, T)
        if nranks > 1:
            rt.distribute_block(h)
        lo, hi = myrank * T // nranks, (myrank + 1) * T // nranks
        return rt, x, h, subs, (hi - lo) * tile, rank_tasks(np, subs, factors)

    def close_run(rt, x, h):
        rt.unpartition(h)
        rt.unregister(h)
        rt.close()

    mode = args.scaling if world > 1 or emulate else "strong"
    rt, x, h, subs, elems, tasks = make_run(mode)
    ntasks = tasks[0].shape[0]                      # tasks every rank submits
    with ClockSampler(local_dev) as clk:
        ms, st = timed_steps(torch, dev, stream, dist, rt, tasks, args.steps, args.warmup)
    launches_per_step = st["sched_launches"] / args.steps          # scheduler-kernel launches
    epochs_per_step = st["epochs"] / args.steps                    # rounds (sub-epochs of a stream launch)
    kern_ms = st["device_ms"] / max(1, st["sched_launches"])       # average launch duration
    span_ms = st["device_span_ms"] / args.steps                    # device time per step (launches overlap)
    host_ms = st["host_build_ms"] / args.steps
    local_tasks = st["tasks_local"] / args.steps
    ms, kern_ms_max, host_ms_max, span_ms_max = allreduce_max([ms, kern_ms, host_ms, span_ms])
    launches_all = int(allreduce_max([float(st["kernel_launches"])], op="sum")[0])   # every rank's kernels

    # ---- streamed (diagnostic, not the headline): the same K steps submitted
    # back to back and waited for once (bt_insert_task_batch is asynchronous:
    # the host builds step i+1 while the device runs step i; every task of
    # every step still executes, ordered by the inferred dependencies)
    streamed_ms = None
    if args.streamed:
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        es0, es1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        es0.record(stream)
        for _ in range(args.steps):
            rt.insert_batch(*tasks)
        rt.wait()
        es1.record(stream)
        torch.cuda.synchronize(dev)
        streamed_ms = allreduce_max([es0.elapsed_time(es1) / args.steps])[0]

    # ---- HBM-bound variant (secondary key): the same tiles, 16 chained sweeps
    # per step (C5-16; fused k = 16 is below the FP32/HBM ridge of ~46), where
    # the north_star's ">= 85 % of HBM bandwidth" is graded
    hbm16 = None
    if args.hbm_variant and S > 16 and not args.no_fusion:
        t16 = rank_tasks(np, subs, factors[:16])
        k16 = max(10, args.steps)
        ms16, st16 = timed_steps(torch, dev, stream, dist, rt, t16, k16, 3)
        hbm16 = allreduce_max([ms16, st16["device_span_ms"] / k16,
                               st16["device_ms"] / max(1, st16["sched_launches"])]) + [k16, st16["sched_launches"] / k16]
    close_run(rt, x, h)
    del x
    torch.cuda.empty_cache()

    # ---- the other scaling mode (N > 1, secondary key)
    other = None
    if world > 1 and args.secondary_scaling:
        omode = "weak" if mode == "strong" else "strong"
        rt2, x2, h2, _, elems2, tasks2 = make_run(omode)
        ms2, st2 = timed_steps(torch, dev, stream, dist, rt2, tasks2, args.steps, args.warmup)
        ms2 = allreduce_max([ms2])[0]
        close_run(rt2, x2, h2)
        del x2
        torch.cuda.empty_cache()
        tot2 = cfg["nx"] * (world if omode == "weak" else 1)
        other = {"scaling": omode, "ms_per_step": ms2, "value": 8.0 * tot2 / (ms2 * 1e-3) / 1e9, "unit": "GB/s",
                 "workload": workload_name(cfg, world, omode)}

    # ---- e2e: host (pinned) buffers through the public API, copies inside the region
    # (this rank's block of the vector: owner-computes, each rank uploads and
    # writes back the tiles it owns)
    e2e_ms = None
    h2d = d2h = 0
    if args.e2e_steps > 0:
        my_tiles = elems // tile
        rt = B.Runtime(device=local_dev, stream=stream.cuda_stream, flags=flags, chunk_bytes=args.chunk_bytes,
                       host_threads=threads, pipeline_rounds=args.rounds)
        addr, host = B.pinned_empty(elems * 4)
        host[:] = synth_tile_values(torch, elems, 2000 + rank, dev).cpu().numpy()
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()

        def e2e_step():
            he = rt.register(addr, elems, 0)
            se = rt.partition(he, my_tiles)
            c2, s2, g2 = rank_tasks(np, se, factors)
            rt.insert_batch(c2, s2, g2)
            rt.wait()
            rt.unpartition(he)
            rt.unregister(he)                 # device -> host copy of the result

        e2e_step()                            # untimed: replica + epoch buffer allocation
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        rt.stats_reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = e0.elapsed_time(e1) / args.e2e_steps
        st2 = rt.stats()
        h2d = elems * 4 + st2["upload_bytes"] // args.e2e_steps
        d2h = elems * 4 + 64
        e2e_ms = allreduce_max([e2e_ms])[0]
        h2d, d2h = allreduce_max([float(h2d), float(d2h)], op="sum")
        B.bt_free(addr)
        rt.close()

    configs = None
    if world == 1 and not emulate and args.configs:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import bench_configs
        configs = bench_configs.run_all(local_dev)

    if rank == 0:
        peaks, peak_src = load_peaks()
        sms = sm_count(torch, local_dev)
        total_elems = cfg["nx"] * (world if mode == "weak" else 1) * 1.0
        compulsory = 8.0 * total_elems                     # read + write each element once per step
        value = compulsory / (ms * 1e-3) / 1e9
        clocks = clk.summary()
        # roofline of the dominant kernel (the persistent scheduler kernel; a step is one
        # stream launch whose sub-epochs are the pipelined rounds, or with --no-stream one
        # launch per round on two streams):
        # fused chain of S multiplies per element -> FP32-multiply bound when S exceeds the ridge.
        # achieved = algorithmic work per launch / the kernel's average launch duration (CUDA
        # events recorded around each launch on its own stream); adjacent rounds' launches
        # overlap by their tails, so the per-launch share of the step's device span
        # (first launch start -> last launch end) is reported beside it.
        per_launch_elems = elems / launches_per_step
        fmul = per_launch_elems * S
        avg_launch = st["device_ms"] / max(1, st["sched_launches"])
        share_ms = span_ms / launches_per_step
        alu_peak = sms * FP32_LANES_PER_SM * (peaks.get("sm_max_mhz") or 1965.0) * 1e6 / 1e12
        hbm_bytes = 8.0 * per_launch_elems
        t_alu = fmul / (alu_peak * 1e12)
        t_hbm = hbm_bytes / (peaks["hbm_gbs"] * 1e9)
        fused = not args.no_fusion
        if fused and t_alu > t_hbm:
            work, scale = fmul, 1e12
            roof = {"bound": "alu", "peak": alu_peak,
                    "unit": "TFMUL/s", "peak_source": f"{sms} SMs (queried) x {FP32_LANES_PER_SM} FP32 lanes x "
                                                     f"{peaks.get('sm_max_mhz')} MHz (DESIGN.md); FMUL microbenchmark "
                                                     f"36.3 T/s (profiles/r02_probe_b200.jsonl)"}
        else:
            work, scale = (hbm_bytes if fused else 8.0 * per_launch_elems * S), 1e9
            roof = {"bound": "hbm", "peak": peaks["hbm_gbs"],
                    "unit": "GB/s", "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})"}
        roof["achieved"] = work / (avg_launch * 1e-3) / scale
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof["kernel"] = ("bt::scheduler_kernel_sws (stream launch: the step's rounds are sub-epochs of one launch)"
                          if launches_per_step < epochs_per_step else "bt::scheduler_kernel_sw")
        roof["avg_launch_ms"] = avg_launch
        roof["work_per_launch"] = work
        roof["launches_per_step"] = launches_per_step
        roof["epochs_per_step"] = epochs_per_step
        roof["stream_closes"] = int(st.get("stream_closes", 0))     # stream launches ended early (expected 0)
        roof["stream_resumes"] = int(st.get("stream_resumes", 0))   # closed for want of publications (expected 0)
        roof["device_span_ms_per_step"] = span_ms
        roof["span_share_ms"] = share_ms
        roof["achieved_span_share"] = work / (share_ms * 1e-3) / scale
        roof["frac_span_share"] = roof["achieved_span_share"] / roof["peak"]
        roof["frac_step"] = work * launches_per_step / (ms * 1e-3) / scale / roof["peak"]
        roof["hbm_GBps_physical"] = hbm_bytes / (avg_launch * 1e-3) / 1e9
        roof["traffic"] = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
                tr = json.load(fh).get("c5_fused" if fused else "c5_unfused")
                if tr and tr.get("elems_per_launch") == per_launch_elems:
                    roof["traffic"] = tr["dram_bytes_per_launch"]
        except OSError:
            pass
        if emulate:
            # rank 0's share of an N-rank strong-scaling run: its own time only (not a bench line)
            print(json.dumps({"diagnostic": "emulated rank 0 of N (strong scaling)", "N": emulate,
                              "ms_per_step": ms, "streamed_ms_per_step": streamed_ms,
                              "host_build_ms_per_step": host_ms_max, "device_ms_per_step": span_ms_max,
                              "avg_launch_ms": avg_launch, "elements": elems, "tasks_submitted_per_step": ntasks,
                              "tasks_local_per_step": local_tasks, "builder_threads": threads}), flush=True)
            return 0
        job_tasks = ntasks * world if mode == "weak" else ntasks
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": mode,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "frac_of_8TBps": value / (NOMINAL_HBM_GBPS * world),
            "frac_of_measured_hbm": value / (peaks["hbm_gbs"] * world),
            "tasks_per_s": job_tasks / (ms * 1e-3),
            "effective_unfused_GBps": 8.0 * total_elems * S / (ms * 1e-3) / 1e9,
            "host_build_ms_per_step": host_ms_max, "device_ms_per_step": span_ms_max,
            "config": {"workload": workload_name(cfg, world, mode), "tasks_per_step": job_tasks,
                       "tasks_submitted_per_rank": ntasks, "builder_threads": threads,
                       "fusion": fused, "parallelism": (f"owner-computes: bt_data_distribute_block over {world} "
                                                        f"rank(s), rank filter" if mode == "strong" else
                                                        f"{world} independent C5 shards"),
                       "l2": "4 GiB working set > 126 MB L2 (no flush needed)"},
            "gpu_launches": launches_all,
            "clocks": clocks,
            "roofline": roof,
        }
        if hbm16 is not None:
            ms16, span16, launch16, k16, lps16 = hbm16
            kern16 = compulsory / (span16 * 1e-3) / 1e9           # all ranks' bytes / slowest rank's device time
            line["hbm_bound_variant"] = {
                "workload": "C5-16: same 4 GiB and tiles, 16 chained sweeps per step (fused k = 16: HBM-bound)",
                "steps": int(k16), "ms_per_step": ms16, "value": compulsory / (ms16 * 1e-3) / 1e9, "unit": "GB/s",
                "device_span_ms_per_step": span16, "launches_per_step": lps16, "avg_launch_ms": launch16,
                "kernel_GBps": kern16, "frac_of_measured_hbm": kern16 / (peaks["hbm_gbs"] * world),
                "frac_of_8TBps": kern16 / (NOMINAL_HBM_GBPS * world)}
        if streamed_ms is not None:
            line["streamed"] = {"value": compulsory / (streamed_ms * 1e-3) / 1e9, "unit": "GB/s",
                                "ms_per_step": streamed_ms,
                                "note": "diagnostic: K steps submitted back to back, one wait (host build of "
                                        "step i+1 overlaps device step i); the headline waits every step"}
        if other is not None:
            line["other_scaling"] = other
        if e2e_ms is not None:
            e2e_bytes = 8.0 * elems * world                   # every rank's block in and out
            line["e2e"] = {"value": e2e_bytes / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
                           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                           "ms_per_step": e2e_ms, "path": "bt_malloc pinned host buffer (this rank's block) -> "
                           "register (H2D) -> partition -> insert_task_batch -> wait -> unregister (D2H)"}
        if configs is not None:
            line["configs"] = configs
        if world == 1 and not args.skip_cpu:
            line["cpu_baseline"] = cpu_baseline(np)
            line["cpu_baseline_openmp"] = cpu_baseline(np, threads=os.cpu_count() or 1)
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
