"""Long randomized parity stress on the GPU (test infrastructure: uses oracle/).

Random programs (random_small_program shapes, C3-style DAGs with partitions,
unfused chains) under random runtime configurations and every scheduler
variant (BT_FLAG_KERNEL_*), each compared bit for bit with the oracle.  Runs
for --minutes; prints one JSON line per 50 programs and a summary; exits 1 on
the first mismatch (with the seed to reproduce it).

    python tools/stress.py --minutes 10
    python tools/stress.py --minutes 10 --device   # device-homed buffers: stream launches,
                                                   # 1-3 submissions back to back per wait
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402
from paper_1304_0878_b200 import btask as B  # noqa: E402
from paper_1304_0878_b200.programs import run_program  # noqa: E402

KERNELS = [0, B.BT_FLAG_KERNEL_SW, B.BT_FLAG_KERNEL_RW, B.BT_FLAG_KERNEL_WQ]


def run_device(p, repeats, **kw):
    """Device-homed buffers (torch tensors); p submitted `repeats` times, one wait."""
    import torch
    from paper_1304_0878_b200.programs import Session
    tensors = [torch.from_numpy(b.copy()).cuda() for b in p.buffers]
    with B.Runtime(**kw) as rt:
        s = Session(rt, p, device_tensors=tensors)
        for _ in range(repeats):
            s.submit()
        rt.wait()
        st = rt.stats()
        s.finish()
    torch.cuda.synchronize()
    return [t.cpu().numpy() for t in tensors], st


def make(seed, device=False):
    rng = np.random.default_rng(seed)
    shape = int(rng.integers(0, 3)) if not device else int(rng.choice([0, 1, 2, 2, 2]))
    if shape == 0:
        p = W.random_small_program(seed, max_tasks=int(rng.integers(5, 200)), max_handles=int(rng.integers(1, 8)),
                                   max_elems=int(rng.integers(8, 50000)))
    elif shape == 1:
        p = W.c3_random_dag(nbuf=int(rng.integers(2, 12)), nx=int(rng.integers(1, 40000)),
                            ntasks=int(rng.integers(1, 600)), seed=seed)
    else:
        p = W.c4_fine(ntiles=int(rng.integers(1, 400)),
                      tile_nx=int(rng.integers(1, 3000) if not device else rng.choice([rng.integers(1, 3000),
                                                                                       rng.integers(4097, 20000)])),
                      sweeps=int(rng.integers(1, 40)), seed=seed,
                      order="sweep" if rng.random() < 0.5 else "tile")
    kw = dict(chunk_bytes=int(rng.choice([0, 0, 32, 96, 4096, 65536])),
              flags=(0 if rng.random() < 0.6 else B.BT_FLAG_NO_FUSION) | int(rng.choice(KERNELS)) |
              (B.BT_FLAG_PRIORITY if rng.random() < 0.3 else 0),
              host_threads=int(rng.integers(1, 6)), parallel_min=int(rng.integers(1, 64)),
              pipeline_min=int(rng.integers(1, 64)), pipeline_rounds=int(rng.integers(1, 5)),
              max_fused=int(rng.choice([0, 1, 3, 7, 64, 1024])),
              epoch_tasks=int(rng.choice([0, 0, 0, 5, 37])))
    if device:
        kw["pipeline_rounds"] = int(rng.integers(1, 11))
    return p, kw


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--minutes", type=float, default=10.0)
    ap.add_argument("--seed0", type=int, default=700000)
    ap.add_argument("--device", action="store_true", help="device-homed buffers (stream launches)")
    ap.add_argument("--count", type=int, default=0, help="stop after this many programs (0: --minutes only)")
    ap.add_argument("--extra-flags", type=int, default=0, help="OR-ed into every configuration's flags")
    args = ap.parse_args()
    streams = resumes = 0
    t_end = time.time() + 60 * args.minutes
    seed, n, tasks = args.seed0, 0, 0
    while time.time() < t_end and (not args.count or n < args.count):
        p, kw = make(seed, args.device)
        kw["flags"] |= args.extra_flags
        if args.device:
            reps = int(np.random.default_rng(seed + 1).integers(1, 4))
            try:
                t0 = time.time()
                out, st = run_device(p, reps, **kw)
                if os.environ.get("BT_STRESS_VERBOSE"):
                    print(json.dumps({"seed": seed, "s": round(time.time() - t0, 3), "epochs": st["epochs"],
                                      "sched_launches": st["sched_launches"]}), flush=True)
                import torch
                torch.cuda.synchronize()   # a sticky device fault surfaces at the program that caused it
            except Exception as ex:
                print(json.dumps({"error": str(ex), "seed": seed, "program": p.name, "repeats": reps,
                                  "config": {k: int(v) for k, v in kw.items()}}), flush=True)
                return 1
            streams += st["sched_launches"] < st["epochs"]
            resumes += st.get("stream_resumes", 0)
            p = W.Program(p.buffers, p.nparts, np.concatenate([p.tasks] * reps), name=p.name)
        else:
            out, st = run_program(p, device=0, **kw)
        exp = oracle.run(p)
        for b, (o, e) in enumerate(zip(out, exp)):
            if not np.array_equal(o.view(np.uint32), e.view(np.uint32)):
                bad = int(np.count_nonzero(o.view(np.uint32) != e.view(np.uint32)))
                print(json.dumps({"mismatch": True, "seed": seed, "program": p.name, "buffer": b, "elements": bad,
                                  "config": {k: int(v) for k, v in kw.items()}}), flush=True)
                return 1
        n += 1
        tasks += p.ntasks
        if n % 50 == 0:
            print(json.dumps({"programs": n, "tasks": tasks, "last_seed": seed, "with_stream_launch": streams}),
                  flush=True)
        seed += 1
    print(json.dumps({"ok": True, "programs": n, "tasks": tasks, "seeds": [args.seed0, seed - 1],
                      "device_homed": args.device, "with_stream_launch": streams, "stream_resumes": resumes,
                      "env": {k: v for k, v in os.environ.items() if k.startswith("BT_")}}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
