"""Cross-rank reads (bt_comm_init): worker processes.

Each worker is one rank (its own process and runtime) on cuda:0 -- ranks
sharing one GPU is safe here because no kernel waits for another rank: the
rendezvous orders streams with interprocess events only (comm.hpp).  Every
rank registers every buffer, sets the same owners, submits the whole program
and returns the data it owns; the caller compares that with the oracle.
"""
from __future__ import annotations

import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def owners_of(program, nranks: int, seed: int) -> list:
    """Owner rank of every leaf: owners[b] is an int (unpartitioned) or a list per tile."""
    import numpy as np
    rng = np.random.default_rng(seed)
    out = []
    for b, nparts in enumerate(program.nparts):
        if nparts:
            out.append([int(r) for r in rng.integers(0, nranks, nparts)])
        else:
            out.append(int(rng.integers(0, nranks)))
    return out


def leaf_ranges(program, b: int):
    """[(tile or -1, offset, length)] of buffer b's leaves."""
    from oracle.model import tile_range
    nx = len(program.buffers[b])
    if not program.nparts[b]:
        return [(-1, 0, nx)]
    return [(t, *tile_range(nx, program.nparts[b], t)) for t in range(program.nparts[b])]


def worker(rank: int, nranks: int, name: str, program, owners, batch: bool, barrier, q, flags: int = 0,
           rt_kwargs=None, gate=None, lib_path=None):
    try:
        sys.path.insert(0, ROOT)
        if lib_path:   # a test-sensitivity build of the library (tests/test_gpu.py mutants)
            os.environ["BT_LIB_PATH"] = lib_path
        import time
        import numpy as np
        import torch
        from paper_1304_0878_b200 import btask as B
        from paper_1304_0878_b200.programs import Session
        torch.cuda.set_device(0)
        tensors = [torch.from_numpy(b.copy()).cuda() for b in program.buffers]
        torch.cuda.synchronize()
        rt = B.Runtime(rank=rank, nranks=nranks, flags=flags, **(rt_kwargs or {}))
        rt.comm_init(name)
        s = Session(rt, program, device_tensors=tensors)
        for b, own in enumerate(owners):
            if isinstance(own, list):
                for t, r in enumerate(own):
                    rt.set_rank(s.subs[b][t], r)
            else:
                rt.set_rank(s.roots[b], own)
        # gate = (rank, seconds): that rank's stream is held (bt_debug_gate)
        # from before its first task until `seconds` after its submission
        release = rt.debug_gate() if gate and gate[0] == rank else None
        s.submit(batch=batch)
        if release:
            time.sleep(gate[1])
            release()
        rt.wait()
        torch.cuda.synchronize()
        mine = {}
        for b, own in enumerate(owners):
            host = tensors[b].cpu().numpy()
            for t, off, n in leaf_ranges(program, b):
                r = own[t] if isinstance(own, list) else own
                if r == rank:
                    mine[(b, t)] = host[off:off + n].copy()
        stats = rt.stats()
        barrier.wait(timeout=120)      # every rank's copies done before anyone frees memory
        s.finish()
        rt.close()
        q.put((rank, mine, stats, None))
    except Exception:   # report, do not hang the parent
        q.put((rank, None, None, traceback.format_exc()))


def run(program, nranks: int = 2, seed: int = 0, batch: bool = True, timeout: float = 240.0, owners=None,
        flags: int = 0, rt_kwargs=None, gate=None, lib_path=None):
    """Run `program` on nranks processes; returns ({(b, tile): owned data}, [stats per rank], owners)."""
    import multiprocessing as mp
    import uuid
    ctx = mp.get_context("spawn")
    if owners is None:
        owners = owners_of(program, nranks, seed)
    name = f"/bt-test-{os.getpid()}-{uuid.uuid4().hex[:8]}"
    q = ctx.Queue()
    barrier = ctx.Barrier(nranks)
    procs = [ctx.Process(target=worker, args=(r, nranks, name, program, owners, batch, barrier, q, flags, rt_kwargs, gate,
                                                  lib_path))
             for r in range(nranks)]
    for p in procs:
        p.start()
    results, stats, errors = {}, [None] * nranks, []
    try:
        for _ in range(nranks):
            rank, mine, st, err = q.get(timeout=timeout)
            if err:
                errors.append(f"rank {rank}:\n{err}")
                continue
            results.update(mine)
            stats[rank] = st
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    if errors:
        raise RuntimeError("\n".join(errors))
    return results, stats, owners
