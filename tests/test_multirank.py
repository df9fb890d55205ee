"""Owner-computes across ranks on CPU (gloo, world_size 2): every rank submits
the same program (the StarPU-MPI model); each task runs
only on the rank owning its written operand.  The ranks' local task sets must
partition the program, and each local DAG must order every conflicting pair
of its own tasks."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _program(seed):
    rng = np.random.default_rng(seed)
    nbuf, nparts, n = 2, 8, 64
    bufs = [W.unit_interval_floats(rng, n) for _ in range(nbuf)]
    rows = []
    for _ in range(120):
        kind = rng.integers(0, 3)
        b = int(rng.integers(0, nbuf))
        t = int(rng.integers(0, nparts))
        if kind == 0:
            rows.append((W.SCAL, np.float32(rng.uniform(0.5, 2)), b, t, -1, -1))
        else:  # AXPY/COPY between the same tile index of both buffers: same owner
            rows.append((W.AXPY if kind == 1 else W.COPY, np.float32(0.5), b, t, 1 - b, t))
    tasks = W._tasks(len(rows))
    for i, r in enumerate(rows):
        tasks[i] = r
    return W.Program(bufs, [nparts] * nbuf, tasks)


def _worker(rank, world, port, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1304_0878_b200 import btask as B
        from paper_1304_0878_b200.programs import Session
        p = _program(seed)
        rt = B.Runtime(flags=B.BT_FLAG_HOST_ONLY, rank=rank, nranks=world, host_threads=2, parallel_min=4)
        s = Session(rt, p)
        for h in s.roots:
            rt.distribute_block(h)               # part t -> rank floor(t * world / nparts)
        s.submit()
        snap = rt.dag_snapshot()
        s.finish()
        rt.close()
        local = (snap["task_item"] != 0xFFFFFFFF).astype(np.int8)
        out = [None] * world
        dist.all_gather_object(out, {"local": local, "snap": snap})
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_two_ranks_partition_the_program():
    from tests.test_host import check_dag, reach  # noqa: F401
    import oracle
    seed = 4242
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, seed, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = _program(seed)
    l0, l1 = res[0]["local"], res[1]["local"]
    assert np.all(l0 + l1 == 1), "each task runs on exactly one rank"
    # owner = rank of the written operand's tile: tiles 0-3 -> rank 0, 4-7 -> rank 1
    written_tile = np.where(p.tasks["codelet"] == W.SCAL, p.tasks["t0"], p.tasks["t1"])
    assert np.array_equal(l1.astype(bool), written_tile >= 4)
    pairs = oracle.conflict_pairs(p)
    for r in range(2):
        snap = res[r]["snap"]
        ti, tp = snap["task_item"], snap["task_pos"]
        R = reach(snap)
        for (i, j) in pairs:
            if res[r]["local"][i] and res[r]["local"][j]:
                if ti[i] == ti[j]:
                    assert tp[i] < tp[j]
                else:
                    assert int(ti[j]) in R[ti[i]]
            else:
                # no conflicting pair is split across ranks (it would need a cross-rank edge)
                assert res[r]["local"][i] == res[r]["local"][j]


def _sweep_worker(rank, world, port, q):
    """The bench's strong-scaling shape: one vector, T tiles block-distributed,
    every rank submits the whole sweep-major SCAL stream (parallel builder path,
    remote tiles skipped in phase 1)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1304_0878_b200 import btask as B
        T, S = 96, 12
        x = np.ones(T * 16, np.float32)
        rt = B.Runtime(flags=B.BT_FLAG_HOST_ONLY, rank=rank, nranks=world, host_threads=3, parallel_min=64)
        h = rt.register_array(x)
        subs = rt.partition(h, T)
        rt.distribute_block(h)
        c = np.full(T * S, B.BT_CL_SCAL, np.int32)
        f = np.repeat(np.linspace(0.5, 1.5, S).astype(np.float32), T)
        h0 = np.tile(np.asarray(subs, np.uint64), S)
        rt.insert_batch(c, f, h0)
        st = rt.stats()
        snap = rt.dag_snapshot()
        rt.unpartition(h)
        rt.unregister(h)
        rt.close()
        out = [None] * world
        dist.all_gather_object(out, {"local": (snap["task_item"] != 0xFFFFFFFF), "k": snap["item_k"],
                                     "tasks_local": st["tasks_local"], "submitted": st["tasks_submitted"]})
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_block_distributed_sweeps_strong_scaling_shape(world):
    """Every rank submits all T x S tasks; rank r runs exactly the tasks on its
    block of tiles [r*T/N, (r+1)*T/N), fused into one k = S chain per tile."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sweep_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    T, S = 96, 12
    tile = np.tile(np.arange(T), S)
    total = np.zeros(T * S, np.int64)
    for r in range(world):
        lo, hi = r * T // world, (r + 1) * T // world
        assert np.array_equal(res[r]["local"], (tile >= lo) & (tile < hi))
        assert res[r]["submitted"] == T * S and res[r]["tasks_local"] == (hi - lo) * S
        assert sorted(res[r]["k"].tolist()) == [S] * (hi - lo)
        total += res[r]["local"]
    assert np.all(total == 1)
