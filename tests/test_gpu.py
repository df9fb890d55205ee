"""GPU parity: the CUDA path (through the C ABI) against the sequential CPU
oracle, bit for bit (BASELINE.json north_star: "Results must be bit-exact").

Small programs are compared element by element; full-size configs are
compared on samples the oracle evaluates exactly (each task is element-wise,
so element i of every output depends only on element i of the inputs and the
task sequence -- pinned in tests/test_oracle.py::test_element_major_equals_task_major).
"""
import errno

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1304_0878_b200 import build
    build.build()
    from paper_1304_0878_b200 import btask
    return btask


def run_gpu(program, **kw):
    from paper_1304_0878_b200.programs import run_program
    return run_program(program, **kw)


def assert_bits_equal(got, exp, what=""):
    g = np.asarray(got).view(np.uint32)
    e = np.asarray(exp).view(np.uint32)
    if not np.array_equal(g, e):
        bad = np.nonzero(g != e)[0]
        raise AssertionError(f"{what}: {bad.size} of {g.size} elements differ; first at {bad[:5]}: "
                             f"got {g[bad[:5]]} expected {e[bad[:5]]}")


def compare_program(program, **kw):
    out, stats = run_gpu(program, **kw)
    exp = oracle.run(program)
    for b, (o, e) in enumerate(zip(out, exp)):
        assert_bits_equal(o, e, f"{program.name} buffer {b}")
    return stats


@pytest.mark.parametrize("seed", range(6))
def test_direct_launch(B, seed):
    """Epochs of independent items (each task its own epoch: epoch_tasks = 1)
    run as direct launches -- one plain grid, items in the kernel parameters,
    no queue -- with ragged, unaligned tiles and chained SCAL items; bit-exact."""
    p = W.random_small_program(9000 + seed, max_tasks=60, max_handles=6, max_elems=5000)
    stats = compare_program(p, epoch_tasks=1)
    assert stats["epochs"] >= 1 and stats["units"] >= 1
    p2 = W.c2_chain(nx=1 << 14, ntiles=16, sweeps=5)   # 16 fused items of k = 5 in one epoch
    out, st = run_gpu(p2)
    assert_bits_equal(out[0], oracle.run(p2)[0], "direct C2-shaped")
    assert st["kernel_launches"] == 1 and st["block"] == 256, st


def test_direct_launch_groups(B):
    """A direct launch groups items of the same kind, length and factors whose
    operands advance by one stride (device_abi.h DirectItem): ragged tiles
    (two lengths: two groups), AXPY with x and y advancing together, COPY in
    reverse tile order (negative stride: no group), single factors that
    alternate (no group) and repeat (a group) -- one epoch, one launch,
    bit-exact."""
    rng = np.random.default_rng(W.SEED_BASE + 141)
    n, T = 1000, 7                                   # tiles of 143 (x6) and 142
    bufs = [W.unit_interval_floats(rng, n) for _ in range(6)]
    rows = [(W.SCAL, 1.5, 0, t, -1, -1) for t in range(T)]
    rows += [(W.AXPY, 0.25, 1, t, 2, t) for t in range(T)]
    rows += [(W.COPY, 0, 3, t, 4, t) for t in reversed(range(T))]
    rows += [(W.SCAL, (0.75, -2.0)[t % 2], 5, t, -1, -1) for t in range(4)]
    rows += [(W.SCAL, 3.0, 5, t, -1, -1) for t in range(4, T)]
    t = W._tasks(len(rows))
    for i, r in enumerate(rows):
        t[i] = r
    p = W.Program(bufs, [T] * 6, t, name="direct launch groups")
    st = compare_program(p)
    assert st["kernel_launches"] == 1 and st["block"] == 256 and st["items"] == len(rows), st


@pytest.mark.parametrize("seed", range(8))
def test_direct_launch_groups_random(B, seed):
    """Random epochs of independent tasks (each tile written once, sources
    never written): tiles in random order and random subsets, factors from a
    small set, AXPY/COPY between equally partitioned buffers, ragged tile
    lengths -- item groups form and break at random; one direct launch each,
    bit-exact."""
    rng = np.random.default_rng(W.SEED_BASE + 150 + seed)
    for rep in range(6):
        n = int(rng.integers(40, 3000))
        T = int(rng.integers(2, 40))
        bufs = [W.unit_interval_floats(rng, n) for _ in range(6)]
        rows = []
        for b in (0, 1):                                        # SCAL targets
            for t in rng.permutation(T)[: int(rng.integers(1, T + 1))]:
                rows.append((W.SCAL, float(rng.choice([0.5, 1.25, -3.0])), b, int(t), -1, -1))
        for t in rng.permutation(T)[: int(rng.integers(1, T + 1))]:
            rows.append((W.AXPY, float(rng.choice([0.25, -0.75])), 2, int(t), 3, int(t)))
        for t in np.sort(rng.permutation(T)[: int(rng.integers(1, T + 1))]):
            rows.append((W.COPY, 0.0, 4, int(t), 5, int(t)))
        order = rng.permutation(len(rows)) if rng.random() < 0.3 else np.arange(len(rows))
        t = W._tasks(len(rows))
        for i, j in enumerate(order):
            t[i] = rows[j]
        p = W.Program(bufs, [T] * 6, t, name=f"direct groups seed {seed} rep {rep}")
        st = compare_program(p)
        assert st["kernel_launches"] == 1 and st["block"] == 256, st


def test_c1_paper_example(B):
    from tests.golden import load
    pins = load("scal_pins.txt")
    p = W.c1_single()
    out, stats = run_gpu(p)
    assert f"{int(out[0].view(np.uint32)[-1]):08X}" == pins["c1_last"][0][0]
    assert [f"{int(v):08X}" for v in out[0][:8].view(np.uint32)] == pins["paper_example_1to8"][0]
    assert_bits_equal(out[0], oracle.run(p)[0], "C1")
    assert stats["items"] == 1 and stats["units"] == 1


def test_subnormal_inputs_not_flushed(B):
    from tests.golden import load
    rows = load("scal_pins.txt")["subnormal"]
    for inp, fac, outbits in rows:
        x = np.array([int(inp, 16)] * 37, np.uint32).view(np.float32)
        p = W.Program([x.copy()], [0], W._tasks(1))
        p.tasks[0] = (W.SCAL, np.uint32(int(fac, 16)).view(np.float32), 0, -1, -1, -1)
        out, _ = run_gpu(p)
        assert {f"{int(v):08X}" for v in out[0].view(np.uint32)} == {outbits}


KERNELS = {"auto": 0, "sw": 1 << 8, "rw": 1 << 9, "wq": 1 << 10}   # BT_FLAG_KERNEL_*


# ---- IEEE special values on every device path -------------

def special_programs(n=24, finite_scalars=False, base=5100, **kw):
    """Seeded special-value programs (+-0, +-inf, max finite, subnormals; scalars
    +-0, +-inf, 1e+-30) whose sequential result holds no NaN (NaN bit patterns
    are not portable, reading R11): a NaN-producing program is skipped."""
    out, seed = [], base
    while len(out) < n:
        p = W.special_value_program(seed, finite_scalars=finite_scalars, **kw)
        seed += 1
        if not any(np.isnan(b).any() for b in oracle.run(p)):
            out.append(p)
    return out


def _has_specials(programs):
    """The drawn programs do exercise the special cases (not vacuous)."""
    res = [oracle.run(p) for p in programs]
    allv = np.concatenate([np.concatenate(r) for r in res])
    bits = allv.view(np.uint32)
    assert np.isinf(allv).any() and (bits == 0x80000000).any() and (bits == 0).any()
    assert ((bits & 0x7F800000) == 0).any() and ((bits & 0x7FFFFF) != 0).any()


@pytest.mark.parametrize("kernel", ["sw", "rw", "wq"])
def test_special_values_per_kernel(B, kernel):
    """+-0, +-inf, overflow to +-inf, underflow to +-0 and subnormals, through
    each persistent scheduler variant (forced), fused and unfused, with
    multi-chunk items: bit-exact against the oracle."""
    progs = special_programs()
    _has_specials(progs)
    for fusion in (True, False):
        flags = (0 if fusion else B.BT_FLAG_NO_FUSION) | KERNELS[kernel]
        for p in progs:
            compare_program(p, flags=flags, chunk_bytes=96)


def test_special_values_direct_launch(B):
    """The same programs as direct launches (one epoch per task: independent
    items in the kernel parameters) and as whole-program epochs (auto choice)."""
    for p in special_programs():
        compare_program(p, epoch_tasks=1)
        compare_program(p)


def test_special_values_stream_launch(B):
    """Special values through the bench's stream launch: device-homed tiles,
    pipelined sweep-major SCAL runs (fused and unfused) with factors that
    overflow finite values to +-inf (1e30) and underflow them through the
    subnormals to +-0 (1e-30); +-inf and +-0 elements stay put (no factor is
    0 or inf, so no NaN)."""
    rng = np.random.default_rng(W.SEED_BASE + 95)
    ntiles, tile = 400, 8192
    x = W.special_floats(rng, ntiles * tile, frac=0.3)
    f = np.array([1e30, 3.14, -1e-30, 0.5, 1e30, -1.0, 1e-30, 2.0], np.float32)
    p = W.sweep_program(ntiles * tile, ntiles, f, x, name="special-value sweeps")
    exp = oracle.run(repeated(p, 2))[0]
    e = exp.view(np.uint32)
    assert np.isinf(exp).any() and (e == 0x80000000).any() and ((e & 0x7F800000) == 0).any()
    assert not np.isnan(exp).any()
    for flags in (0, B.BT_FLAG_NO_FUSION):
        out, st = run_device(B, p, repeats=2, flags=flags, pipeline_rounds=4, pipeline_min=500, parallel_min=500,
                             host_threads=3)
        assert_bits_equal(out[0], exp, f"special-value stream launch flags={flags}")
        assert st["sched_launches"] == 2 and st["epochs"] >= 4, st


@pytest.mark.parametrize("kernel", ["sw", "rw", "wq"])
@pytest.mark.parametrize("fusion", [True, False])
@pytest.mark.parametrize("chunk_bytes", [0, 96, 4096])
def test_random_programs_per_kernel(B, kernel, fusion, chunk_bytes):
    """Each scheduler variant, forced for every epoch, is bit-exact on random
    SCAL/AXPY/COPY programs (DAGs with ragged tiles, multi-chunk items, chains)."""
    flags = (0 if fusion else B.BT_FLAG_NO_FUSION) | KERNELS[kernel]
    for seed in range(1000, 1040):
        p = W.random_small_program(seed, max_tasks=10)
        compare_program(p, flags=flags, chunk_bytes=chunk_bytes)


@pytest.mark.parametrize("kernel", ["sw", "rw", "wq"])
def test_chains_per_kernel(B, kernel):
    """Unfused dependency chains (in-slot / in-warp continuations) and wide
    independent units, per scheduler variant, against the oracle."""
    for order in ("sweep", "tile"):
        p = W.c4_fine(ntiles=300, tile_nx=1024, sweeps=12, order=order)
        compare_program(p, flags=B.BT_FLAG_NO_FUSION | KERNELS[kernel])
    p = W.c4_fine(ntiles=1, tile_nx=1000, sweeps=300)   # one 1-wide chain, ragged vector tail
    compare_program(p, flags=B.BT_FLAG_NO_FUSION | KERNELS[kernel])


@pytest.mark.parametrize("fusion", [True, False])
@pytest.mark.parametrize("chunk_bytes", [0, 32, 96, 65536])
def test_random_programs(B, fusion, chunk_bytes):
    """>= 200 random programs, byte-identical to submission order.
    The kernel is the runtime's per-epoch choice (test_random_programs_per_kernel
    forces each variant)."""
    flags = 0 if fusion else B.BT_FLAG_NO_FUSION
    for seed in range(70):
        p = W.random_small_program(seed, max_tasks=10)
        compare_program(p, flags=flags, chunk_bytes=chunk_bytes)


def test_random_programs_larger_ragged(B):
    for seed in range(40):
        p = W.random_small_program(5000 + seed, max_tasks=40, max_handles=6, max_elems=5000)
        compare_program(p, chunk_bytes=1024)


def test_single_inserts_equal_batch(B):
    for seed in range(20):
        p = W.random_small_program(7000 + seed, max_tasks=12)
        compare_program(p, batch=False)


def test_c2_full_fused_and_unfused(B):
    p = W.c2_chain()                                      # 2^24 floats, 256 tiles, 16 sweeps
    exp = oracle.run(p)[0]
    for flags in (0, B.BT_FLAG_NO_FUSION):
        out, stats = run_gpu(p, flags=flags)
        assert_bits_equal(out[0], exp, f"C2 flags={flags}")
        assert stats["tasks_submitted"] == 4096
        if flags == 0:
            assert stats["items"] == 256 and stats["edges"] == 0
        else:
            assert stats["items"] == 4096 and stats["edges"] == 3840


def test_c2b_unpartitioned_chain(B):
    rng = np.random.default_rng(W.SEED_BASE + 11)
    x = W.unit_interval_floats(rng, 1 << 20)
    p = W.sweep_program(1 << 20, 1, np.full(16, np.float32(3.14), np.float32), x)
    p.nparts = [0]
    p.tasks["t0"] = -1
    compare_program(p)


@pytest.mark.parametrize("chunk_bytes", [0, 96, 4096])
def test_priority_ready_queue(B, chunk_bytes):
    """DAG epochs on the "sw" bodies use the upward-rank priority levels
    (BT_FLAG_PRIORITY, scheduler_kernel_swp): bit-exact on
    random programs and a reduced C3, with multi-chunk items; the default FIFO agrees."""
    progs = [W.random_small_program(7100 + s, max_tasks=10, max_elems=2000) for s in range(30)]
    progs.append(W.c3_random_dag(nbuf=12, nx=40000, ntasks=500, seed=99))
    n_prio = 0
    for p in progs:
        st = compare_program(p, flags=KERNELS["sw"] | B.BT_FLAG_PRIORITY, chunk_bytes=chunk_bytes)
        n_prio += st["prio_epochs"]
        st2 = compare_program(p, flags=KERNELS["sw"], chunk_bytes=chunk_bytes)
        assert st2["prio_epochs"] == 0
    assert n_prio >= 15


def _segment(bufs, nparts, rows):
    """Oracle run of one segment (fixed partitioning) on the current contents."""
    t = W._tasks(len(rows))
    for i, r in enumerate(rows):
        t[i] = r
    return oracle.run(W.Program([b.copy() for b in bufs], list(nparts), t))


@pytest.mark.parametrize("kernel", ["sw", "rw", "wq"])
@pytest.mark.parametrize("fusion", [True, False])
@pytest.mark.parametrize("chunk_bytes", [0, 256])
def test_chunkwise_release(B, kernel, fusion, chunk_bytes):
    """Chunk-wise release (device_abi.h K_ITEM_DEPS) in one epoch: items of
    many chunks after a same-length predecessor on the same handle (chunk c
    waits for chunk c only), with several predecessors (per-unit counters),
    and after predecessors inherited through a partition / unpartition /
    re-partition inside the epoch (other handles: whole-item release), per
    scheduler variant, one wait at the end; against the oracle run segment by
    segment (sequential composition)."""
    import torch
    rng = np.random.default_rng(W.SEED_BASE + 131)
    n = 10_003                                   # ragged: 157 chunks of 64 floats at chunk_bytes 256
    bufs = [W.unit_interval_floats(rng, n) for _ in range(3)]
    X, Y, Z = 0, 1, 2
    S, A, C = W.SCAL, W.AXPY, W.COPY
    seg1 = [(S, 1.5, X, -1, -1, -1), (A, 0.25, X, -1, Y, -1), (C, 0, Y, -1, Z, -1), (S, -0.75, Y, -1, -1, -1),
            (A, 0.5, Z, -1, X, -1), (S, 1.25, X, -1, -1, -1)]
    seg2 = [(A, 0.125, X, 0, Y, 0), (S, -1.5, X, 1, -1, -1), (C, 0, Y, 2, X, 2), (A, -0.25, X, 1, Y, 1),
            (S, 0.75, Z, 0, -1, -1), (S, 1.125, Y, 0, -1, -1)]
    seg3 = [(A, 0.375, Y, -1, X, -1), (S, 2.0, X, -1, -1, -1), (A, -0.5, X, -1, Z, -1), (C, 0, Z, -1, Y, -1)]
    seg4 = [(S, 0.5, X, 0, -1, -1), (S, -1.25, X, 2, -1, -1), (A, 0.25, Z, 0, Y, 0)]
    seg5 = [(A, 1.5, X, -1, Y, -1), (S, 0.625, Y, -1, -1, -1)]
    parts2, parts4 = [3, 3, 1], [3, 1, 1]
    exp = _segment(bufs, [0, 0, 0], seg1)
    exp = _segment(exp, parts2, seg2)
    exp = _segment(exp, [0, 0, 0], seg3)
    exp = _segment(exp, parts4, seg4)
    exp = _segment(exp, [0, 0, 0], seg5)
    flags = (0 if fusion else B.BT_FLAG_NO_FUSION) | KERNELS[kernel]
    tensors = [torch.from_numpy(b.copy()).cuda() for b in bufs]
    with B.Runtime(flags=flags, chunk_bytes=chunk_bytes) as rt:
        hs = [rt.register_tensor(t) for t in tensors]

        def submit(rows, views):
            for c, f, b0, t0, b1, t1 in rows:
                h0 = views[b0][t0] if t0 >= 0 else hs[b0]
                if c == S:
                    rt.scal(h0, f)
                    continue
                h1 = views[b1][t1] if t1 >= 0 else hs[b1]
                if c == A:
                    rt.axpy(f, h0, h1)
                else:
                    rt.copy(h0, h1)

        def partition(nparts):
            return [rt.partition(h, k) for h, k in zip(hs, nparts)]

        submit(seg1, None)
        submit(seg2, partition(parts2))
        for h in hs:
            rt.unpartition(h)
        submit(seg3, None)
        submit(seg4, partition(parts4))
        for h in hs:
            rt.unpartition(h)
        submit(seg5, None)
        rt.wait()
        st = rt.stats()
        for h in hs:
            rt.unregister(h)
    torch.cuda.synchronize()
    assert st["tasks_submitted"] == len(seg1 + seg2 + seg3 + seg4 + seg5) and st["epochs"] == 1, st
    for b in range(3):
        assert_bits_equal(tensors[b].cpu().numpy(), exp[b], f"buffer {b}")


def test_c3_reduced(B):
    p = W.c3_random_dag(nbuf=64, nx=1 << 12, ntasks=10000)
    stats = compare_program(p, chunk_bytes=4096)
    assert stats["tasks_submitted"] == 10000


def test_c3_full_sampled(B):
    """C3 at full size (64 x 2^20 floats, 10,000 tasks); the oracle runs the same
    task stream on a 4,096-element column sample (element-wise tasks)."""
    p = W.c3_random_dag()
    out, stats = run_gpu(p)
    rng = np.random.default_rng(3)
    idx = np.unique(np.concatenate([rng.integers(0, 1 << 20, 4096), [0, 1, (1 << 20) - 1]]))
    sub = W.Program([b[idx].copy() for b in p.buffers], p.nparts, p.tasks)
    exp = oracle.run(sub)
    for b in range(64):
        assert np.all(np.isfinite(exp[b]))
        assert_bits_equal(out[b][idx], exp[b], f"C3 buffer {b}")


@pytest.mark.parametrize("fusion", [False, True])
def test_c4_full(B, fusion):
    p = W.c4_fine()                                       # 1,000,000 tasks on 4 KiB tiles
    out, stats = run_gpu(p, flags=0 if fusion else B.BT_FLAG_NO_FUSION)
    exp = oracle.scal_chain(p.buffers[0], p.meta["factors"])
    assert_bits_equal(out[0], exp, "C4")
    assert stats["tasks_submitted"] == 1_000_000
    assert stats["items"] == (15625 if fusion else 1_000_000)


def test_c4_tile_major_order(B):
    p = W.c4_fine(ntiles=2000, sweeps=16, order="tile")
    out, _ = run_gpu(p, flags=B.BT_FLAG_NO_FUSION)
    assert_bits_equal(out[0], oracle.scal_chain(p.buffers[0], p.meta["factors"]), "C4 tile-major")


@pytest.mark.slow
def test_c5_full_sampled(B):
    p = W.c5_sharded()                                    # 4 GiB, 16,384 tiles x 64 sweeps
    x0 = p.buffers[0]
    rng = np.random.default_rng(4)
    idx = np.unique(np.concatenate([rng.integers(0, x0.shape[0], 1 << 20),
                                    np.arange(16384) * 65536, np.arange(16384) * 65536 + 65535]))
    exp = oracle.scal_chain(x0[idx], p.meta["factors"])
    out, stats = run_gpu(p)
    assert stats["items"] == 16384 and stats["tasks_submitted"] == 1 << 20
    assert_bits_equal(out[0][idx], exp, "C5 sample")
    assert np.all(np.isfinite(out[0][::4099]))


def test_device_homed_tensor_and_acquire(B):
    import torch
    rng = np.random.default_rng(12)
    x = W.unit_interval_floats(rng, 10_000)
    t = torch.from_numpy(x.copy()).cuda()
    with B.Runtime() as rt:
        h = rt.register_tensor(t)
        subs = rt.partition(h, 7)
        for s in subs:
            rt.scal(s, 3.14)
        rt.wait()
        rt.unpartition(h)
        rt.unregister(h)
    torch.cuda.synchronize()
    p = W.Program([x.copy()], [7], W._tasks(7))
    p.tasks["codelet"] = W.SCAL
    p.tasks["scalar"] = np.float32(3.14)
    p.tasks["t0"] = np.arange(7)
    assert_bits_equal(t.cpu().numpy(), oracle.run(p)[0], "device-homed")


def test_acquire_release_rw_roundtrip(B):
    x = np.arange(1, 1001, dtype=np.float32)
    with B.Runtime() as rt:
        h = rt.register_array(x)
        rt.scal(h, 2.0)
        rt.acquire(h, B.BT_RW)                         # host copy valid
        assert np.array_equal(x, np.arange(1, 1001, dtype=np.float32) * 2)
        assert rt.insert(B.BT_CL_SCAL, [h], [B.BT_RW], 2.0) == -errno.EBUSY
        x[:] = 1.0                                     # host write under RW acquire
        rt.release(h)
        rt.scal(h, 3.0)
        rt.unregister(h)
    assert np.all(x == 3.0)


def test_epochs_flush_and_autoflush(B):
    p = W.c4_fine(ntiles=300, sweeps=20)
    exp = oracle.scal_chain(p.buffers[0], p.meta["factors"])
    out, stats = run_gpu(p, epoch_tasks=1000)
    assert_bits_equal(out[0], exp, "auto-flush")
    assert stats["epochs"] >= 6
    from paper_1304_0878_b200.programs import Session
    with B.Runtime() as rt:
        s = Session(rt, p)
        h0, h1 = s.handle_arrays()
        t = p.tasks
        for lo in range(0, p.ntasks, 1700):
            rt.insert_batch(t["codelet"][lo:lo + 1700], t["scalar"][lo:lo + 1700], h0[lo:lo + 1700])
            rt.flush()
        rt.wait()
        assert_bits_equal(s.finish()[0], exp, "explicit flush")


def test_empty_wait_and_tiny(B):
    with B.Runtime() as rt:
        rt.wait()
        x = np.array([1.5], np.float32)
        h = rt.register_array(x)
        rt.scal(h, 3.14)
        rt.wait()
        rt.unregister(h)
    assert x[0] == np.float32(1.5) * np.float32(3.14)


@pytest.mark.parametrize("kernel", ["auto", "sw", "rw", "wq"])
def test_trace_timestamps(B, kernel):
    """One trace record per unit (continuations are off while tracing)."""
    p = W.c4_fine(ntiles=500, sweeps=8)
    from paper_1304_0878_b200.programs import Session
    with B.Runtime(flags=B.BT_FLAG_TIMESTAMPS | B.BT_FLAG_NO_FUSION | KERNELS[kernel]) as rt:
        s = Session(rt, p)
        s.submit()
        rt.wait()
        tr = rt.trace()
        s.finish()
    assert tr is not None
    t, item = tr
    assert t.shape == (4000, 4) and np.all(t[:, 0] > 0)
    assert sorted(item.tolist()) == list(range(4000))
    # multi-chunk items: each (item, chunk) unit writes its own record
    # (unit_base[item] + chunk, no shared counter): every item 4 times
    with B.Runtime(flags=B.BT_FLAG_TIMESTAMPS | B.BT_FLAG_NO_FUSION | KERNELS[kernel], chunk_bytes=1024) as rt:
        s = Session(rt, p)
        s.submit()
        rt.wait()
        t2, item2 = rt.trace()
        s.finish()
    assert t2.shape == (16000, 4) and np.all(t2[:, 0] > 0)
    assert np.array_equal(np.bincount(item2, minlength=4000), np.full(4000, 4))


@pytest.mark.parametrize("rounds,threads", [(2, 2), (3, 4), (4, 3)])
def test_pipelined_rounds(B, rounds, threads):
    """Long SCAL runs built and launched in rounds on two streams (forced on
    small runs), interleaved with AXPY/COPY tasks and further SCAL runs."""
    rng = np.random.default_rng(91 + rounds)
    nbuf, nparts, n = 3, 300, 300 * 64
    bufs = [W.unit_interval_floats(rng, n) for _ in range(nbuf)]
    rows = []
    for blk in range(5):
        for _ in range(int(rng.integers(2000, 4000))):
            b = int(rng.integers(0, nbuf))
            rows.append((W.SCAL, np.float32(rng.uniform(0.9, 1.1)), b, int(rng.integers(0, nparts)), -1, -1))
        for _ in range(int(rng.integers(1, 20))):
            b0, b1 = rng.choice(nbuf, 2, replace=False)
            t = int(rng.integers(0, nparts))
            rows.append((W.AXPY if rng.random() < .5 else W.COPY, np.float32(0.25), int(b0), t, int(b1), t))
    tasks = W._tasks(len(rows))
    for i, r in enumerate(rows):
        tasks[i] = r
    p = W.Program(bufs, [nparts] * nbuf, tasks)
    for fusion in (True, False):
        compare_program(p, flags=0 if fusion else B.BT_FLAG_NO_FUSION, pipeline_rounds=rounds, pipeline_min=500,
                        parallel_min=500, host_threads=threads)


def test_c5_shape_pipelined_default(B):
    """The bench's path (default rounds) on a reduced C5: 1024 tiles x 64 sweeps."""
    p = W.c5_sharded(nx=1024 * 4096, ntiles=1024, sweeps=64)
    out, stats = run_gpu(p, pipeline_min=1024)
    assert_bits_equal(out[0], oracle.scal_chain(p.buffers[0], p.meta["factors"]), "C5 reduced, pipelined")
    assert stats["epochs"] >= 4


# ---- stream launches: the rounds of a pipelined run as
# sub-epochs of one persistent launch, published while it runs ----

def run_device(B, program, repeats=1, **kw):
    """Device-homed buffers (torch tensors); the program submitted `repeats`
    times back to back with one wait at the end."""
    import torch
    from paper_1304_0878_b200.programs import Session
    tensors = [torch.from_numpy(b.copy()).cuda() for b in program.buffers]
    with B.Runtime(**kw) as rt:
        s = Session(rt, program, device_tensors=tensors)
        for _ in range(repeats):
            s.submit()
        rt.wait()
        st = rt.stats()
        s.finish()
    torch.cuda.synchronize()
    return [t.cpu().numpy() for t in tensors], st


def repeated(program, k):
    return W.Program(program.buffers, program.nparts, np.concatenate([program.tasks] * k), name=program.name)


@pytest.mark.parametrize("rounds,threads", [(2, 2), (4, 3), (6, 5), (10, 4)])
@pytest.mark.parametrize("fusion", [True, False])
def test_stream_launch(B, rounds, threads, fusion):
    """32 KiB tiles ("sw" units), sweep-major SCAL runs: every run's rounds join
    one launch (fewer scheduler launches than epochs); unfused, each sub-epoch
    is a DAG of chains released on the device.  Three runs in flight back to
    back, then one wait; bit-exact against the oracle."""
    p = W.c5_sharded(nx=600 * 8192, ntiles=600, sweeps=12)
    flags = 0 if fusion else B.BT_FLAG_NO_FUSION
    out, st = run_device(B, p, repeats=3, flags=flags, pipeline_rounds=rounds, pipeline_min=500,
                         parallel_min=500, host_threads=threads)
    assert_bits_equal(out[0], oracle.run(repeated(p, 3))[0], f"stream launch r={rounds}")
    assert st["epochs"] >= 2 * 3 and st["sched_launches"] == 3 and st["stream_closes"] == 0, st
    out2, st2 = run_device(B, p, repeats=1, flags=flags | B.BT_FLAG_NO_STREAM, pipeline_rounds=rounds,
                           pipeline_min=500, parallel_min=500, host_threads=threads)
    assert_bits_equal(out2[0], oracle.run(p)[0], f"per-round launches r={rounds}")
    assert st2["sched_launches"] == st2["epochs"], st2


def test_stream_launch_deferred(B, tmp_path):
    """BT_STREAM_DEFER=1 (for tools that serialise launches): the stream launch
    is enqueued after its last sub-epoch is published; same results."""
    import subprocess
    import sys
    code = (
        "import numpy as np, oracle, workloads as W\n"
        "from tests.test_gpu import run_device, repeated, assert_bits_equal\n"
        "from paper_1304_0878_b200 import btask as B\n"
        "p = W.c5_sharded(nx=300 * 8192, ntiles=300, sweeps=8)\n"
        "for flags in (0, B.BT_FLAG_NO_FUSION):\n"
        "    out, st = run_device(B, p, repeats=2, flags=flags, pipeline_rounds=4, pipeline_min=200,\n"
        "                         parallel_min=200, host_threads=3)\n"
        "    assert_bits_equal(out[0], oracle.run(repeated(p, 2))[0], 'deferred stream launch')\n"
        "    assert st['sched_launches'] == 2 and st['epochs'] >= 4, st\n"
        "from tests.test_gpu import uneven_rounds_program\n"
        "q = uneven_rounds_program()\n"
        "out, st = run_device(B, q, repeats=2, pipeline_rounds=4, pipeline_min=500, parallel_min=500,\n"
        "                     host_threads=3)\n"
        "assert_bits_equal(out[0], oracle.run(repeated(q, 2))[0], 'deferred launch closed early')\n"
        "assert st['stream_closes'] >= 1, st\n"
        "print('ok')\n")
    import os
    env = dict(os.environ, BT_STREAM_DEFER="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=os.path.dirname(os.path.dirname(__file__)), env=env,
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


_STREAM_ENV_CODE = (
    "import numpy as np, oracle, workloads as W\n"
    "from tests.test_gpu import run_device, repeated, assert_bits_equal\n"
    "from paper_1304_0878_b200 import btask as B\n"
    "p = W.c5_sharded(nx=300 * 8192, ntiles=300, sweeps=8)\n"
    "res = 0\n"
    "for flags in (0, B.BT_FLAG_NO_FUSION):\n"
    "    out, st = run_device(B, p, repeats=2, flags=flags, pipeline_rounds=4, pipeline_min=200,\n"
    "                         parallel_min=200, host_threads=3)\n"
    "    assert_bits_equal(out[0], oracle.run(repeated(p, 2))[0], 'stream launch')\n"
    "    assert st['epochs'] >= 4 and st['stream_closes'] == 0, st\n"
    "    res += st['stream_resumes']\n"
    "print('ok resumes', res)\n")


def _run_stream_env(env_extra):
    import os
    import subprocess
    import sys
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", _STREAM_ENV_CODE], cwd=os.path.dirname(os.path.dirname(__file__)),
                       env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
    return int(r.stdout.split("ok resumes")[1].split()[0])


def test_stream_launch_auto_defer_launch_blocking(B):
    """CUDA_LAUNCH_BLOCKING=1 serialises launches (as ncu and compute-sanitizer
    do): the stream launch is deferred automatically after the last
    publication -- no close, no resume, same bits."""
    assert _run_stream_env({"CUDA_LAUNCH_BLOCKING": "1"}) == 0


def test_stream_launch_closes_and_resumes_when_blocked(B):
    """The same with auto-deferral disabled: the launch call blocks until the
    kernel ends, the kernel runs sub-epoch 0, waits 50 ms for publications
    that cannot come, closes itself, and the run's resume launch runs the
    abandoned tickets and the rest -- bit-exact, never the watchdog."""
    assert _run_stream_env({"CUDA_LAUNCH_BLOCKING": "1", "BT_STREAM_NODEFER": "1"}) >= 2


def test_stream_launch_closes_and_resumes_slow_host(B):
    """A host that publishes late (2 ms per sub-epoch, quiescence limit 0.2 ms)
    while the launch really runs: closes race with publications; every run
    stays bit-exact (the resume launch picks up what the close left)."""
    n = _run_stream_env({"BT_DEBUG_PUBLISH_DELAY_US": "2000", "BT_QUIESCE_US": "200"})
    assert n >= 1


def test_failed_pipelined_run_reports_and_poisons(B):
    """An epoch-memory allocation that fails inside a pipelined run (injected:
    BT_DEBUG_FAIL_DEV_ALLOC) is returned from bt_insert_task_batch with no task
    counted as submitted, and the runtime is poisoned -- never a silent
    sequential replay that would scale tiles twice."""
    import os
    import subprocess
    import sys
    code = (
        "import errno, numpy as np, torch, workloads as W\n"
        "from paper_1304_0878_b200 import btask as B\n"
        "from paper_1304_0878_b200.programs import Session\n"
        "p = W.c5_sharded(nx=300 * 8192, ntiles=300, sweeps=8)\n"
        "x = torch.from_numpy(p.buffers[0].copy()).cuda()\n"
        "rt = B.Runtime(pipeline_rounds=4, pipeline_min=200, parallel_min=200, host_threads=3)\n"
        "s = Session(rt, p, device_tensors=[x])\n"
        "h0, _ = s.handle_arrays()\n"
        "c = np.ascontiguousarray(p.tasks['codelet']); f = np.ascontiguousarray(p.tasks['scalar'])\n"
        "import ctypes\n"
        "n = ctypes.c_size_t(12345)\n"
        "rc = B.bt_insert_task_batch(rt.rt, len(c), c.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),\n"
        "    f.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), h0.ctypes.data_as(ctypes.POINTER(B.bt_handle)),\n"
        "    None, ctypes.byref(n))\n"
        "assert rc < 0 and n.value == 0, (rc, n.value)\n"
        "assert B.bt_task_wait_for_all(rt.rt) == -errno.EIO\n"
        "print('ok', rc, rt.last_error())\n")
    env = dict(os.environ, BT_DEBUG_FAIL_DEV_ALLOC="3")
    r = subprocess.run([sys.executable, "-c", code], cwd=os.path.dirname(os.path.dirname(__file__)), env=env,
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def uneven_rounds_program():
    rng = np.random.default_rng(77)
    nparts, tile = 400, 8192
    x = W.unit_interval_floats(rng, nparts * tile)
    # round 0 (tiles 0-99): chains of 12 (fused: 100 items); rounds 1-3: one
    # task per tile (300 items) -- launches are balanced by tasks, not items
    rows = []
    for _ in range(12):
        for t in range(100):
            rows.append((W.SCAL, np.float32(rng.uniform(0.9, 1.1)), 0, t, -1, -1))
    for t in range(100, nparts):
        rows.append((W.SCAL, np.float32(rng.uniform(0.9, 1.1)), 0, t, -1, -1))
    tasks = W._tasks(len(rows))
    for i, r in enumerate(rows):
        tasks[i] = r
    return W.Program([x], [nparts], tasks, name="uneven rounds")


def test_stream_launch_closes_early(B):
    """Rounds of very different sizes: a later round outgrows the epoch
    buffers sized at the first one, closes the running launch (its remaining
    sub-epochs are published empty) and runs as ordinary epochs -- no
    allocation while the launch waits, same results."""
    p = uneven_rounds_program()
    out, st = run_device(B, p, repeats=2, pipeline_rounds=4, pipeline_min=500, parallel_min=500, host_threads=3)
    assert_bits_equal(out[0], oracle.run(repeated(p, 2))[0], "uneven rounds")
    assert st["stream_closes"] >= 1, st


def test_stream_launch_mixed_program(B):
    """Pipelined SCAL runs (stream launches) between AXPY/COPY tasks on the same
    device-homed tiles: the dependencies across launches and the ordinary
    epochs in between hold."""
    rng = np.random.default_rng(4242)
    nbuf, nparts, n = 2, 200, 200 * 8192
    bufs = [W.unit_interval_floats(rng, n) for _ in range(nbuf)]
    rows = []
    for blk in range(4):
        f = W.sweep_factors(rng, 6)
        for s_ in range(6):
            for t in range(nparts):
                rows.append((W.SCAL, f[s_], blk % nbuf, t, -1, -1))
        for _ in range(int(rng.integers(1, 30))):
            t = int(rng.integers(0, nparts))
            rows.append((W.AXPY if rng.random() < .5 else W.COPY, np.float32(0.25), 1 - blk % nbuf, t, blk % nbuf, t))
    tasks = W._tasks(len(rows))
    for i, r in enumerate(rows):
        tasks[i] = r
    p = W.Program(bufs, [nparts] * nbuf, tasks, name="stream launches between AXPY/COPY")
    out, st = run_device(B, p, pipeline_rounds=4, pipeline_min=500, parallel_min=500, host_threads=3)
    exp = oracle.run(p)
    for b in range(nbuf):
        assert_bits_equal(out[b], exp[b], f"mixed buffer {b}")
    assert st["sched_launches"] < st["epochs"], st


# ---- host <-> device coherence: chunked upload, eager write-back, dirty path ----

def _sweeps(B, rt, subs, factors):
    n = len(subs)
    c = np.full(n * len(factors), B.BT_CL_SCAL, np.int32)
    s = np.repeat(factors.astype(np.float32), n)
    h0 = np.tile(np.asarray(subs, np.uint64), len(factors))
    rt.insert_batch(c, s, h0)


def test_large_host_buffer_pipelined_writeback(B):
    """64 MiB host buffer: chunked upload, pipelined rounds, eager write-back of
    each round's range; unregister must leave the exact result in the buffer."""
    rng = np.random.default_rng(31)
    x0 = W.unit_interval_floats(rng, 1 << 24)
    f = W.sweep_factors(rng, 12)
    x = x0.copy()
    with B.Runtime(pipeline_min=1024) as rt:
        h = rt.register_array(x)
        subs = rt.partition(h, 1024)
        _sweeps(B, rt, subs, f)
        rt.wait()
        rt.unpartition(h)
        rt.unregister(h)
    assert_bits_equal(x, oracle.scal_chain(x0, f), "write-back")


def test_large_host_buffer_written_twice_and_acquire(B):
    """A range written by two epochs (dirty): unregister copies everything back;
    an acquire in between sees the first batch's result."""
    rng = np.random.default_rng(32)
    x0 = W.unit_interval_floats(rng, 1 << 24)
    f1, f2 = W.sweep_factors(rng, 5), W.sweep_factors(rng, 7)
    x = x0.copy()
    with B.Runtime(pipeline_min=1024) as rt:
        h = rt.register_array(x)
        subs = rt.partition(h, 512)
        _sweeps(B, rt, subs, f1)
        rt.wait()
        rt.acquire(subs[3], B.BT_R)
        lo = 3 * (1 << 24) // 512
        mid = oracle.scal_chain(x0, f1)
        assert_bits_equal(x[lo:lo + (1 << 24) // 512], mid[lo:lo + (1 << 24) // 512], "acquire after batch 1")
        rt.release(subs[3])
        _sweeps(B, rt, subs, f2)
        rt.wait()
        rt.unpartition(h)
        rt.unregister(h)
    assert_bits_equal(x, oracle.scal_chain(mid, f2), "dirty write-back")


def test_large_host_buffer_untouched_and_axpy(B):
    rng = np.random.default_rng(33)
    a0 = W.unit_interval_floats(rng, 1 << 24)
    b0 = W.unit_interval_floats(rng, 1 << 24)
    a, b = a0.copy(), b0.copy()
    with B.Runtime() as rt:
        ha, hb = rt.register_array(a), rt.register_array(b)
        rt.axpy(0.5, ha, hb)               # reads a (chunked upload), writes b
        rt.wait()
        rt.unregister(ha)
        rt.unregister(hb)
    assert_bits_equal(a, a0, "untouched")
    assert_bits_equal(b, (np.float32(0.5) * a0 + b0).astype(np.float32), "axpy")


def test_write_first_copy_skips_upload(B):
    """NEXT-4 (reading R7 "W": prior contents not read): a host
    buffer whose first access is a COPY destination is never uploaded -- its
    initial contents (here NaN garbage) cannot matter -- while a buffer read
    first is uploaded once.  Bytes counted by bt_stats.h2d_data_bytes; the
    results are the oracle's; unregister writes every result back."""
    rng = np.random.default_rng(W.SEED_BASE + 96)
    n = 1 << 20
    x0 = W.unit_interval_floats(rng, n)
    y0 = np.full(n, np.nan, np.float32)          # write-only first: never read
    z0 = np.full(n, np.nan, np.float32)
    rows = [(W.COPY, 0.0, 0, -1, 1, -1), (W.SCAL, np.float32(2.5), 1, -1, -1, -1),
            (W.COPY, 0.0, 1, -1, 2, -1), (W.AXPY, np.float32(0.25), 0, -1, 2, -1)]
    p = W.Program([x0, y0, z0], [0, 0, 0], W._tasks(len(rows)), name="W-first")
    for i, r in enumerate(rows):
        p.tasks[i] = r
    exp = oracle.run(p)
    bufs = p.copy_buffers()
    with B.Runtime() as rt:
        from paper_1304_0878_b200.programs import Session
        sess = Session(rt, p, host_buffers=bufs)
        sess.submit(batch=False)
        rt.wait()
        st = rt.stats()
        sess.finish()
    for b in range(3):
        assert_bits_equal(bufs[b], exp[b], f"W-first buffer {b}")
    assert st["h2d_data_bytes"] == 4 * n, st          # x only
    assert st["d2h_data_bytes"] == 2 * 4 * n, st      # y and z written back, x untouched


def test_partial_write_first_tiles(B):
    """Per-range coherence: tiles 1 and 2 of a partitioned host buffer are COPY
    destinations first (no upload), tiles 0 and 3 are scaled (uploaded); tile 2
    is then written again (dirty: copied back at unregister)."""
    rng = np.random.default_rng(W.SEED_BASE + 97)
    nt, tile = 4, 1 << 18
    x0 = W.unit_interval_floats(rng, nt * tile)
    x0[tile:3 * tile] = np.nan
    src = W.unit_interval_floats(rng, nt * tile)
    rows = [(W.COPY, 0.0, 1, 1, 0, 1), (W.COPY, 0.0, 1, 2, 0, 2), (W.SCAL, np.float32(0.5), 0, 0, -1, -1),
            (W.SCAL, np.float32(3.0), 0, 3, -1, -1), (W.SCAL, np.float32(1.5), 0, 2, -1, -1)]
    p = W.Program([x0, src], [nt, nt], W._tasks(len(rows)), name="partial W-first")
    for i, r in enumerate(rows):
        p.tasks[i] = r
    exp = oracle.run(p)
    bufs = p.copy_buffers()
    with B.Runtime() as rt:
        from paper_1304_0878_b200.programs import Session
        sess = Session(rt, p, host_buffers=bufs)
        sess.submit(batch=False)
        rt.wait()
        st = rt.stats()
        sess.finish()
    for b in range(2):
        assert_bits_equal(bufs[b], exp[b], f"partial W-first buffer {b}")
    # x: tiles 0 and 3 uploaded; src: tiles 1 and 2 read
    assert st["h2d_data_bytes"] == 4 * 4 * tile, st


def test_stress_random_configurations(B):
    """Random programs under random runtime configurations (work-unit size,
    fusion, builder threads, pipelining thresholds, epoch auto-flush): every
    path of the builder and both kernels against the oracle."""
    rng = np.random.default_rng(2024)
    for trial in range(60):
        p = W.random_small_program(9000 + trial, max_tasks=int(rng.integers(5, 80)),
                                   max_handles=int(rng.integers(1, 6)), max_elems=int(rng.integers(8, 20000)))
        kw = dict(chunk_bytes=int(rng.choice([0, 32, 64, 512, 4096, 65536])),
                  flags=0 if rng.random() < 0.7 else B.BT_FLAG_NO_FUSION,
                  host_threads=int(rng.integers(1, 6)), parallel_min=int(rng.integers(1, 8)),
                  pipeline_min=int(rng.integers(1, 16)), pipeline_rounds=int(rng.integers(1, 5)),
                  max_fused=int(rng.choice([0, 1, 2, 3, 7])),
                  epoch_tasks=int(rng.choice([0, 0, 3, 11])))
        compare_program(p, **kw)


def test_c_example_program(B, tmp_path):
    """examples/vector_scal.c: the paper's running example written in C
    against include/btask.h, linked with libbtask.so."""
    import os
    import re
    import struct
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib_dir = os.path.join(root, "paper_1304_0878_b200")
    exe = str(tmp_path / "vector_scal")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-I", os.path.join(root, "include"),
                           os.path.join(root, "examples", "vector_scal.c"), "-L", lib_dir, "-lbtask",
                           f"-Wl,-rpath,{lib_dir}", "-o", exe])
    out = subprocess.check_output([exe], text=True, timeout=120)
    from tests.golden import load
    pins = load("scal_pins.txt")
    last = float(re.search(r"vector\[1023\] = (\S+)", out).group(1))
    assert f"{struct.unpack('<I', struct.pack('<f', last))[0]:08X}" == pins["c1_last"][0][0]
    assert "attempt to use unregistered pointer" in out
    big0 = float(re.search(r"big\[0\] = (\S+)", out).group(1))
    assert f"{struct.unpack('<I', struct.pack('<f', big0))[0]:08X}" == pins["chain_k16"][0][0]
    assert "1025 tasks in 65 items (960 fused)" in out   # 1 + 16 x 64 tasks; chains fuse per tile


@pytest.mark.slow
def test_bench_launch_configuration_c5(B):
    """bench.py's exact path at full size: device-homed 4 GiB tensor, 16,384
    tiles, the C5 task stream through bt_insert_task_batch with the default
    configuration (pipelined rounds as sub-epochs of one stream launch of the
    "sw" kernel per step), two steps; sampled elements against the oracle."""
    import importlib.util
    import os
    import torch
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    n, T, S = 1 << 30, 16384, 64
    f = W.sweep_factors(np.random.default_rng(W.SEED_BASE + 4), S)
    x = bench.synth_tile_values(torch, n, 1000, torch.device("cuda", 0))
    rng = np.random.default_rng(5)
    idx = np.unique(np.concatenate([rng.integers(0, n, 1 << 18), np.arange(T) * (n // T), [n - 1]]))
    x0 = x[torch.from_numpy(idx).cuda()].cpu().numpy()
    stream = torch.cuda.current_stream()
    with B.Runtime(stream=stream.cuda_stream) as rt:
        h = rt.register_tensor(x)
        subs = rt.partition(h, T)
        c, s, h0 = bench.rank_tasks(np, subs, f)
        for _ in range(2):
            rt.insert_batch(c, s, h0)
            rt.wait()
        st = rt.stats()
        rt.unpartition(h)
        rt.unregister(h)
    assert st["epochs"] >= 8 and st["items"] == 2 * T
    assert st["sched_launches"] == 2 and st["stream_closes"] == 0, st   # one stream launch per step
    got = x[torch.from_numpy(idx).cuda()].cpu().numpy()
    exp = oracle.scal_chain(oracle.scal_chain(x0, f), f)
    assert_bits_equal(got, exp, "bench configuration, two steps")


# ---- cross-rank reads (bt_comm_init) ----------------

def _check_owned(program, results, owners):
    from tests import xrank
    exp = oracle.run(program)
    seen = 0
    for b in range(len(program.buffers)):
        for t, off, n in xrank.leaf_ranges(program, b):
            assert (b, t) in results, f"leaf {(b, t)} owned by nobody"
            assert_bits_equal(results[(b, t)], exp[b][off:off + n], f"{program.name} buffer {b} tile {t}")
            seen += 1
    assert seen == len(results)


@pytest.mark.parametrize("batch", [True, False])
def test_cross_rank_reads_random_programs(B, batch):
    """Two ranks (processes) with random owners per leaf run random SCAL/AXPY/COPY
    programs; an AXPY/COPY reading another rank's data copies it over (CUDA IPC)
    at its submission point.  Every leaf's owner ends with the oracle's bits."""
    from tests import xrank
    for seed in range(4):
        p = W.random_small_program(3000 + seed, max_tasks=12, max_elems=4096)
        results, stats, owners = xrank.run(p, nranks=2, seed=seed, batch=batch)
        _check_owned(p, results, owners)


def test_cross_rank_shared_copies(B):
    """Shared copies across ranks (NEXT-4, "lazy MSI across ranks"): rank 1
    reads X (rank 0's) into five of its buffers with no write of X in between
    -- one transfer, four skipped on both ranks --, then rank 0 scales X and
    rank 1 reads it again (a new transfer), and a tile of a partitioned
    buffer is read twice; every owner's data is the oracle's."""
    from tests import xrank
    n = 1 << 16
    rng = np.random.default_rng(W.SEED_BASE + 99)
    bufs = [W.unit_interval_floats(rng, n) for _ in range(7)] + [W.unit_interval_floats(rng, 4 * n)]
    rows = [(W.COPY, 0.0, 0, -1, 1 + i, -1) for i in range(5)]          # 1 transfer + 4 skips
    rows += [(W.SCAL, np.float32(1.25), 0, -1, -1, -1),                  # X written on rank 0
             (W.AXPY, np.float32(0.5), 0, -1, 6, -1),                    # new transfer
             (W.AXPY, np.float32(0.25), 0, -1, 6, -1),                   # skip
             (W.COPY, 0.0, 7, 1, 1, -1), (W.COPY, 0.0, 7, 1, 2, -1)]     # tile 1 of buffer 7: transfer + skip
    p = W.Program(bufs, [0] * 7 + [4], W._tasks(len(rows)), name="shared copies across ranks")
    for i, r in enumerate(rows):
        p.tasks[i] = r
    owners = [0, 1, 1, 1, 1, 1, 1, [0, 0, 1, 1]]
    results, stats, owners = xrank.run(p, nranks=2, owners=owners, batch=False)
    _check_owned(p, results, owners)
    for st in stats:
        assert st["cross_rank_copies"] == 3 and st["cross_rank_skips"] == 4 + 1 + 1, st


@pytest.mark.parametrize("protocol", ["host", "flag_kernels"])
def test_cross_rank_other_protocols(B, protocol):
    """The same random cross-rank programs with the host protocol (shared-memory
    counters + interprocess events, BT_COMM_HOST=1) and with the device
    protocol's one-thread flag kernels instead of stream memory operations."""
    import os
    from tests import xrank
    var = {"host": "BT_COMM_HOST", "flag_kernels": "BT_COMM_FLAG_KERNELS"}[protocol]
    os.environ[var] = "1"
    try:
        for seed in range(3):
            p = W.random_small_program(3100 + seed, max_tasks=12, max_elems=4096)
            results, stats, owners = xrank.run(p, nranks=2, seed=seed)
            _check_owned(p, results, owners)
        p = _gated_program()
        results, stats, owners = xrank.run(p, nranks=2, owners=[0, 1], gate=(0, 0.3), batch=False)
        _check_owned(p, results, owners)
    finally:
        del os.environ[var]


def test_cross_rank_c3_dag_and_sharded_sweeps(B):
    """C3-shaped random DAG (AXPY/COPY across owners -> many rendezvous) and a
    C5-shaped owner-computes sweep (tile halves per rank; each rank's local
    run is a pipelined stream launch) over two ranks: every owner's data is
    the oracle's."""
    from tests import xrank
    p = W.c3_random_dag(nbuf=12, nx=1 << 13, ntasks=400, seed=4711)
    results, stats, owners = xrank.run(p, nranks=2, seed=5)
    _check_owned(p, results, owners)
    q = W.c5_sharded(nx=512 * 8192, ntiles=512, sweeps=8)
    owners = [[0 if t < 256 else 1 for t in range(512)]]
    results, stats, owners = xrank.run(q, nranks=2, owners=owners,
                                       rt_kwargs=dict(pipeline_min=256, parallel_min=256))
    _check_owned(q, results, owners)
    assert all(st["sched_launches"] < st["epochs"] for st in stats), [(st["epochs"], st["sched_launches"], st["stream_closes"], st["kernel_launches"], st["grid"], st["block"]) for st in stats]


def test_cross_rank_write_after_read(B):
    """WAR across ranks: X (rank 0) is read by rank 1 (COPY X->Y), then
    overwritten by rank 0 right away; rank 1 must still see the old X.  Also
    RAW the other way (AXPY Y->Z on rank 0 reads Y from rank 1).  4 MiB
    buffers, 24 rounds, three ranks."""
    from tests import xrank
    n = 1 << 20
    rng = np.random.default_rng(W.SEED_BASE + 90)
    bufs = [W.unit_interval_floats(rng, n) for _ in range(4)]
    rows = []
    for i in range(24):
        f = float(np.float32(0.9 + 0.2 * rng.random()))
        rows += [(W.SCAL, f, 0, -1, -1, -1),          # X *= f        (rank 0)
                 (W.COPY, 0.0, 0, -1, 1, -1),         # Y = X          (rank 1 reads X)
                 (W.SCAL, 1.0 / f, 0, -1, -1, -1),    # X *= 1/f      (rank 0, after rank 1's copy)
                 (W.AXPY, 0.5, 1, -1, 2, -1),         # Z += 0.5 Y     (rank 2 reads Y)
                 (W.SCAL, 0.75, 1, -1, -1, -1),       # Y *= 0.75      (rank 1)
                 (W.COPY, 0.0, 2, -1, 3, -1)]         # W = Z          (rank 0 reads Z)
    p = W.Program(bufs, [0, 0, 0, 0], W._tasks(len(rows)), name="cross-rank WAR/RAW")
    for i, r in enumerate(rows):
        p.tasks[i] = r
    results, stats, owners = xrank.run(p, nranks=3, owners=[0, 1, 2, 0])
    _check_owned(p, results, owners)


def test_cross_rank_read_after_long_write(B):
    """RAW across ranks: rank 0 runs a long unfused chain on X (64 MiB x 48
    dependent scalings) and rank 1 copies X right after it was submitted: the
    copy must wait for the chain's last scaling on rank 0's stream."""
    from tests import xrank
    n = 1 << 24
    rng = np.random.default_rng(W.SEED_BASE + 91)
    bufs = [W.unit_interval_floats(rng, n), np.zeros(n, np.float32)]
    rows = [(W.SCAL, float(np.float32(0.9 + 0.2 * rng.random())), 0, -1, -1, -1) for _ in range(48)]
    rows.append((W.COPY, 0.0, 0, -1, 1, -1))
    p = W.Program(bufs, [0, 0], W._tasks(len(rows)), name="cross-rank RAW after a long chain")
    for i, r in enumerate(rows):
        p.tasks[i] = r
    results, stats, owners = xrank.run(p, nranks=2, owners=[0, 1], batch=False, flags=B.BT_FLAG_NO_FUSION)
    _check_owned(p, results, owners)


def _gated_program():
    """X (rank 0) scaled, copied into Y (rank 1 reads X: RAW across ranks), then
    scaled again (rank 0 overwrites what rank 1 read: WAR across ranks)."""
    n = 1 << 20
    rng = np.random.default_rng(W.SEED_BASE + 93)
    bufs = [W.unit_interval_floats(rng, n), np.zeros(n, np.float32)]
    rows = [(W.SCAL, np.float32(3.14), 0, -1, -1, -1), (W.COPY, 0.0, 0, -1, 1, -1),
            (W.SCAL, np.float32(0.5), 0, -1, -1, -1)]
    p = W.Program(bufs, [0, 0], W._tasks(len(rows)), name="gated cross-rank RAW/WAR")
    for i, r in enumerate(rows):
        p.tasks[i] = r
    return p


@pytest.mark.parametrize("gate_rank", [0, 1])
def test_cross_rank_gated_orderings(B, gate_rank):
    """bt_debug_gate holds one rank's stream for 0.5 s: the owner's (rank 0:
    its SCAL before the copy is late -- the reader's copy must wait for it,
    RAW) or the reader's (rank 1: its copy is late -- the owner's next SCAL of
    X must wait for it, WAR).  Y must hold 3.14 * X either way."""
    from tests import xrank
    p = _gated_program()
    results, stats, owners = xrank.run(p, nranks=2, owners=[0, 1], gate=(gate_rank, 0.5), batch=False)
    _check_owned(p, results, owners)


@pytest.mark.parametrize("mutant,gate_rank", [("BT_COMM_MUTANT_NO_RAW", 0), ("BT_COMM_MUTANT_NO_WAR", 1)])
def test_cross_rank_gated_mutants_fail(B, tmp_path, mutant, gate_rank):
    """Test sensitivity: a library built without the RAW (resp. WAR) stream
    ordering of cross-rank reads must FAIL the gated test above on one GPU."""
    from paper_1304_0878_b200 import build
    from tests import xrank
    lib = build.build(out=str(tmp_path / "libbtask_mutant.so"), defines=[mutant])
    p = _gated_program()
    results, stats, owners = xrank.run(p, nranks=2, owners=[0, 1], gate=(gate_rank, 0.5), batch=False,
                                       lib_path=lib)
    with pytest.raises(AssertionError):
        _check_owned(p, results, owners)


@pytest.mark.parametrize("kernel", ["auto", "sw", "rw", "wq"])
@pytest.mark.parametrize("max_fused", [1024, 256, 7])
def test_long_chain_max_fused(B, kernel, max_fused):
    """1,000 chained SCALs on one ragged 4,099-element vector: fused into items
    of up to max_fused factors (1,024 = the kernels' shared-memory factor
    capacity), each with every rounding in submission order."""
    rng = np.random.default_rng(W.SEED_BASE + 92)
    x = W.unit_interval_floats(rng, 4099)
    f = W.sweep_factors(rng, 1000)
    p = W.sweep_program(x.shape[0], 1, f, x, name="1000-chain")
    stats = compare_program(p, max_fused=max_fused, flags=KERNELS[kernel])
    assert stats["items"] == -(-1000 // max_fused)


@pytest.mark.parametrize("kernel", ["auto", "sw", "rw", "wq"])
def test_item_with_many_successors(B, kernel):
    """An item with more successors than the descriptor's count field holds
    (8,191: the escaped count precedes the successor list, device_abi.h DItem):
    X is scaled, read by 9,000 AXPYs into the tiles of Y (RAW fan-out), then
    scaled again (WAR fan-in of 9,000 predecessors)."""
    rng = np.random.default_rng(W.SEED_BASE + 98)
    n, nt = 256, 9000
    x = W.unit_interval_floats(rng, n)
    y = W.unit_interval_floats(rng, n * nt)
    rows = [(W.SCAL, np.float32(1.5), 0, -1, -1, -1)]
    rows += [(W.AXPY, np.float32(0.25), 0, -1, 1, t) for t in range(nt)]
    rows += [(W.SCAL, np.float32(0.5), 0, -1, -1, -1)]
    p = W.Program([x, y], [0, nt], W._tasks(len(rows)), name="fan-out 9,000")
    for i, r in enumerate(rows):
        p.tasks[i] = r
    stats = compare_program(p, flags=KERNELS[kernel])
    assert stats["edges"] >= 2 * nt, stats


def test_one_element_tiles(B):
    """Degenerate partitions: 1-element tiles (nparts = nx) and 3-element tiles
    (every 256-bit vector path falls back to the scalar head/tail), with
    SCAL/AXPY/COPY across tiles of two buffers."""
    rng = np.random.default_rng(W.SEED_BASE + 93)
    for nx, nparts in ((777, 777), (3 * 500 + 2, 500)):
        bufs = [W.unit_interval_floats(rng, nx), W.unit_interval_floats(rng, nx)]
        rows = []
        lens = [len(range(*W_tile(nx, nparts, t))) for t in range(nparts)]
        for _ in range(3000):
            kind = int(rng.integers(0, 3))
            b0, t0 = int(rng.integers(0, 2)), int(rng.integers(0, nparts))
            if kind == 0:
                rows.append((W.SCAL, float(np.float32(0.9 + 0.2 * rng.random())), b0, t0, -1, -1))
                continue
            same = [t for t in range(nparts) if lens[t] == lens[t0]]
            t1 = int(rng.choice(same))
            b1 = 1 - b0
            if kind == 1:
                rows.append((W.AXPY, float(np.float32(rng.uniform(-0.5, 0.5))), b0, t0, b1, t1))
            else:
                rows.append((W.COPY, 0.0, b0, t0, b1, t1))
        p = W.Program(bufs, [nparts, nparts], W._tasks(len(rows)), name=f"{nparts} tiles over {nx}")
        for i, r in enumerate(rows):
            p.tasks[i] = r
        compare_program(p)


def W_tile(nx, nparts, t):
    off, n = oracle.model.tile_range(nx, nparts, t)
    return off, off + n


def test_two_runtimes_interleaved(B):
    """Two runtimes in one process on one GPU (own streams, pools, epochs):
    their programs are submitted interleaved and each matches the oracle."""
    from paper_1304_0878_b200.programs import Session
    progs = [W.random_small_program(4100 + i, max_tasks=40, max_elems=3000) for i in range(2)]
    with B.Runtime(flags=B.BT_FLAG_NO_FUSION) as r0, B.Runtime(host_threads=3) as r1:
        sess = [Session(r0, progs[0]), Session(r1, progs[1])]
        for s_ in sess:
            s_.submit(batch=False)
        r1.wait()
        r0.wait()
        outs = [s_.finish() for s_ in sess]
    for p, out in zip(progs, outs):
        for b, (o, e) in enumerate(zip(out, oracle.run(p))):
            assert_bits_equal(o, e, f"{p.name} buffer {b}")
