"""Host-side tests (no GPU): the C ABI loads and exports every declared symbol,
the dependency builder enforces exactly the oracle's conflict relation, and
the ABI's error conventions."""
import ctypes
import errno
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import workloads as W
from paper_1304_0878_b200 import build as pbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "btask.h")


@pytest.fixture(scope="module")
def B():
    pbuild.build()
    from paper_1304_0878_b200 import btask
    return btask


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(bt_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol(B):
    names = declared_functions()
    assert len(names) >= 25
    out = subprocess.check_output(["nm", "-D", "--defined-only", B.LIB_PATH], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(B.EXPORTED) == set(names), set(names) ^ set(B.EXPORTED)


def test_library_is_sm100a(B):
    out = subprocess.check_output(["cuobjdump", "--list-elf", B.LIB_PATH], text=True)
    assert "sm_100a" in out


def test_init_without_gpu_is_enodev_unless_host_only(B):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = B.bt_config()
    B.bt_config_init(ctypes.byref(cfg))
    h = ctypes.c_void_p()
    assert B.bt_init(ctypes.byref(cfg), ctypes.byref(h)) == -errno.ENODEV
    cfg.flags = B.BT_FLAG_HOST_ONLY
    assert B.bt_init(ctypes.byref(cfg), ctypes.byref(h)) == 0
    assert B.bt_task_wait_for_all(h) == -errno.ENODEV           # nothing executes on the CPU
    assert B.bt_shutdown(h) == 0


def test_init_rejects_two_forced_kernels(B):
    """BT_FLAG_KERNEL_* (testing): at most one scheduler variant may be forced."""
    cfg = B.bt_config()
    B.bt_config_init(ctypes.byref(cfg))
    h = ctypes.c_void_p()
    cfg.flags = B.BT_FLAG_HOST_ONLY | B.BT_FLAG_KERNEL_SW | B.BT_FLAG_KERNEL_WQ
    assert B.bt_init(ctypes.byref(cfg), ctypes.byref(h)) == -errno.EINVAL
    cfg.flags = B.BT_FLAG_HOST_ONLY | B.BT_FLAG_KERNEL_WQ
    assert B.bt_init(ctypes.byref(cfg), ctypes.byref(h)) == 0
    assert B.bt_shutdown(h) == 0


def test_comm_init_conventions_without_gpu(B):
    """bt_comm_init (cross-rank reads) needs a GPU runtime with nranks >= 2."""
    cfg = B.bt_config()
    B.bt_config_init(ctypes.byref(cfg))
    h = ctypes.c_void_p()
    cfg.flags = B.BT_FLAG_HOST_ONLY
    cfg.nranks, cfg.rank = 2, 1
    assert B.bt_init(ctypes.byref(cfg), ctypes.byref(h)) == 0
    assert B.bt_comm_init(h, b"/bt-test-host") == -errno.ENODEV
    assert "host-only" in B.bt_last_error(h).decode()
    assert B.bt_shutdown(h) == 0


def host_rt(B, **kw):
    return B.Runtime(flags=B.BT_FLAG_HOST_ONLY | kw.pop("flags", 0), **kw)


def snapshot_program(B, program, **kw):
    from paper_1304_0878_b200.programs import Session
    batch = kw.pop("batch", True)
    rt = host_rt(B, **kw)
    s = Session(rt, program)
    s.submit(batch=batch)
    snap = rt.dag_snapshot()
    s.finish()
    rt.close()
    return snap


def reach(snap):
    m = snap["nitems"]
    off, succ = snap["succ_off"], snap["succ"]
    R = [set() for _ in range(m)]
    for i in reversed(range(m)):          # successors always have larger ids
        for s in succ[off[i]:off[i + 1]]:
            assert s > i
            R[i].add(int(s))
            R[i] |= R[s]
    return R


def check_dag(program, snap):
    pairs = oracle.conflict_pairs(program)
    ti, tp = snap["task_item"], snap["task_pos"]
    R = reach(snap)
    # sufficiency: every conflicting pair is ordered (same item in chain order, or a path)
    for (i, j) in pairs:
        if ti[i] == ti[j]:
            assert tp[i] < tp[j], (i, j)
        else:
            assert int(ti[j]) in R[ti[i]], (i, j)
    # necessity: each edge joins items holding a conflicting pair
    members = {}
    for t, it in enumerate(ti):
        members.setdefault(int(it), []).append(t)
    off, succ = snap["succ_off"], snap["succ"]
    for p in range(snap["nitems"]):
        for s in succ[off[p]:off[p + 1]]:
            assert any((i, j) in pairs for i in members[p] for j in members[int(s)]), (p, s)
    # fused items: SCALs of one operand, positions in submission order
    t = program.tasks
    for it, ts in members.items():
        assert [int(tp[x]) for x in ts] == list(range(len(ts)))
        if len(ts) > 1:
            assert all(t["codelet"][x] == W.SCAL for x in ts)
            assert len({(int(t["b0"][x]), int(t["t0"][x])) for x in ts}) == 1
    assert snap["item_npred"].tolist() == [
        sum(1 for p in range(snap["nitems"]) if q in succ[off[p]:off[p + 1]]) for q in range(snap["nitems"])]


@pytest.mark.parametrize("fusion", [True, False])
@pytest.mark.parametrize("threads,pmin", [(1, 0), (1, 1), (4, 1), (3, 2)])
def test_builder_matches_conflict_relation_random(B, fusion, threads, pmin):
    """Sequential builder (1 thread) and the parallel SCAL-run lanes (forced on
    every run of >= pmin SCALs) both enforce exactly the conflict relation."""
    for seed in range(150):
        p = W.random_small_program(seed, max_tasks=10)
        snap = snapshot_program(B, p, flags=0 if fusion else B.BT_FLAG_NO_FUSION, host_threads=threads,
                                parallel_min=pmin)
        assert snap["ntasks"] == p.ntasks
        check_dag(p, snap)


@pytest.mark.parametrize("fusion", [True, False])
def test_parallel_lanes_long_scal_runs(B, fusion):
    """Long SCAL runs over partitioned buffers, split by AXPY/COPY tasks that
    tie tiles together, built by 5 lanes; max_fused forces chain splits."""
    rng = np.random.default_rng(77)
    for rep in range(6):
        nbuf, nparts, n = 3, 7, 70
        bufs = [W.unit_interval_floats(rng, n) for _ in range(nbuf)]
        rows = []
        for blk in range(4):
            for _ in range(int(rng.integers(20, 60))):
                b = int(rng.integers(0, nbuf))
                rows.append((W.SCAL, np.float32(rng.uniform(0.5, 2)), b, int(rng.integers(0, nparts)), -1, -1))
            b0, b1 = rng.choice(nbuf, 2, replace=False)
            t = int(rng.integers(0, nparts))
            rows.append((W.AXPY if blk % 2 else W.COPY, np.float32(0.25), int(b0), t, int(b1), t))
        tasks = W._tasks(len(rows))
        for i, r in enumerate(rows):
            tasks[i] = r
        p = W.Program(bufs, [nparts] * nbuf, tasks)
        snap = snapshot_program(B, p, flags=0 if fusion else B.BT_FLAG_NO_FUSION, host_threads=5,
                                parallel_min=8, max_fused=4)
        check_dag(p, snap)


def test_builder_single_task_paper_example(B):
    snap = snapshot_program(B, W.c1_single())
    assert snap["nitems"] == 1 and snap["nedges"] == 0


def test_builder_spec_examples(B):
    # RAW, WAR (R, R, W), disjoint handles
    x = np.ones(8, np.float32)
    p = W.Program([x.copy(), x.copy(), x.copy()], [0, 0, 0], W._tasks(3))
    p.tasks[0] = (W.COPY, 0, 0, -1, 1, -1)      # R0 W1
    p.tasks[1] = (W.COPY, 0, 0, -1, 2, -1)      # R0 W2
    p.tasks[2] = (W.SCAL, 2, 0, -1, -1, -1)     # RW0 -> after both readers (WAR)
    snap = snapshot_program(B, p)
    assert snap["nitems"] == 3
    assert snap["item_npred"].tolist() == [0, 0, 2]
    check_dag(p, snap)


def test_fusion_shapes(B):
    # C2 shape at reduced size: 16 sweeps x 8 tiles -> 8 items of k=16, no edges
    p = W.c2_chain(nx=1024, ntiles=8, sweeps=16)
    snap = snapshot_program(B, p)
    assert snap["nitems"] == 8 and snap["nedges"] == 0 and set(snap["item_k"].tolist()) == {16}
    check_dag(p, snap)
    snap = snapshot_program(B, p, flags=B.BT_FLAG_NO_FUSION)
    assert snap["nitems"] == 128 and snap["nedges"] == 120
    check_dag(p, snap)
    # max_fused caps chains: 16 = 5 + 5 + 5 + 1 per tile
    snap = snapshot_program(B, p, max_fused=5)
    assert snap["nitems"] == 8 * 4 and snap["nedges"] == 8 * 3
    check_dag(p, snap)


def test_c3_dag_statistics(B):
    p = W.c3_random_dag(nbuf=64, nx=64, ntasks=10000)
    snap = snapshot_program(B, p)
    # ~2.31 edges per task for this generator (simulated)
    assert 2.0 < snap["nedges"] / 10000 < 2.7
    R = None  # full closure is O(n^2) here; check a sample of conflict pairs instead
    ti = snap["task_item"]
    assert len(set(ti.tolist())) == snap["nitems"]


def test_partition_unpartition_dependencies(B):
    """A whole-vector task after unpartition waits for every tile task, and
    tile tasks after partition wait for the earlier whole-vector task."""
    x = np.ones(10, np.float32)
    rt = host_rt(B)
    h = rt.register_array(x)
    rt.scal(h, 2.0)                        # T0 whole
    subs = rt.partition(h, 3)
    rt.scal(subs[0], 3.0)                  # T1 tile 0 (after T0)
    rt.scal(subs[2], 3.0)                  # T2 tile 2 (after T0)
    rt.unpartition(h)
    rt.scal(h, 5.0)                        # T3 whole (after T1, T2)
    snap = rt.dag_snapshot()
    rt.unregister(h)
    rt.close()
    ti = snap["task_item"]
    R = reach(snap)
    assert int(ti[1]) in R[ti[0]] and int(ti[2]) in R[ti[0]]
    assert int(ti[3]) in R[ti[1]] and int(ti[3]) in R[ti[2]]
    assert int(ti[2]) not in R[ti[1]] and int(ti[1]) not in R[ti[2]]


def test_whole_predecessor_flags(B):
    """Chunk-wise release (device_abi.h K_ITEM_DEPS; bt_dag_view.item_flags):
    an item waits for whole predecessors exactly when some predecessor's
    operand on the handle it was found through starts at another address --
    partition-inherited state (a part other than the first, or the parent of a
    part after unpartition) -- and chunk by chunk otherwise, including across
    operands of AXPY/COPY on the same handles and through a re-partition that
    reuses another parent's freed slots."""
    WHOLE = B.BT_DAG_WHOLE_PREDS
    n = 12
    a, b, c = (np.ones(n, np.float32) for _ in range(3))
    rt = host_rt(B, flags=B.BT_FLAG_NO_FUSION)
    ha, hb, hc = rt.register_array(a), rt.register_array(b), rt.register_array(c)
    rt.scal(ha, 2.0)                 # T0
    rt.axpy(0.5, ha, hb)             # T1: after T0 (a, same base)
    rt.copy(hb, hc)                  # T2: after T1 (b as T1's y, same base)
    rt.scal(ha, 3.0)                 # T3: after T0 (WAW) and T1 (WAR), both through a
    pa = rt.partition(ha, 3)         # parts of 4: part 0 starts at a, parts 1-2 do not
    rt.scal(pa[0], 5.0)              # T4: after T3 through part 0's inherited state, same base
    rt.scal(pa[1], 5.0)              # T5: after T3 through part 1's inherited state, another base
    rt.unpartition(ha)
    rt.scal(ha, 7.0)                 # T6: after T4 (base a) and T5 (base a + 16 bytes)
    pc = rt.partition(hc, 3)         # c's parts
    rt.scal(pc[2], 1.5)              # T7: after T2 (base c) through part 2: another base
    rt.unpartition(hc)
    pb = rt.partition(hb, 3)         # reuses c's freed 3-part slots: b's part 2 has c's part 2's slot id
    rt.scal(pb[2], 1.5)              # T8: after T1/T2 on b (bases b) through part 2 of b: another base
    rt.scal(pb[2], 2.5)              # T9: after T8, same part: same base
    snap = rt.dag_snapshot()
    rt.unpartition(hb)
    for h in (ha, hb, hc):
        rt.unregister(h)
    rt.close()
    ti, fl, npred = snap["task_item"], snap["item_flags"], snap["item_npred"]
    assert snap["nitems"] == 10 and fl.shape == (10,)
    whole = [bool(fl[ti[t]] & WHOLE) for t in range(10)]
    assert whole == [False, False, False, False, False, True, True, True, True, False], whole
    assert [int(npred[ti[t]]) for t in (0, 1, 2, 3, 4, 5, 9)] == [0, 1, 1, 2, 1, 1, 1]


def test_error_conventions(B):
    rt = host_rt(B)
    x = np.ones(16, np.float32)
    h = rt.register_array(x)
    # lookup: exact base only, message of PAPER.md:346
    assert rt.lookup(x.ctypes.data) == h
    with pytest.raises(B.BtError) as ei:
        rt.lookup(x.ctypes.data + 4)
    assert ei.value.code == -errno.ENOENT and "attempt to use unregistered pointer" in str(ei.value)
    # overlapping registration
    with pytest.raises(B.BtError) as ei:
        rt.register(x.ctypes.data + 8, 4)
    assert ei.value.code == -errno.EEXIST
    # wrong modes / scalar size -> EINVAL, "failed to insert task"
    assert rt.insert(B.BT_CL_SCAL, [h], [B.BT_R], 2.0) == -errno.EINVAL
    assert "failed to insert task `vector_scal'" in rt.last_error()
    assert rt.insert(B.BT_CL_SCAL, [h], [B.BT_W], 2.0) == -errno.EINVAL
    assert rt.insert(B.BT_CL_COPY, [h, h], [B.BT_R, B.BT_RW]) == -errno.EINVAL
    assert rt.insert(B.BT_CL_AXPY, [h, h], [B.BT_R, B.BT_RW]) == -errno.EINVAL   # missing scalar
    assert rt.insert(99, [h], [B.BT_RW], 1.0) == -errno.EINVAL
    y = np.ones(8, np.float32)
    hy = rt.register_array(y)
    assert rt.insert(B.BT_CL_AXPY, [h, hy], [B.BT_R, B.BT_RW], 1.0) == -errno.EINVAL   # lengths differ
    # partitioned parent -> EBUSY; sub-handles fine
    subs = rt.partition(h, 4)
    assert rt.insert(B.BT_CL_SCAL, [h], [B.BT_RW], 2.0) == -errno.EBUSY
    assert rt.insert(B.BT_CL_SCAL, [subs[1]], [B.BT_RW], 2.0) == 0
    with pytest.raises(B.BtError) as ei:
        rt.unregister(h)
    assert ei.value.code == -errno.EBUSY
    rt.unpartition(h)
    # stale sub-handle after unpartition, stale handle after unregister
    assert rt.insert(B.BT_CL_SCAL, [subs[1]], [B.BT_RW], 2.0) == -errno.ENOENT
    rt.unregister(h)
    assert rt.insert(B.BT_CL_SCAL, [h], [B.BT_RW], 2.0) == -errno.ENOENT
    with pytest.raises(B.BtError) as ei:
        rt.unregister(h)                                  # double unregister
    assert ei.value.code == -errno.ENOENT
    rt.unregister(hy)
    # degenerate sizes (nx == 0, nparts == 0 or > nx) are rejected
    z = np.ones(3, np.float32)
    with pytest.raises(B.BtError) as ei:
        rt.register(z.ctypes.data, 0)
    assert ei.value.code == -errno.EINVAL
    hz = rt.register_array(z)
    for bad in (0, 4):
        with pytest.raises(B.BtError) as ei:
            rt.partition(hz, bad)
        assert ei.value.code == -errno.EINVAL
    assert len(rt.partition(hz, 3)) == 3          # one element per part is fine
    with pytest.raises(B.BtError) as ei:
        rt.partition(hz, 2)                        # already partitioned
    assert ei.value.code == -errno.EBUSY
    rt.unpartition(hz)
    rt.unregister(hz)
    # re-registration of the same memory is allowed after unregister
    h2 = rt.register_array(x)
    rt.unregister(h2)
    rt.close()


def test_shutdown_with_live_handles_is_ebusy(B):
    rt = host_rt(B)
    x = np.ones(4, np.float32)
    h = rt.register_array(x)
    with pytest.raises(B.BtError) as ei:
        rt.close()
    assert ei.value.code == -errno.EBUSY
    rt.unregister(h)
    rt.close()


def test_batch_equals_single_inserts(B):
    for seed in range(30):
        p = W.random_small_program(seed + 1000, max_tasks=10)
        a = snapshot_program(B, p, batch=True)
        b = snapshot_program(B, p, batch=False)
        for k in ("task_item", "task_pos", "item_k", "item_npred", "succ_off", "succ"):
            assert np.array_equal(a[k], b[k]), k


def test_batch_marshalling(B):
    """insert_batch passes the arrays' addresses as they are (strided or
    mistyped inputs are converted first) and rejects arrays of different
    lengths before the call (the C ABI takes one count for all of them)."""
    x = np.ones(64, np.float32)
    rt = host_rt(B)
    h = rt.register_array(x)
    subs = rt.partition(h, 4)
    t = W._tasks(8)
    t["codelet"] = W.SCAL
    t["scalar"] = np.float32(2.0)
    hs = np.asarray(subs, np.uint64)[np.arange(8) % 4]
    assert rt.insert_batch(t["codelet"], t["scalar"], hs) == 8      # strided fields of a structured array
    assert rt.insert_batch(np.ones(8, np.int64), np.ones(8), hs.astype(np.int64)) == 8   # converted
    with pytest.raises(ValueError):
        rt.insert_batch(np.ones(8, np.int32), np.ones(7, np.float32), hs)
    with pytest.raises(ValueError):
        rt.insert_batch(np.ones(8, np.int32), np.ones(8, np.float32), hs, hs[:5])
    snap = rt.dag_snapshot()
    assert snap["ntasks"] == 16
    rt.unpartition(h)
    rt.unregister(h)
    rt.close()


def test_rank_filter_and_cross_rank_error(B):
    x = np.ones(64, np.float32)
    y = np.ones(64, np.float32)
    rt = host_rt(B, rank=1, nranks=2)
    hx, hy = rt.register_array(x), rt.register_array(y)
    subs = rt.partition(hx, 4)
    rt.distribute_block(hx)                    # tiles 0,1 -> rank 0; 2,3 -> rank 1
    for t in range(4):
        rt.scal(subs[t], 2.0)
    rt.set_rank(hy, 0)
    assert rt.insert(B.BT_CL_SCAL, [hy], [B.BT_RW], 2.0) == 0   # runs on rank 0: skipped here
    snap = rt.dag_snapshot()
    assert snap["task_item"].tolist()[:2] == [0xFFFFFFFF] * 2
    assert snap["nitems"] == 2
    rt.set_rank(hy, 1)
    rt.unpartition(hx)
    rt.set_rank(hx, 0)
    assert rt.insert(B.BT_CL_AXPY, [hx, hy], [B.BT_R, B.BT_RW], 1.0) == -errno.EXDEV
    rt.unregister(hx)
    rt.unregister(hy)
    rt.close()


def test_stats_struct_matches_header(B):
    """The binding's bt_stats mirrors the header's field order (ABI drift guard)."""
    src = open(HEADER).read()
    body = re.search(r"typedef struct bt_stats \{(.*?)\} bt_stats;", src, flags=re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"\b(\w+)\s*;", body)
    assert [f for f, _ in B.bt_stats._fields_] == fields


def test_device_abi_layout(tmp_path):
    """Host-written offsets of the device ABI (runtime.cpp writes StreamCtl's
    header by offset; DirectArgs travels as a kernel parameter, <= 32,764 bytes)."""
    src = tmp_path / "abi.cpp"
    src.write_text('#include <cstdio>\n#include <cstddef>\n#include "device_abi.h"\nusing namespace bt;\n'
                   'int main() { printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(EpochArgs), offsetof(StreamCtl, nsub), '
                   'offsetof(StreamCtl, subs), sizeof(StreamCtl), sizeof(DirectArgs), sizeof(DirectItem)); }\n')
    exe = tmp_path / "abi"
    subprocess.check_call(["g++", "-std=c++17", "-I", os.path.join(ROOT, "paper_1304_0878_b200", "csrc"), str(src),
                           "-o", str(exe)])
    ea, nsub, subs, sc, da, di = map(int, subprocess.check_output([str(exe)], text=True).split())
    assert nsub == 20 and subs == 64 and sc % 64 == 0 and sc >= 64 + 16 * ea
    assert da <= 32764 and di == 48   # kernel parameter limit (CUDA >= 12.1); DirectItem: a strided group


def test_library_contains_every_kernel(B):
    """sm_100a SASS for the persistent kernels, the stream launch, the direct
    launch and the set-up kernel."""
    out = subprocess.check_output(["cuobjdump", "--list-text", B.LIB_PATH], text=True)
    for k in ("scheduler_kernel_sw", "scheduler_kernel_sws", "scheduler_kernel_rw", "scheduler_kernel_wq",
              "scheduler_kernel_swp", "direct_kernel", "stage_kernel", "flag_wait_kernel", "flag_write_kernel",
              "gate_kernel"):
        assert k in out, k


def test_descriptor_packing(tmp_path):
    """The 32-byte work-item descriptor (device_abi.h DItem): the packed meta
    word round-trips kind, single-predecessor bit, k up to 2047 and successor
    counts, escaping at 8,191; single-unit test without division."""
    src = tmp_path / "meta.cpp"
    src.write_text(
        '#include <cstdio>\n#include <initializer_list>\n#include "device_abi.h"\nusing namespace bt;\n'
        'int main() { int bad = 0; DItem d{};\n'
        ' for (unsigned kind = 1; kind <= 3; ++kind) for (int sp = 0; sp < 2; ++sp)\n'
        '  for (unsigned k : {1u, 2u, 64u, 1024u, 2047u}) for (unsigned long ns : {0ul, 1ul, 2ul, 8190ul, 8191ul, 9000ul, 1ul << 20}) {\n'
        '   d.meta = make_meta(kind, sp, k, ns);\n'
        '   unsigned f = d.nsucc_field();\n'
        '   bad += d.kind() != kind || d.single_pred() != (bool)sp || d.k() != k ||\n'
        '          f != (ns < K_NSUCC_ESC ? ns : K_NSUCC_ESC); }\n'
        ' bad += units_of(1, 16384) != 1 || units_of(16384, 16384) != 1 || units_of(16385, 16384) != 2 ||\n'
        '        units_of(100, 24) != 5 || units_of(0xFFFFFFFFu, 8) != 0x20000000u;\n'
        ' printf("%d %zu\\n", bad, sizeof(DItem)); return 0; }\n')
    exe = tmp_path / "meta"
    subprocess.check_call(["g++", "-std=c++17", "-I", os.path.join(ROOT, "paper_1304_0878_b200", "csrc"), str(src),
                           "-o", str(exe)])
    bad, size = map(int, subprocess.check_output([str(exe)], text=True).split())
    assert bad == 0 and size == 32


def test_register_rejects_vectors_of_2_32_elements(B):
    """Descriptors hold 32-bit lengths (reading R22): 2^32 elements -> -EINVAL."""
    rt = B.Runtime(flags=B.BT_FLAG_HOST_ONLY)
    h = B.bt_handle()
    rc = B.bt_vector_data_register(rt.rt, ctypes.byref(h), 0, None, 1 << 32, 4)
    assert rc == -errno.EINVAL and "2^32" in rt.last_error()
    assert B.bt_vector_data_register(rt.rt, ctypes.byref(h), 0, None, (1 << 32) - 1, 4) == 0
    assert B.bt_data_unregister(rt.rt, h.value) == 0
    rt.close()
