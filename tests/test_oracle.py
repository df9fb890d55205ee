"""Pins for the CPU oracle (no GPU).  Each test ties the oracle to something
other than itself: the paper's worked example, exact-rational rounding
(tests/exact_f32.py), closed forms, numpy as a library special case, and
brute force over every dependency-respecting order of small programs.
"""
import hashlib
import itertools
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W
from tests import exact_f32 as X
from tests.golden import load

PINS = load("scal_pins.txt")
F314 = np.float32(3.14)


def hx(v):
    return f"{X.f32_bits(v):08X}"


def one_scal(x, f):
    p = W.Program([np.array(x, np.float32)], [0], W._tasks(1))
    p.tasks[0] = (W.SCAL, np.float32(f), 0, -1, -1, -1)
    return oracle.run(p)[0]


def test_build_flags_no_excess_precision():
    assert oracle.lib().oracle_flt_eval_method() == 0


def test_factor_314_bits():
    # R1: decimal 3.14 rounded to binary32, directly (exact rational) and via double
    assert PINS["factor_3.14"][0][0] == "4048F5C3"
    assert hx(X.round_f32(Fraction("3.14"))) == "4048F5C3"
    assert hx(F314) == "4048F5C3"


def test_paper_example_1_to_8():
    """PAPER.md:201-214 with SPEC.md:645's 1..8 vector."""
    y = one_scal(np.arange(1, 9), F314)
    got = [hx(v) for v in y]
    assert got == PINS["paper_example_1to8"][0]
    assert got == [hx(X.mul(np.float32(i), F314)) for i in range(1, 9)]
    # [1,2,3] x 3.14 -> [3.14, 6.28, 9.42]: the nearest floats
    assert [float(v) for v in y[:3]] == [float(np.float32(s)) for s in ("3.14", "6.28", "9.42")]


@pytest.mark.parametrize("start,key", [(1, "c1"), (0, "c1_from0")])
def test_c1_hash_and_exact(start, key):
    x = np.arange(start, start + 1024, dtype=np.float32)
    y = one_scal(x, F314)
    assert hashlib.sha256(y.astype("<f4").tobytes()).hexdigest()[:16] == PINS[f"{key}_sha256_prefix"][0][0]
    assert hx(y[-1]) == PINS[f"{key}_last"][0][0]
    exact = np.array([X.mul(v, F314) for v in x], np.float32)
    assert np.array_equal(y.view(np.uint32), exact.view(np.uint32))


def test_c1_program_generator_matches_paper():
    p = W.c1_single()
    assert p.buffers[0].shape == (1024,) and p.tasks.shape == (1,)
    y = oracle.run(p)[0]
    assert hashlib.sha256(y.tobytes()).hexdigest()[:16] == PINS["c1_sha256_prefix"][0][0]


@pytest.mark.parametrize("k", [2, 3, 16, 64])
def test_chain_of_314(k):
    """k sequential scalings of 1.0 (iterated product, not round(f^k))."""
    p = W.sweep_program(1, 1, np.full(k, F314, np.float32), np.ones(1, np.float32))
    y = oracle.run(p)[0][0]
    assert hx(y) == PINS[f"chain_k{k}"][0][0]
    v = np.float32(1.0)
    for _ in range(k):
        v = X.mul(v, F314)
    assert hx(y) == hx(v)


def test_chain_not_power_shortcut():
    # round(exact 3.14f^3) differs from the iterated product at k=3 (reading R13)
    exact = X.round_f32(X.f32_to_fraction(F314) ** 3)
    assert hx(exact) != PINS["chain_k3"][0][0]


@pytest.mark.parametrize("j,k", [(1, 16), (-1, 20), (3, 7), (-2, 9)])
def test_power_of_two_chain_is_exact(j, k):
    rng = np.random.default_rng(5)
    x = W.unit_interval_floats(rng, 257)
    p = W.sweep_program(257, 3, np.full(k, np.float32(2.0 ** j), np.float32), x)
    y = oracle.run(p)[0]
    assert np.array_equal(y, (x.astype(np.float64) * 2.0 ** (j * k)).astype(np.float32))


def test_identity_sign_and_zero_factors():
    rng = np.random.default_rng(6)
    x = (W.unit_interval_floats(rng, 100) * np.where(rng.random(100) < .5, -1, 1)).astype(np.float32)
    assert np.array_equal(one_scal(x, 1.0).view(np.uint32), x.view(np.uint32))
    assert np.array_equal(one_scal(x, -1.0).view(np.uint32), (x.view(np.uint32) ^ np.uint32(0x80000000)))
    z = one_scal(x, 0.0)
    assert np.all(z == 0) and np.array_equal(np.signbit(z), np.signbit(x))
    z = one_scal(x, -0.0)
    assert np.all(z == 0) and np.array_equal(np.signbit(z), ~np.signbit(x))


def test_subnormals_preserved():
    for inp, fac, out in PINS["subnormal"]:
        xv = X.bits_to_f32(int(inp, 16))
        fv = X.bits_to_f32(int(fac, 16))
        y = one_scal([xv], fv)[0]
        assert hx(y) == out
        assert hx(X.mul(xv, fv)) == out


def test_overflow_to_inf():
    y = one_scal([np.float32(3e38), np.float32(-3e38)], np.float32(4.0))
    assert np.isposinf(y[0]) and np.isneginf(y[1])
    assert np.isposinf(X.mul(np.float32(3e38), np.float32(4.0)))


def test_scal_matches_exact_rounding_random():
    rng = np.random.default_rng(7)
    x = (rng.standard_normal(300) * 10.0 ** rng.integers(-30, 30, 300)).astype(np.float32)
    f = np.float32(rng.uniform(-3, 3))
    y = one_scal(x, f)
    assert np.array_equal(y.view(np.uint32), np.array([X.mul(v, f) for v in x], np.float32).view(np.uint32))


def test_scal_matches_numpy_library():
    rng = np.random.default_rng(8)
    x = rng.standard_normal(1 << 16).astype(np.float32)
    f = np.float32(0.987654)
    assert np.array_equal(one_scal(x, f).view(np.uint32), (x * f).view(np.uint32))


def _two_buffer_program(x, y, codelet, a):
    p = W.Program([np.array(x, np.float32), np.array(y, np.float32)], [0, 0], W._tasks(1))
    p.tasks[0] = (codelet, np.float32(a), 0, -1, 1, -1)
    return p


def test_axpy_two_roundings_exact():
    rng = np.random.default_rng(9)
    x = rng.standard_normal(400).astype(np.float32)
    y = rng.standard_normal(400).astype(np.float32)
    a = np.float32(0.3141)
    out = oracle.run(_two_buffer_program(x, y, W.AXPY, a))
    assert np.array_equal(out[0], x)                       # x is read-only
    exact = np.array([X.axpy(a, xi, yi) for xi, yi in zip(x, y)], np.float32)
    assert np.array_equal(out[1].view(np.uint32), exact.view(np.uint32))
    # library special case: numpy float32 (no contraction)
    assert np.array_equal(out[1].view(np.uint32), (a * x + y).view(np.uint32))
    # the oracle is not contracting: on these inputs a single-rounding FMA differs somewhere
    fused = np.array([X.fma(a, xi, yi) for xi, yi in zip(x, y)], np.float32)
    assert not np.array_equal(fused.view(np.uint32), exact.view(np.uint32))


def test_copy_is_bit_identity():
    x = np.array([0.0, -0.0, np.inf, -np.inf, 1e-45, 3.14, -2.5], np.float32)
    y = np.full_like(x, 7.0)
    out = oracle.run(_two_buffer_program(x, y, W.COPY, 0.0))
    assert np.array_equal(out[1].view(np.uint32), x.view(np.uint32))


def test_aliasing_axpy_same_handle():
    # reading R6: AXPY(x, x) is y[i] = a*x[i] + x[i] element by element
    x = np.array([1.5, -2.25, 3.0], np.float32)
    p = W.Program([x.copy()], [0], W._tasks(1))
    p.tasks[0] = (W.AXPY, np.float32(0.5), 0, -1, 0, -1)
    out = oracle.run(p)[0]
    assert np.array_equal(out, np.array([X.axpy(0.5, v, v) for v in x], np.float32))


@pytest.mark.parametrize("nx,n", [(10, 3), (64, 4), (7, 7), (1, 1), (1000, 7), (5, 2)])
def test_tile_range_matches_numpy_array_split(nx, n):
    parts = np.array_split(np.arange(nx), n)       # library: first nx % n parts one longer
    for t in range(n):
        off, ln = oracle.tile_range(nx, n, t)
        assert ln == len(parts[t]) and (ln == 0 or off == parts[t][0])


def test_element_major_equals_task_major():
    rng = np.random.default_rng(10)
    x = W.unit_interval_floats(rng, 4096)
    f = W.sweep_factors(rng, 37)
    task_major = oracle.run(W.sweep_program(4096, 16, f, x.copy()))[0]
    assert np.array_equal(oracle.scal_chain(x, f).view(np.uint32), task_major.view(np.uint32))
    tile_major = oracle.run(W.sweep_program(4096, 16, f, x.copy(), order="tile"))[0]
    assert np.array_equal(tile_major.view(np.uint32), task_major.view(np.uint32))


def test_order_of_factors_matters():
    # reading R13: swapping two factors changes bits for some inputs (so the
    # oracle really applies them in submission order)
    rng = np.random.default_rng(11)
    x = W.unit_interval_floats(rng, 4096)
    f = np.array([np.float32(3.14), np.float32(0.7)], np.float32)
    assert not np.array_equal(oracle.scal_chain(x, f), oracle.scal_chain(x, f[::-1]))


# ---- sequential consistency over the conflict relation ----

def _linear_extensions(n, pairs):
    preds = {j: {i for (i, jj) in pairs if jj == j} for j in range(n)}
    for perm in itertools.permutations(range(n)):
        pos = {t: k for k, t in enumerate(perm)}
        if all(pos[i] < pos[j] for (i, j) in pairs):
            yield perm


def _run_in_order(program, order):
    bufs = program.copy_buffers()
    off0, len0, off1, len1 = oracle.model.resolve(program)
    t = program.tasks
    idx = np.array(order, np.int64)
    oracle.run_tasks(bufs, t["codelet"][idx], t["scalar"][idx], t["b0"][idx], off0[idx], len0[idx],
                     t["b1"][idx], off1[idx], len1[idx])
    return b"".join(b.tobytes() for b in bufs)


def test_every_conflict_respecting_order_is_byte_identical():
    """Brute force: for random programs (<= 7 tasks), every linear extension of
    the conflict DAG reproduces submission order byte for byte."""
    checked = 0
    for seed in range(120):
        p = W.random_small_program(seed, max_tasks=7)
        pairs = oracle.conflict_pairs(p)
        ref = _run_in_order(p, range(p.ntasks))
        assert ref == b"".join(b.tobytes() for b in oracle.run(p))
        for order in _linear_extensions(p.ntasks, pairs):
            assert _run_in_order(p, order) == ref
            checked += 1
    assert checked > 500


def test_conflict_relation_is_not_vacuous():
    """Swapping some conflicting pair changes the bytes in many programs, so
    the conflict relation carries real ordering constraints."""
    changed = 0
    for seed in range(120):
        p = W.random_small_program(seed, max_tasks=6)
        ref = _run_in_order(p, range(p.ntasks))
        for (i, j) in oracle.conflict_pairs(p):
            if j == i + 1:
                order = list(range(p.ntasks))
                order[i], order[j] = order[j], order[i]
                if _run_in_order(p, order) != ref:
                    changed += 1
    assert changed > 20


def test_conflict_pairs_small_cases():
    # SPEC.md:420-422 examples: RAW, WAR (R,R,W), disjoint handles
    x = np.ones(4, np.float32)
    p = W.Program([x.copy(), x.copy(), x.copy()], [0, 0, 0], W._tasks(3))
    p.tasks[0] = (W.COPY, 0, 2, -1, 0, -1)     # T0 writes buffer 0 (W)
    p.tasks[1] = (W.COPY, 0, 0, -1, 1, -1)     # T1 reads 0 -> RAW on 0
    p.tasks[2] = (W.SCAL, 2, 2, -1, -1, -1)    # T2 RW on 2: WAR with T0's read of 2
    assert oracle.conflict_pairs(p) == {(0, 1), (0, 2)}
    q = W.Program([x.copy(), x.copy()], [0, 0], W._tasks(3))
    q.tasks[0] = (W.COPY, 0, 0, -1, 1, -1)     # R 0
    q.tasks[1] = (W.AXPY, 1, 0, -1, 1, -1)     # R 0, RW 1
    q.tasks[2] = (W.SCAL, 3, 0, -1, -1, -1)    # W 0 -> after both readers
    assert oracle.conflict_pairs(q) == {(0, 1), (0, 2), (1, 2)}
    r = W.Program([x.copy(), x.copy()], [0, 0], W._tasks(2))
    r.tasks[0] = (W.SCAL, 2, 0, -1, -1, -1)
    r.tasks[1] = (W.SCAL, 2, 1, -1, -1, -1)
    assert oracle.conflict_pairs(r) == set()


def test_partitioned_tiles_do_not_conflict():
    x = np.ones(10, np.float32)
    p = W.Program([x], [3], W._tasks(3))
    p.tasks[0] = (W.SCAL, 2, 0, 0, -1, -1)
    p.tasks[1] = (W.SCAL, 2, 0, 1, -1, -1)
    p.tasks[2] = (W.SCAL, 2, 0, 0, -1, -1)
    assert oracle.conflict_pairs(p) == {(0, 2)}


def test_openmp_variant_equals_sequential():
    """The OpenMP timing variant (element-parallel inside each task, tasks in
    order) is byte-identical to the sequential oracle: on small property
    programs and on C3/C2-shaped programs large enough (>= 65,536 elements per
    task) to take its parallel loops, with 1, 4 and 8 threads."""
    progs = [W.random_small_program(600 + s, max_tasks=10) for s in range(40)]
    progs.append(W.c3_random_dag(nbuf=6, nx=1 << 17, ntasks=60, seed=11))
    progs.append(W.c2_chain(nx=1 << 19, ntiles=4, sweeps=5))
    for p in progs:
        ref = oracle.run(p)
        for th in (1, 4, 8):
            got = oracle.run(p, threads=th)
            for a, b in zip(ref, got):
                assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (p.name, th)
