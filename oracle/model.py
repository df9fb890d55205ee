"""Program interpretation for the oracle (TEST INFRASTRUCTURE ONLY).

Plain, slow, obviously-correct definitions:

* ``tile_range``     -- the vector block filter (section 5.1, lines
  944-966: "partitioned into smaller pieces"; sub-data t of n), remainder
  rule of DESIGN.md reading R10: the first nx mod n tiles get one extra
  element.
* ``run``            -- execute the tasks one by one in submission order
  ("compiling the annotated program without StarPU's
  compiler plug-in still leads a valid sequential program")
  by calling ``oracle_run`` in oracle.c.
* ``access_sets``    -- which elements each task reads / writes: SCAL x:RW
  (PAPER.md:136 ``.modes = { STARPU_RW }``), AXPY x:R y:RW, COPY x:R y:W
  (BASELINE.json configs[2]); two operands naming the same elements OR their
  modes (reading R6).
* ``conflict_pairs`` -- the definition of a dependency (PAPER.md:118-120:
  "These access modes, along with the sequence of task invocations, allows
  StarPU to determine at run-time the dependency graph"): tasks i < j
  conflict iff they touch a common element of a common buffer and at least
  one of the two accesses writes it.  Any execution that runs every
  conflicting pair in submission order yields the sequential result; this is
  what the product's dependency builder must (transitively) enforce.
"""
from __future__ import annotations

import ctypes
import enum
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fno-unsafe-math-optimizations",
           "-std=c11", "-fPIC", "-shared", "-Wall", "-Werror", "-fopenmp"]

SCAL, AXPY, COPY = 1, 2, 3          # oracle.h ORACLE_SCAL / _AXPY / _COPY


class AccessMode(enum.IntFlag):
    R = 1
    W = 2
    RW = 3


def build_lib(force: bool = False) -> str:
    """Compile oracle.c with gcc (no fast-math, no FP contraction)."""
    stale = (not os.path.exists(_LIB) or
             os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC),
                                          os.path.getmtime(os.path.join(_HERE, "oracle.h"))))
    if force or stale:
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", *_CFLAGS, _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_lib())
        i64p = ctypes.POINTER(ctypes.c_int64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        f32p = ctypes.POINTER(ctypes.c_float)
        _lib.oracle_run.argtypes = [ctypes.c_int64, i32p, f32p, i32p, i64p, i64p, i32p, i64p, i64p,
                                    ctypes.POINTER(f32p)]
        _lib.oracle_run.restype = ctypes.c_int
        _lib.oracle_run_omp.argtypes = _lib.oracle_run.argtypes + [ctypes.c_int]
        _lib.oracle_run_omp.restype = ctypes.c_int
        _lib.oracle_scal_chain.argtypes = [f32p, ctypes.c_int64, f32p, ctypes.c_int64]
        _lib.oracle_scal_chain.restype = None
        _lib.oracle_flt_eval_method.restype = ctypes.c_int
    return _lib


def tile_range(nx: int, nparts: int, t: int) -> tuple[int, int]:
    """(offset, length) of sub-data t when nx elements are split into nparts
    blocks; the first nx % nparts blocks hold one extra element (R10)."""
    if not (0 <= t < nparts):
        raise IndexError(f"tile {t} of {nparts}")
    base, extra = divmod(nx, nparts)
    off = t * base + min(t, extra)
    return off, base + (1 if t < extra else 0)


def _operand(program, b: int, t: int) -> tuple[int, int]:
    nx = program.buffers[b].shape[0]
    if t < 0:
        return 0, nx
    return tile_range(nx, program.nparts[b], t)


def resolve(program):
    """Per-task (buffer, offset, length) of both operands, as int arrays."""
    n = program.ntasks
    off0 = np.zeros(n, np.int64); len0 = np.zeros(n, np.int64)
    off1 = np.zeros(n, np.int64); len1 = np.zeros(n, np.int64)
    tasks = program.tasks
    # Vectorised where every buffer is partitioned uniformly (large configs);
    # the formula is tile_range's, applied element-wise.
    for b, buf in enumerate(program.buffers):
        nx = buf.shape[0]
        p = program.nparts[b]
        for col, off, ln in (("0", off0, len0), ("1", off1, len1)):
            sel = tasks["b" + col] == b
            if not sel.any():
                continue
            tt = tasks["t" + col][sel].astype(np.int64)
            if p == 0:
                if (tt >= 0).any():
                    raise ValueError("tile index on an unpartitioned buffer")
                off[sel] = 0
                ln[sel] = nx
            else:
                if ((tt < 0) | (tt >= p)).any():
                    raise ValueError("tile index out of range / whole-buffer access to a partitioned buffer")
                base, extra = divmod(nx, p)
                off[sel] = tt * base + np.minimum(tt, extra)
                ln[sel] = base + (tt < extra)
    return off0, len0, off1, len1


def run_tasks(buffers: list, codelet, scalar, b0, off0, len0, b1, off1, len1, threads: int = 0) -> None:
    """Low-level: execute tasks in order on the given float32 host buffers (in place).
    threads > 0: the OpenMP variant (element-parallel inside each task)."""
    L = lib()
    for b in buffers:
        assert b.dtype == np.float32 and b.flags.c_contiguous
    c = np.ascontiguousarray(codelet, np.int32)
    s = np.ascontiguousarray(scalar, np.float32)
    arrs = [np.ascontiguousarray(a, np.int32 if i in (0, 3) else np.int64)
            for i, a in enumerate([b0, off0, len0, b1, off1, len1])]
    arrs[3] = np.where(arrs[3] < 0, 0, arrs[3]).astype(np.int32)     # unused operand 1 of SCAL
    f32p = ctypes.POINTER(ctypes.c_float)
    ptrs = (f32p * max(1, len(buffers)))(*[b.ctypes.data_as(f32p) for b in buffers])
    P = lambda a, t: a.ctypes.data_as(ctypes.POINTER(t))
    args = (len(c), P(c, ctypes.c_int32), P(s, ctypes.c_float),
            P(arrs[0], ctypes.c_int32), P(arrs[1], ctypes.c_int64), P(arrs[2], ctypes.c_int64),
            P(arrs[3], ctypes.c_int32), P(arrs[4], ctypes.c_int64), P(arrs[5], ctypes.c_int64), ptrs)
    rc = L.oracle_run_omp(*args, threads) if threads > 0 else L.oracle_run(*args)
    if rc != 0:
        raise ValueError("oracle_run rejected the program")


def run(program, buffers: list | None = None, threads: int = 0) -> list:
    """Final contents of every buffer after all tasks, in submission order
    (threads > 0: the OpenMP variant, timing only)."""
    bufs = program.copy_buffers() if buffers is None else buffers
    off0, len0, off1, len1 = resolve(program)
    t = program.tasks
    run_tasks(bufs, t["codelet"], t["scalar"], t["b0"], off0, len0, t["b1"], off1, len1, threads=threads)
    return bufs


def scal_chain(x: np.ndarray, factors: np.ndarray) -> np.ndarray:
    """Element-major chain of SCALs: each element times f_1..f_k in order."""
    y = np.array(x, dtype=np.float32, copy=True)
    f = np.ascontiguousarray(factors, np.float32)
    f32p = ctypes.POINTER(ctypes.c_float)
    lib().oracle_scal_chain(y.ctypes.data_as(f32p), y.shape[0], f.ctypes.data_as(f32p), f.shape[0])
    return y


def access_sets(program) -> list:
    """Per task: list of (buffer, lo, hi, AccessMode) with identical ranges merged."""
    off0, len0, off1, len1 = resolve(program)
    out = []
    for i, row in enumerate(program.tasks):
        c = int(row["codelet"])
        acc = {}
        r0 = (int(row["b0"]), int(off0[i]), int(off0[i] + len0[i]))
        if c == SCAL:
            acc[r0] = AccessMode.RW
        else:
            r1 = (int(row["b1"]), int(off1[i]), int(off1[i] + len1[i]))
            acc[r0] = AccessMode.R
            acc[r1] = acc.get(r1, AccessMode(0)) | (AccessMode.RW if c == AXPY else AccessMode.W)
        out.append([(b, lo, hi, m) for (b, lo, hi), m in acc.items()])
    return out


def conflict_pairs(program) -> set:
    """All (i, j), i < j, that touch a common element with >= 1 writer (O(n^2); small programs)."""
    acc = access_sets(program)
    pairs = set()
    for j in range(len(acc)):
        for i in range(j):
            hit = False
            for (bi, loi, hii, mi) in acc[i]:
                for (bj, loj, hij, mj) in acc[j]:
                    if bi == bj and loi < hij and loj < hii and ((mi | mj) & AccessMode.W):
                        hit = True
            if hit:
                pairs.add((i, j))
    return pairs
