"""Seeded synthetic task programs shaped like the paper's workloads.

This module is the ONE place shared by the oracle (``oracle/``) and the CUDA
path (``paper_1304_0878_b200``): it only draws random inputs and describes a
program in a neutral form.  It holds none of the method's arithmetic (no
multiply, no dependency rule, no tile-range formula); each side interprets the
description on its own.

Program model (section 2; section 5.1):

* ``buffers``  -- initial float32 contents of each registered vector
  (``starpu_vector_data_register``).
* ``nparts``   -- number of tiles each buffer is partitioned into right after
  registration (0 = used whole).  Tiles follow the block filter of PAPER.md:
  944-966; the range rule is each side's own (reading R10).
* ``tasks``    -- structured array, one row per ``starpu_insert_task`` call in
  submission order: ``codelet`` (SCAL/AXPY/COPY),
  ``scalar`` (the single float VALUE argument, 0 for COPY), and two operands
  ``(b0, t0)``, ``(b1, t1)``: buffer index and tile index (-1 = the whole,
  unpartitioned buffer).  SCAL uses operand 0 only (x:RW); AXPY and COPY read
  operand 0 (x:R) and write operand 1 (y:RW resp. y:W).

Recipes (seed = 13040878 + config index):

* C1  ``c1_single``       1 buffer of 1,024 floats, x[i] = i+1, one SCAL by 3.14f
                          (PAPER.md:205 ``float factor = 3.14``).
* C2  ``c2_chain``        2^24 floats in [1,2) split into 256 tiles; 16 sweeps,
                          sweep-major, each ``SCAL(3.14f; tile t)``.
* C3  ``c3_random_dag``   64 buffers x 2^20 floats in [1,2); 10,000 tasks, each
                          kind with probability 1/3: SCAL f = +-U[0.75,1.25],
                          AXPY a = +-U[1/16,1/2], COPY; x != y uniform.
* C4  ``c4_fine``         15,625 tiles x 1,024 floats; 64 sweeps sweep-major;
                          per-sweep factor f_s = float32(0.9 + 0.2 u_s).
* C5  ``c5_sharded``      2^30 floats in [1,2), 16,384 tiles x 65,536; 64 sweeps
                          with per-sweep factors as C4; tiles owner-computes.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 13040878

# Codelet ids of the neutral description (names only; each side maps them).
SCAL, AXPY, COPY = 1, 2, 3

TASK_DTYPE = np.dtype([("codelet", np.int32), ("scalar", np.float32),
                       ("b0", np.int32), ("t0", np.int32),
                       ("b1", np.int32), ("t1", np.int32)])


@dataclass
class Program:
    buffers: list            # list[np.ndarray float32], initial contents
    nparts: list             # list[int], 0 = unpartitioned
    tasks: np.ndarray        # TASK_DTYPE rows in submission order
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def ntasks(self) -> int:
        return int(self.tasks.shape[0])

    def copy_buffers(self):
        return [b.copy() for b in self.buffers]


def _tasks(n: int) -> np.ndarray:
    t = np.zeros(n, dtype=TASK_DTYPE)
    t["b1"] = -1
    t["t1"] = -1
    return t


def unit_interval_floats(rng: np.random.Generator, n: int) -> np.ndarray:
    """x in [1,2): exponent 0 with 23 random mantissa bits."""
    bits = np.uint32(0x3F800000) | (rng.integers(0, 1 << 23, size=n, dtype=np.uint32))
    return bits.view(np.float32)


def sweep_factors(rng: np.random.Generator, sweeps: int) -> np.ndarray:
    """Per-sweep factors f_s = float32(0.9 + 0.2 u_s), distinct per sweep."""
    return (0.9 + 0.2 * rng.random(sweeps)).astype(np.float32)


def c1_single(nx: int = 1024) -> Program:
    x = np.arange(1, nx + 1, dtype=np.float32)
    t = _tasks(1)
    t[0] = (SCAL, np.float32(3.14), 0, -1, -1, -1)
    return Program([x], [0], t, name="C1 single vector_scal, 1024 floats, factor 3.14")


def sweep_program(nx: int, ntiles: int, factors: np.ndarray, x: np.ndarray,
                  order: str = "sweep", name: str = "") -> Program:
    """SCAL sweeps over every tile of one partitioned vector.

    order='sweep': for s: for t: SCAL(f_s; tile t)   (sweep-major)
    order='tile' : for t: for s: SCAL(f_s; tile t)   (tile-major)
    """
    sweeps = len(factors)
    t = _tasks(ntiles * sweeps)
    t["codelet"] = SCAL
    t["b0"] = 0
    if order == "sweep":
        t["t0"] = np.tile(np.arange(ntiles, dtype=np.int32), sweeps)
        t["scalar"] = np.repeat(factors, ntiles)
    elif order == "tile":
        t["t0"] = np.repeat(np.arange(ntiles, dtype=np.int32), sweeps)
        t["scalar"] = np.tile(factors, ntiles)
    else:
        raise ValueError(order)
    return Program([x], [ntiles], t, name=name,
                   meta={"factors": factors, "sweeps": sweeps, "ntiles": ntiles, "order": order})


def c2_chain(nx: int = 1 << 24, ntiles: int = 256, sweeps: int = 16, seed: int = SEED_BASE + 1) -> Program:
    rng = np.random.default_rng(seed)
    x = unit_interval_floats(rng, nx)
    f = np.full(sweeps, np.float32(3.14), dtype=np.float32)
    return sweep_program(nx, ntiles, f, x, name=f"C2 chain of {sweeps} over {nx} floats / {ntiles} tiles")


def c4_fine(ntiles: int = 15625, tile_nx: int = 1024, sweeps: int = 64, seed: int = SEED_BASE + 3,
            order: str = "sweep") -> Program:
    rng = np.random.default_rng(seed)
    nx = ntiles * tile_nx
    x = unit_interval_floats(rng, nx)
    f = sweep_factors(rng, sweeps)
    return sweep_program(nx, ntiles, f, x, order=order,
                         name=f"C4 {ntiles * sweeps} fine tasks on {tile_nx * 4}-byte tiles")


def c5_sharded(nx: int = 1 << 30, ntiles: int = 16384, sweeps: int = 64, seed: int = SEED_BASE + 4,
               materialize: bool = True) -> Program:
    rng = np.random.default_rng(seed)
    f = sweep_factors(rng, sweeps)
    x = unit_interval_floats(rng, nx) if materialize else np.empty(0, np.float32)
    return sweep_program(nx, ntiles, f, x,
                         name=f"C5 {nx} floats x {sweeps} chained scalings, {ntiles} tiles")


def c3_random_dag(nbuf: int = 64, nx: int = 1 << 20, ntasks: int = 10000, seed: int = SEED_BASE + 2) -> Program:
    rng = np.random.default_rng(seed)
    bufs = [unit_interval_floats(rng, nx) for _ in range(nbuf)]
    t = _tasks(ntasks)
    kind = rng.integers(0, 3, size=ntasks)
    sign = np.where(rng.random(ntasks) < 0.5, -1.0, 1.0)
    fs = (sign * rng.uniform(0.75, 1.25, size=ntasks)).astype(np.float32)
    fa = (sign * rng.uniform(1.0 / 16, 0.5, size=ntasks)).astype(np.float32)
    x = rng.integers(0, nbuf, size=ntasks)
    y = (x + rng.integers(1, nbuf, size=ntasks)) % nbuf          # y != x, uniform
    t["codelet"] = np.choose(kind, [SCAL, AXPY, COPY])
    t["scalar"] = np.choose(kind, [fs, fa, np.zeros(ntasks, np.float32)]).astype(np.float32)
    t["b0"] = x
    t["t0"] = -1
    t["b1"] = np.where(kind == 0, -1, y)
    t["t1"] = -1
    return Program(bufs, [0] * nbuf, t, name=f"C3 random DAG {ntasks} tasks over {nbuf} buffers")


def random_small_program(seed: int, max_tasks: int = 10, max_handles: int = 4, max_elems: int = 64,
                         allow_partition: bool = True) -> Program:
    """SPEC.md:461/647-style property programs: <= 10 tasks, <= 4 handles,
    <= 64 elements, random modes; some buffers partitioned into tiles with a
    ragged remainder."""
    rng = np.random.default_rng(seed)
    nbuf = int(rng.integers(1, max_handles + 1))
    n = int(rng.integers(1, max_elems + 1))          # common length: AXPY/COPY operands match
    bufs, nparts = [], []
    for _ in range(nbuf):
        bufs.append(unit_interval_floats(rng, n))
        p = int(rng.integers(2, 5)) if (allow_partition and n >= 4 and rng.random() < 0.5) else 0
        nparts.append(p)
    ntask = int(rng.integers(1, max_tasks + 1))
    t = _tasks(ntask)

    for i in range(ntask):
        kind = int(rng.integers(0, 3))
        b0 = int(rng.integers(0, nbuf))
        t0 = int(rng.integers(0, nparts[b0])) if nparts[b0] else -1
        if kind == 0:
            f = np.float32(rng.choice([-1.0, 1.0]) * rng.uniform(0.5, 2.0))
            t[i] = (SCAL, f, b0, t0, -1, -1)
            continue
        # y: same tile index of a buffer with the same partitioning (equal
        # lengths without computing any range); y may alias x (reading R6).
        same = [b for b in range(nbuf) if nparts[b] == nparts[b0]]
        b1 = int(rng.choice(same))
        t1 = t0
        if nparts[b0] and b1 == b0 and rng.random() < 0.5:
            t1 = int(rng.integers(0, nparts[b0]))      # other tile of the same buffer...
            if t1 != t0:
                b1 = b0                                # ...only kept if lengths are certainly equal
                t1 = t0 if n % nparts[b0] else t1
        t[i] = (AXPY if kind == 1 else COPY,
                np.float32(rng.uniform(-0.5, 0.5)) if kind == 1 else np.float32(0),
                b0, t0, b1, t1)
    return Program(bufs, nparts, t, name=f"random small program seed {seed}")


# IEEE special and extreme binary32 values: signed zeros,
# infinities, the largest finite value, subnormals, values near overflow.
# Bit patterns only; NaN is never drawn (its bits are not portable, R11).
SPECIAL_BITS = np.array([0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x7F7FFFFF, 0xFF7FFFFF,
                         0x00000001, 0x80000001, 0x007FFFFF, 0x00800000, 0x80800000, 0x7E967699,
                         0xFE967699, 0x3F800000, 0xBF800000, 0x4048F5C3, 0x0DA24260, 0x8DA24260],
                        dtype=np.uint32)
# scalars: +-0, +-inf, huge, tiny, ordinary
SPECIAL_SCALAR_BITS = np.array([0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x7149F2CA, 0xF149F2CA,
                                0x0DA24260, 0x8DA24260, 0x4048F5C3, 0xC048F5C3, 0x3F000000, 0x3F800000],
                               dtype=np.uint32)


def special_floats(rng: np.random.Generator, n: int, frac: float = 0.5) -> np.ndarray:
    """[1,2) floats with a fraction `frac` of elements replaced by SPECIAL_BITS."""
    x = unit_interval_floats(rng, n).view(np.uint32).copy()
    sel = rng.random(n) < frac
    x[sel] = rng.choice(SPECIAL_BITS, size=int(sel.sum()))
    return x.view(np.float32)


def special_value_program(seed: int, max_tasks: int = 10, max_handles: int = 4, max_elems: int = 300,
                          finite_scalars: bool = False) -> Program:
    """random_small_program with special values in the buffers and special
    scalars (finite_scalars: only the nonzero finite ones, so no SCAL can turn
    inf into NaN).  The caller rejects programs whose result holds a NaN."""
    p = random_small_program(seed, max_tasks=max_tasks, max_handles=max_handles, max_elems=max_elems)
    rng = np.random.default_rng(seed + 7777)
    pal = SPECIAL_SCALAR_BITS
    if finite_scalars:
        pal = pal[(pal & 0x7F800000) != 0x7F800000]
        pal = pal[(pal & 0x7FFFFFFF) != 0]
    bufs = [special_floats(rng, len(b)) for b in p.buffers]
    t = p.tasks.copy()
    t["scalar"] = np.where(t["codelet"] == COPY, np.float32(0),
                           rng.choice(pal, size=len(t)).view(np.float32))
    return Program(bufs, p.nparts, t, name=f"special-value program seed {seed}")
