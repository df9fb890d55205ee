"""ctypes binding of libbtask.so (include/btask.h), argument marshalling only.

Every ``bt_*`` function here has the name and argument order of the C entry
point and returns its int status; nothing is computed in Python.  ``Runtime``
is a thin convenience wrapper raising ``BtError`` on negative status.

There is no fallback: if ``libbtask.so`` is missing, importing this module
raises (build it with ``python -m paper_1304_0878_b200.build``).
"""
from __future__ import annotations

import ctypes
import errno
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BT_LIB_PATH") or os.path.join(_PKG, "libbtask.so")   # override: experiments only

BT_ABI_VERSION = 5
BT_R, BT_W, BT_RW = 1, 2, 3
BT_CL_SCAL, BT_CL_AXPY, BT_CL_COPY = 1, 2, 3
BT_FLAG_NO_FUSION, BT_FLAG_HOST_ONLY, BT_FLAG_TIMESTAMPS, BT_FLAG_SYNC_EPOCH, BT_FLAG_NO_STREAM = 1, 2, 4, 8, 16
BT_FLAG_PRIORITY = 32
BT_DAG_WHOLE_PREDS = 1   # bt_dag_view.item_flags
BT_FLAG_KERNEL_SW, BT_FLAG_KERNEL_RW, BT_FLAG_KERNEL_WQ = 1 << 8, 1 << 9, 1 << 10

bt_handle = ctypes.c_uint64


class bt_config(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_uint32), ("device", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("flags", ctypes.c_uint32),
                ("chunk_bytes", ctypes.c_uint32), ("max_fused", ctypes.c_uint32), ("ctas_per_sm", ctypes.c_int),
                ("epoch_tasks", ctypes.c_uint64), ("host_threads", ctypes.c_int), ("parallel_min", ctypes.c_uint32),
                ("pipeline_rounds", ctypes.c_int), ("pipeline_min", ctypes.c_uint32)]


class bt_stats(ctypes.Structure):
    _fields_ = [("tasks_submitted", ctypes.c_uint64), ("tasks_local", ctypes.c_uint64), ("items", ctypes.c_uint64),
                ("fused_tasks", ctypes.c_uint64), ("edges", ctypes.c_uint64), ("units", ctypes.c_uint64),
                ("epochs", ctypes.c_uint64), ("upload_bytes", ctypes.c_uint64), ("host_build_ms", ctypes.c_double),
                ("device_ms", ctypes.c_double), ("device_span_ms", ctypes.c_double), ("grid", ctypes.c_uint32),
                ("block", ctypes.c_uint32), ("kernel_launches", ctypes.c_uint64),
                ("sched_launches", ctypes.c_uint64), ("stream_closes", ctypes.c_uint64),
                ("stream_resumes", ctypes.c_uint64), ("prio_epochs", ctypes.c_uint64),
                ("h2d_data_bytes", ctypes.c_uint64), ("d2h_data_bytes", ctypes.c_uint64),
                ("cross_rank_copies", ctypes.c_uint64), ("cross_rank_skips", ctypes.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class bt_dag_view(ctypes.Structure):
    _fields_ = [("ntasks", ctypes.c_uint64), ("nitems", ctypes.c_uint64), ("nedges", ctypes.c_uint64),
                ("task_item", ctypes.POINTER(ctypes.c_uint32)), ("task_pos", ctypes.POINTER(ctypes.c_uint32)),
                ("item_kind", ctypes.POINTER(ctypes.c_uint8)), ("item_k", ctypes.POINTER(ctypes.c_uint32)),
                ("item_npred", ctypes.POINTER(ctypes.c_uint32)), ("succ_off", ctypes.POINTER(ctypes.c_uint32)),
                ("succ", ctypes.POINTER(ctypes.c_uint32)), ("item_flags", ctypes.POINTER(ctypes.c_uint8))]


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built: run `python -m paper_1304_0878_b200.build` "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

_P = ctypes.POINTER
_c = ctypes
_SIGS = {
    "bt_config_init": (_c.c_int, [_P(bt_config)]),
    "bt_init": (_c.c_int, [_P(bt_config), _P(_c.c_void_p)]),
    "bt_shutdown": (_c.c_int, [_c.c_void_p]),
    "bt_vector_data_register": (_c.c_int, [_c.c_void_p, _P(bt_handle), _c.c_int, _c.c_void_p, _c.c_size_t,
                                            _c.c_size_t]),
    "bt_data_lookup": (_c.c_int, [_c.c_void_p, _c.c_void_p, _P(bt_handle)]),
    "bt_data_partition": (_c.c_int, [_c.c_void_p, bt_handle, _c.c_uint32]),
    "bt_data_get_sub_data": (_c.c_int, [_c.c_void_p, bt_handle, _c.c_uint32, _P(bt_handle)]),
    "bt_data_get_children": (_c.c_int, [_c.c_void_p, bt_handle, _P(bt_handle), _c.c_uint32]),
    "bt_data_unpartition": (_c.c_int, [_c.c_void_p, bt_handle]),
    "bt_data_set_rank": (_c.c_int, [_c.c_void_p, bt_handle, _c.c_int]),
    "bt_data_distribute_block": (_c.c_int, [_c.c_void_p, bt_handle]),
    "bt_comm_init": (_c.c_int, [_c.c_void_p, _c.c_char_p]),
    "bt_insert_task": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_void_p, _c.c_size_t, _P(bt_handle), _P(_c.c_int),
                                   _c.c_uint]),
    # (const int32_t *codelets, const float *scalars, const bt_handle *h0, const bt_handle *h1):
    # raw addresses, so a call marshals four integers (ndarray.ctypes.data_as costs ~3 us each)
    "bt_insert_task_batch": (_c.c_int, [_c.c_void_p, _c.c_size_t, _c.c_void_p, _c.c_void_p, _c.c_void_p,
                                         _c.c_void_p, _P(_c.c_size_t)]),
    "bt_flush": (_c.c_int, [_c.c_void_p]),
    "bt_task_wait_for_all": (_c.c_int, [_c.c_void_p]),
    "bt_data_acquire": (_c.c_int, [_c.c_void_p, bt_handle, _c.c_int]),
    "bt_data_release": (_c.c_int, [_c.c_void_p, bt_handle]),
    "bt_data_unregister": (_c.c_int, [_c.c_void_p, bt_handle]),
    "bt_malloc": (_c.c_int, [_P(_c.c_void_p), _c.c_size_t]),
    "bt_free": (_c.c_int, [_c.c_void_p]),
    "bt_strerror": (_c.c_char_p, [_c.c_int]),
    "bt_last_error": (_c.c_char_p, [_c.c_void_p]),
    "bt_stats_get": (_c.c_int, [_c.c_void_p, _P(bt_stats)]),
    "bt_stats_reset": (_c.c_int, [_c.c_void_p]),
    "bt_dag_snapshot": (_c.c_int, [_c.c_void_p, _P(bt_dag_view)]),
    "bt_trace": (_c.c_int, [_c.c_void_p, _P(_P(_c.c_uint64)), _P(_P(_c.c_uint32)), _P(_c.c_uint64)]),
    "bt_debug_gate": (_c.c_int, [_c.c_void_p, _P(_P(_c.c_uint32))]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f

EXPORTED = tuple(_SIGS)


class BtError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{errno.errorcode.get(-code, code)}] {msg}")
        self.code = code


def _u64p(a: np.ndarray):
    return a.ctypes.data_as(_P(bt_handle))


class Runtime:
    """Pythonic wrapper over one bt_runtime (one GPU)."""

    def __init__(self, device: int = -1, stream=None, rank: int = 0, nranks: int = 1, flags: int = 0,
                 chunk_bytes: int = 0, max_fused: int = 0, ctas_per_sm: int = 0, epoch_tasks: int = 0,
                 host_threads: int = 0, parallel_min: int = 0, pipeline_rounds: int = 0, pipeline_min: int = 0):
        cfg = bt_config()
        bt_config_init(ctypes.byref(cfg))
        cfg.device, cfg.rank, cfg.nranks, cfg.flags = device, rank, nranks, flags
        cfg.stream = stream
        cfg.chunk_bytes, cfg.max_fused, cfg.ctas_per_sm, cfg.epoch_tasks = chunk_bytes, max_fused, ctas_per_sm, \
            epoch_tasks
        cfg.host_threads, cfg.parallel_min = host_threads, parallel_min
        cfg.pipeline_rounds, cfg.pipeline_min = pipeline_rounds, pipeline_min
        h = ctypes.c_void_p()
        rc = bt_init(ctypes.byref(cfg), ctypes.byref(h))
        if rc:
            raise BtError(rc, f"bt_init: {bt_strerror(rc).decode()}")
        self.rt = h
        self._keep = {}

    def _check(self, rc: int, what: str):
        if rc:
            raise BtError(rc, f"{what}: {bt_last_error(self.rt).decode()}")
        return rc

    def close(self):
        if self.rt:
            self._check(bt_shutdown(self.rt), "bt_shutdown")
            self.rt = None

    # -- data -------------------------------------------------------------
    def register(self, ptr: int, nx: int, home_node: int = 0) -> int:
        out = bt_handle()
        self._check(bt_vector_data_register(self.rt, ctypes.byref(out), home_node, ptr, nx, 4),
                    "bt_vector_data_register")
        return out.value

    def register_array(self, arr: np.ndarray) -> int:
        assert arr.dtype == np.float32 and arr.flags.c_contiguous
        h = self.register(arr.ctypes.data, arr.shape[0], 0)
        self._keep[h] = arr
        return h

    def register_tensor(self, t) -> int:
        """Device-homed registration of a contiguous float32 CUDA tensor (used in place)."""
        assert t.is_cuda and t.is_contiguous() and str(t.dtype) == "torch.float32"
        h = self.register(t.data_ptr(), t.numel(), 1)
        self._keep[h] = t
        return h

    def lookup(self, ptr: int) -> int:
        out = bt_handle()
        self._check(bt_data_lookup(self.rt, ptr, ctypes.byref(out)), "bt_data_lookup")
        return out.value

    def partition(self, h: int, nparts: int) -> list:
        self._check(bt_data_partition(self.rt, h, nparts), "bt_data_partition")
        return self.sub_handles(h, nparts)

    def sub_handles(self, h: int, nparts: int) -> list:
        out = np.zeros(nparts, np.uint64)
        self._check(bt_data_get_children(self.rt, h, _u64p(out), nparts), "bt_data_get_children")
        return out.tolist()

    def sub_handle(self, h: int, i: int) -> int:
        out = bt_handle()
        self._check(bt_data_get_sub_data(self.rt, h, i, ctypes.byref(out)), "bt_data_get_sub_data")
        return out.value

    def unpartition(self, h: int):
        self._check(bt_data_unpartition(self.rt, h), "bt_data_unpartition")

    def set_rank(self, h: int, rank: int):
        self._check(bt_data_set_rank(self.rt, h, rank), "bt_data_set_rank")

    def distribute_block(self, h: int):
        self._check(bt_data_distribute_block(self.rt, h), "bt_data_distribute_block")

    def comm_init(self, name: str):
        """bt_comm_init: collective over the job's ranks (cross-rank reads)."""
        self._check(bt_comm_init(self.rt, name.encode()), "bt_comm_init")

    def acquire(self, h: int, mode: int = BT_R):
        self._check(bt_data_acquire(self.rt, h, mode), "bt_data_acquire")

    def release(self, h: int):
        self._check(bt_data_release(self.rt, h), "bt_data_release")

    def unregister(self, h: int):
        self._check(bt_data_unregister(self.rt, h), "bt_data_unregister")
        self._keep.pop(h, None)

    # -- tasks ------------------------------------------------------------
    def insert(self, codelet: int, handles, modes, scalar=None) -> int:
        hs = (bt_handle * len(handles))(*handles)
        ms = (ctypes.c_int * len(modes))(*modes)
        if scalar is None:
            return bt_insert_task(self.rt, codelet, None, 0, hs, ms, len(handles))
        f = ctypes.c_float(scalar)
        return bt_insert_task(self.rt, codelet, ctypes.byref(f), 4, hs, ms, len(handles))

    def scal(self, h: int, f: float):
        self._check(self.insert(BT_CL_SCAL, [h], [BT_RW], f), "bt_insert_task")

    def axpy(self, a: float, x: int, y: int):
        self._check(self.insert(BT_CL_AXPY, [x, y], [BT_R, BT_RW], a), "bt_insert_task")

    def copy(self, x: int, y: int):
        self._check(self.insert(BT_CL_COPY, [x, y], [BT_R, BT_W]), "bt_insert_task")

    def insert_batch(self, codelets: np.ndarray, scalars: np.ndarray, h0: np.ndarray, h1: np.ndarray | None = None):
        c = np.ascontiguousarray(codelets, np.int32)
        s = np.ascontiguousarray(scalars, np.float32)
        a0 = np.ascontiguousarray(h0, np.uint64)
        a1 = None if h1 is None else np.ascontiguousarray(h1, np.uint64)
        if not (c.shape[0] == s.shape[0] == a0.shape[0] and (a1 is None or a1.shape[0] == c.shape[0])):
            raise ValueError("insert_batch: arrays of different lengths")
        n = ctypes.c_size_t()
        rc = bt_insert_task_batch(self.rt, c.shape[0], c.ctypes.data, s.ctypes.data, a0.ctypes.data,
                                  None if a1 is None else a1.ctypes.data, ctypes.byref(n))
        self._check(rc, f"bt_insert_task_batch (accepted {n.value})")
        return n.value

    def flush(self):
        self._check(bt_flush(self.rt), "bt_flush")

    def wait(self):
        self._check(bt_task_wait_for_all(self.rt), "bt_task_wait_for_all")

    # -- introspection ----------------------------------------------------
    def stats(self) -> dict:
        s = bt_stats()
        self._check(bt_stats_get(self.rt, ctypes.byref(s)), "bt_stats_get")
        return s.as_dict()

    def stats_reset(self):
        self._check(bt_stats_reset(self.rt), "bt_stats_reset")

    def dag_snapshot(self) -> dict:
        v = bt_dag_view()
        self._check(bt_dag_snapshot(self.rt, ctypes.byref(v)), "bt_dag_snapshot")
        n, m, e = v.ntasks, v.nitems, v.nedges

        def arr(p, cnt, dt):
            return np.ctypeslib.as_array(p, shape=(cnt,)).astype(dt, copy=True) if cnt else np.zeros(0, dt)
        return {"ntasks": n, "nitems": m, "nedges": e,
                "task_item": arr(v.task_item, n, np.uint32), "task_pos": arr(v.task_pos, n, np.uint32),
                "item_kind": arr(v.item_kind, m, np.uint8), "item_k": arr(v.item_k, m, np.uint32),
                "item_npred": arr(v.item_npred, m, np.uint32), "succ_off": arr(v.succ_off, m + 1, np.uint32),
                "succ": arr(v.succ, e, np.uint32), "item_flags": arr(v.item_flags, m, np.uint8)}

    def trace(self):
        t = ctypes.POINTER(ctypes.c_uint64)()
        it = ctypes.POINTER(ctypes.c_uint32)()
        n = ctypes.c_uint64()
        rc = bt_trace(self.rt, ctypes.byref(t), ctypes.byref(it), ctypes.byref(n))
        if rc:
            return None
        cnt = n.value
        return (np.ctypeslib.as_array(t, shape=(4 * cnt,)).reshape(cnt, 4).copy(),
                np.ctypeslib.as_array(it, shape=(cnt,)).copy())

    def last_error(self) -> str:
        return bt_last_error(self.rt).decode()

    def debug_gate(self):
        """Test hook: hold the runtime's stream; returns a callable that opens the gate."""
        flag = ctypes.POINTER(ctypes.c_uint32)()
        self._check(bt_debug_gate(self.rt, ctypes.byref(flag)), "bt_debug_gate")

        def release():
            flag[0] = 1
        return release

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        if self.rt and not exc[0]:
            self.close()


def pinned_empty(nbytes: int):
    """bt_malloc'd (page-locked) host buffer; returns (address, numpy float32 view)."""
    p = ctypes.c_void_p()
    rc = bt_malloc(ctypes.byref(p), nbytes)
    if rc:
        raise BtError(rc, "bt_malloc")
    buf = (ctypes.c_char * nbytes).from_address(p.value)
    return p.value, np.frombuffer(buf, dtype=np.float32)
