"""Drive a neutral ``workloads.Program`` through the C ABI (product side).

Registration, partitioning, batched
``starpu_insert_task``-style submission, wait and
unregister -- every step runs in libbtask.so; this module only maps
the program's (buffer, tile) operands to handles.
"""
from __future__ import annotations

import numpy as np

from . import btask as B


class Session:
    """Registered buffers + handle tables of one program on one runtime."""

    def __init__(self, rt: "B.Runtime", program, host_buffers: list | None = None, device_tensors: list | None = None):
        self.rt = rt
        self.program = program
        self.bufs = host_buffers if host_buffers is not None else program.copy_buffers()
        self.roots, self.subs = [], []
        for b, nparts in enumerate(program.nparts):
            if device_tensors is not None:
                h = rt.register_tensor(device_tensors[b])
            else:
                h = rt.register_array(self.bufs[b])
            self.roots.append(h)
            self.subs.append(rt.partition(h, nparts) if nparts else [])

    def handle_arrays(self):
        t = self.program.tasks
        return self._handles(t["b0"], t["t0"]), self._handles(t["b1"], t["t1"])

    def _handles(self, b, tile):
        out = np.zeros(len(b), np.uint64)
        for bi in np.unique(b):
            if bi < 0:
                continue
            sel = b == bi
            if self.subs[bi]:
                out[sel] = np.asarray(self.subs[bi], np.uint64)[tile[sel]]
            else:
                out[sel] = self.roots[bi]
        return out

    def submit(self, h0=None, h1=None, batch: bool = True):
        t = self.program.tasks
        if h0 is None:
            h0, h1 = self.handle_arrays()
        if batch:
            only_scal = bool(np.all(t["codelet"] == B.BT_CL_SCAL))
            self.rt.insert_batch(t["codelet"], t["scalar"], h0, None if only_scal else h1)
        else:
            for i, row in enumerate(t):
                c = int(row["codelet"])
                if c == B.BT_CL_SCAL:
                    self.rt.scal(int(h0[i]), float(row["scalar"]))
                elif c == B.BT_CL_AXPY:
                    self.rt.axpy(float(row["scalar"]), int(h0[i]), int(h1[i]))
                else:
                    self.rt.copy(int(h0[i]), int(h1[i]))

    def finish(self) -> list:
        """Unpartition + unregister everything (final data lands in the host buffers)."""
        for b, h in enumerate(self.roots):
            if self.subs[b]:
                self.rt.unpartition(h)
            self.rt.unregister(h)
        return self.bufs


def run_program(program, batch: bool = True, **rt_kwargs) -> tuple[list, dict]:
    """Execute a program on the GPU through the ABI; returns (final buffers, stats)."""
    with B.Runtime(**rt_kwargs) as rt:
        s = Session(rt, program)
        s.submit(batch=batch)
        rt.wait()
        out = s.finish()
        return out, rt.stats()
