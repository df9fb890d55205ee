"""Sequential CPU oracle for the task-stream hot path.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_1304_0878_b200`` never imports it and
shares no code with it (not even a header or a constant generator).

See ``oracle/oracle.c`` for the arithmetic and ``oracle/model.py`` for the
program interpretation (tile ranges, access sets, the conflict relation).

Parity status: every function here is pinned (tests/test_oracle.py); none is
"parity unpinned".
"""
from .model import (AccessMode, access_sets, build_lib, conflict_pairs, lib, run, run_tasks,
                    scal_chain, tile_range)

__all__ = ["AccessMode", "access_sets", "build_lib", "conflict_pairs", "lib", "run", "run_tasks",
           "scal_chain", "tile_range"]
