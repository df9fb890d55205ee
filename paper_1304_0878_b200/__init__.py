"""B200-native task-stream executor for the StarPU task model of arXiv:1304.0878.

The product is ``libbtask.so`` (C ABI in ``include/btask.h``): a host
dependency builder, a persistent sm_100a scheduler kernel and hand-written
task kernels.  ``paper_1304_0878_b200.btask`` is the ctypes binding; import it
explicitly (it raises if the library is not built -- there is no fallback).
``paper_1304_0878_b200.build`` compiles the library.  This package never
imports ``oracle/``.
"""
