/*
 * btask.h -- C ABI of the B200 task-stream executor (libbtask.so).
 *
 * The calls mirror the runtime constructs of arXiv:1304.0878 (PAPER.md, the
 * LaTeX source; "P:n" = PAPER.md line n, "S:n" = SPEC.md line n):
 *
 *   starpu_vector_data_register  -> bt_vector_data_register
 *   starpu_data_lookup  -> bt_data_lookup
 *   starpu_insert_task  -> bt_insert_task / bt_insert_task_batch
 *   starpu_task_wait_for_all -> bt_task_wait_for_all
 *   #pragma starpu acquire  -> bt_data_acquire / bt_data_release
 *   starpu_data_unregister      -> bt_data_unregister
 *   filters / get_sub_data  -> bt_data_partition / bt_data_get_sub_data /
 *                                               bt_data_unpartition
 *   starpu_data_set_rank-> bt_data_set_rank (owner-computes home rank)
 *   starpu_malloc / starpu_free  -> bt_malloc / bt_free (pinned host memory)
 *
 * Conventions (all entry points):
 *   - Every call returns int: 0 on success, a NEGATIVE errno on failure, the
 *     convention of the generated task body "err = starpu_insert_task(...);
 *     if (err != 0) ... strerror(-err)".  bt_last_error() holds a
 *     message, e.g. "attempt to use unregistered pointer" or
 *     "failed to insert task `scal': Invalid argument".
 *   - Handles are opaque 64-bit values with a generation tag; 0 is never a
 *     valid handle.  A stale handle (after unregister) yields -ENOENT, never
 *     undefined behaviour.
 *   - Threading: one submitting host thread per runtime.  The runtime
 *     uses its own worker threads internally; they never call back.
 *   - Blocking: bt_insert_task* are asynchronous ("the invocation
 *     statement just adds the task call to the scheduler's queue");
 *     bt_task_wait_for_all, bt_data_acquire, bt_data_unregister block.
 *   - Ownership: a host buffer passed to bt_vector_data_register stays owned
 *     by the caller, must stay valid and must not be touched (except between
 *     bt_data_acquire and bt_data_release) until bt_data_unregister returns,
 *     at which point it holds the final data.  Device replicas are
 *     owned by the runtime.  A device pointer registered with home_node = 1
 *     (e.g. a torch CUDA tensor) stays owned by the caller and is used in
 *     place.
 *   - A sticky device error (kernel fault, failed copy) poisons the runtime:
 *     that call and every later call return -EIO.
 *   - No CPU execution path exists: every task runs in the sm_100a kernels.
 *     Without a usable GPU, bt_init returns -ENODEV unless BT_FLAG_HOST_ONLY
 *     is set, in which case tasks are only analysed (bt_dag_snapshot) and
 *     bt_task_wait_for_all returns -ENODEV.
 */
#ifndef BTASK_H
#define BTASK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BT_ABI_VERSION 5   /* 2: bt_stats.kernel_launches, BT_FLAG_KERNEL_*; 3: bt_stats.sched_launches,
                               BT_FLAG_NO_STREAM; 4: bt_stats.stream_resumes, bt_stats.prio_epochs,
                               BT_FLAG_PRIORITY, bt_debug_gate; 5: bt_dag_view.item_flags */

typedef struct bt_runtime bt_runtime;
typedef uint64_t bt_handle;

/* Access modes ("read-only, write-only, or read-write").
 * Bit flags; the generated call passes 3 for RW. */
enum { BT_R = 1, BT_W = 2, BT_RW = 3 };

/* Built-in codelets (P:127-139 starpu_codelet: fixed nbuffers and modes).
 *   BT_CL_SCAL  vector_scal   cl_args = float f          buffers: x:RW
 *               x[i] = x[i] * f
 *   BT_CL_AXPY  axpy          cl_args = float a          buffers: x:R, y:RW
 *               y[i] = (a * x[i]) + y[i], two roundings  (BASELINE.json configs[2])
 *   BT_CL_COPY  copy          cl_args = none             buffers: x:R, y:W
 *               y[i] = x[i]                              (BASELINE.json configs[2])
 * Arithmetic is IEEE-754 binary32, round to nearest even, no FMA contraction,
 * subnormals preserved; results are bit-identical to executing the tasks one
 * by one in submission order. */
enum { BT_CL_SCAL = 1, BT_CL_AXPY = 2, BT_CL_COPY = 3 };

/* bt_config.flags */
enum {
  BT_FLAG_NO_FUSION  = 1u << 0, /* never fuse consecutive SCAL(RW) tasks of one (sub)handle */
  BT_FLAG_HOST_ONLY  = 1u << 1, /* no GPU: analyse only (bt_dag_snapshot); nothing executes */
  BT_FLAG_TIMESTAMPS = 1u << 2, /* record %globaltimer per work unit (bt_trace) */
  BT_FLAG_SYNC_EPOCH = 1u << 3, /* debugging: synchronise after every epoch launch */
  BT_FLAG_NO_STREAM  = 1u << 4, /* one launch per pipelined round instead of one stream launch per
                                   run ("Stream launches"); for comparisons */
  BT_FLAG_PRIORITY   = 1u << 5, /* DAG epochs on the CTA-wide "sw" bodies: ready work ordered by upward rank
                                   (priority levels) instead of FIFO.
                                   Off by default: measured neutral on C3, slower on smaller DAGs */
  /* testing: force one scheduler variant for every epoch instead of the
   * per-epoch choice (DESIGN.md section "Persistent scheduler kernels"); at
   * most one of the three may be set (-EINVAL otherwise) */
  BT_FLAG_KERNEL_SW  = 1u << 8,  /* CTA-wide units, one scheduler warp */
  BT_FLAG_KERNEL_RW  = 1u << 9,  /* CTA-wide units, pop + release warps, in-slot chains */
  BT_FLAG_KERNEL_WQ  = 1u << 10  /* one warp per unit */
};

typedef struct bt_config {
  uint32_t abi_version;   /* must be BT_ABI_VERSION (bt_config_init sets it) */
  int device;             /* CUDA device ordinal; -1 = the calling thread's current device */
  void *stream;           /* cudaStream_t all work is ordered on; NULL = runtime-owned stream */
  int rank;               /* owner-computes rank of this process; default 0 */
  int nranks;             /* number of ranks; default 1 */
  uint32_t flags;         /* BT_FLAG_* */
  uint32_t chunk_bytes;   /* work-unit size in bytes of the written operand (large tasks are
                             split into chunks run by different CTAs); 0 = default (256 KiB) */
  uint32_t max_fused;     /* max SCAL tasks fused into one work item; 0 = default (256) */
  int ctas_per_sm;        /* persistent CTAs per SM; 0 = maximum occupancy */
  uint64_t epoch_tasks;   /* auto-flush an epoch after this many pending tasks; 0 = never */
  int host_threads;       /* dependency-builder threads (parallel SCAL runs); 0 = min(16, cores - 2) */
  uint32_t parallel_min;  /* shortest SCAL run of a batch built in parallel; 0 = default (16384) */
  int pipeline_rounds;    /* a long SCAL run is built and launched in this many rounds of
                             handles, so the device starts while the host still builds;
                             0 = default (4), 1 = off */
  uint32_t pipeline_min;  /* shortest SCAL run that is pipelined; 0 = default (131072) */
} bt_config;

/* Fill *cfg with defaults.  Returns 0. */
int bt_config_init(bt_config *cfg);

/* Create a runtime bound to one GPU.  -EINVAL (bad config), -ENODEV (no GPU /
 * bad device id, unless BT_FLAG_HOST_ONLY), -ENOMEM.  *out is set on success. */
int bt_init(const bt_config *cfg, bt_runtime **out);

/* Destroy.  Waits for outstanding work.  -EBUSY if handles are still registered
 * (they stay registered; call bt_data_unregister first). */
int bt_shutdown(bt_runtime *rt);

/* starpu_vector_data_register.  Registers nx elements of elemsize
 * bytes (elemsize must be 4: float32) at ptr.
 *   home_node 0: ptr is host memory.  A device replica is allocated on the
 *                runtime's GPU and filled from ptr (asynchronously, before any
 *                task on the handle).  ptr may be NULL on a rank that is not
 *                the data's home; then no storage exists here.
 *   home_node 1: ptr is device memory on the runtime's GPU; used in place.
 * -EEXIST if [ptr, ptr+nx*elemsize) overlaps a live registration,
 * -EINVAL (nx == 0, elemsize != 4, bad home_node), -ENOMEM. */
int bt_vector_data_register(bt_runtime *rt, bt_handle *out, int home_node, void *ptr,
                            size_t nx, size_t elemsize);

/* starpu_data_lookup: exact base pointer -> handle.
 * -ENOENT, message "attempt to use unregistered pointer". */
int bt_data_lookup(bt_runtime *rt, const void *ptr, bt_handle *out);

/* Block filter: split h into nparts contiguous sub-handles; sub t
 * covers [t*(nx/nparts) + min(t, nx%nparts), ...) with the first nx%nparts
 * parts one element longer.  Views, no copy.  While partitioned, tasks on h
 * itself return -EBUSY.  -EINVAL (nparts == 0 or > nx), -EBUSY (already
 * partitioned, or acquired). */
int bt_data_partition(bt_runtime *rt, bt_handle h, uint32_t nparts);

/* starpu_data_get_sub_data: handle of part i.  -EINVAL (not
 * partitioned / i out of range). */
int bt_data_get_sub_data(bt_runtime *rt, bt_handle h, uint32_t i, bt_handle *out);

/* All parts at once: out[i] = part i for i < nparts (nparts must equal the
 * partition's count).  -EINVAL otherwise. */
int bt_data_get_children(bt_runtime *rt, bt_handle h, bt_handle *out, uint32_t nparts);

/* Undo bt_data_partition; later tasks on h are ordered after every earlier task
 * on any part.  -EINVAL if not partitioned, -EBUSY if a part is itself
 * partitioned or acquired. */
int bt_data_unpartition(bt_runtime *rt, bt_handle h);

/* starpu_data_set_rank: home rank of h (and of its parts).
 * Tasks execute on the rank owning their written operand ("owner computes",
 * P:1058-1061); tasks whose written operand lives on another rank are skipped
 * here.  -EINVAL (rank out of range). */
int bt_data_set_rank(bt_runtime *rt, bt_handle h, int rank);

/* Block distribution of the parts of a partitioned h: part t -> rank
 * floor(t * nranks / nparts).  -EINVAL if h is not partitioned. */
int bt_data_distribute_block(bt_runtime *rt, bt_handle h);

/* Cross-rank reads between the ranks of one node (StarPU-MPI, P:1041-1061:
 * data a task only reads is transferred to the rank that runs it).
 * Collective: every rank of the job (one process each, ranks 0..nranks-1 of
 * bt_config) calls it once with the same `name`, a POSIX shared-memory name
 * unique to the job ("/bt-<job id>"); it returns when all ranks have joined.
 * Call it before registering data: device replicas of host-homed data are
 * then allocated shareably (cudaMalloc; device-homed data must be cudaMalloc'ed
 * memory, e.g. a torch tensor).
 * Afterwards an AXPY/COPY whose read operand x lives on rank a and whose
 * written operand y lives on rank b != a no longer fails with -EXDEV: every
 * rank submits it (same order on all ranks); rank a and rank b meet there --
 * b copies x's current value (ordered after a's earlier writers of x) from
 * a's device memory (CUDA IPC; a peer copy over NVLink between GPUs) into b's
 * own replica of x, a's later writers of x wait for that copy, and the task
 * runs on b; other ranks skip it.  Every rank must register x (with local
 * storage) and partition it alike.  A non-owner's replica of x holds the last
 * value it received; only owners' data is defined after the program.
 * A reader keeps what it received as a shared copy: a later read of the same
 * range by the same rank skips the transfer (on both ranks) while no task has
 * written the data since -- every rank sees every task, so both decide alike.
 * Host writes to data other ranks read (bt_data_acquire BT_RW + release) must
 * then be collective: every rank calls bt_data_release at the same point of
 * the task stream (a release invalidates the shared copies).
 * Returns 0, -EINVAL (nranks < 2, bad name, ranks disagree), -ENODEV
 * (host-only runtime), -EBUSY (already initialised), -ETIMEDOUT (a rank did
 * not join within 60 s), -EIO.  A rendezvous that times out (60 s) returns
 * -EIO from the insert and poisons the runtime. */
int bt_comm_init(bt_runtime *rt, const char *name);

/* starpu_insert_task, asynchronous.
 *   codelet    BT_CL_*
 *   cl_args    packed scalar arguments, little-endian, declaration order, no
 *              padding: one float for SCAL/AXPY, none for COPY
 *   handles    nbuffers (sub)handles, modes[i] the access mode passed for
 *              handles[i]; must equal the codelet's modes, else
 *              -EINVAL.  The same handle may appear twice (modes OR-ed).
 * Dependencies (RAW, WAR, WAW) on every earlier task are inferred from the
 * modes and the submission order.
 * -ENOENT unknown/stale handle ("attempt to use unregistered pointer"),
 * -EINVAL (bad codelet/modes/nbuffers/cl_args_size, operand length mismatch),
 * -EBUSY (partitioned parent, or acquired handle), -EXDEV (the task reads
 * data homed on another rank and bt_comm_init was not called),
 * -ENOMEM, -EIO. */
int bt_insert_task(bt_runtime *rt, int codelet, const void *cl_args, size_t cl_args_size,
                   const bt_handle *handles, const int *modes, unsigned nbuffers);

/* Exactly equivalent to ntasks bt_insert_task calls in order, with the
 * codelet's own modes: task i is codelets[i] with scalar scalars[i] (ignored
 * for COPY), operand 0 = h0[i], operand 1 = h1[i] (h1 may be NULL when every
 * codelet is SCAL).  Stops at the first failing task: *nsubmitted (if not
 * NULL) receives the number of tasks accepted, and that task's error is
 * returned. */
int bt_insert_task_batch(bt_runtime *rt, size_t ntasks, const int32_t *codelets,
                         const float *scalars, const bt_handle *h0, const bt_handle *h1,
                         size_t *nsubmitted);

/* Close the current epoch: build its DAG, upload it and launch the persistent
 * scheduler kernel on the runtime's stream, without waiting.  Tasks submitted
 * afterwards form a new epoch that runs after it (stream order).  No-op if
 * nothing is pending.  -EIO, -ENOMEM, -ENODEV (host-only runtime). */
int bt_flush(bt_runtime *rt);

/* starpu_task_wait_for_all ("#pragma starpu wait"): flush,
 * then block until every submitted task has completed.  -EIO on device fault
 * (sticky), -ENODEV for a host-only runtime. */
int bt_task_wait_for_all(bt_runtime *rt);

/* #pragma starpu acquire: wait for every task on h, then make the
 * registered host buffer hold the current contents (device -> host copy).
 * mode BT_R or BT_RW; with BT_RW, host writes are uploaded at bt_data_release.
 * Until bt_data_release, tasks on h return -EBUSY.  A partitioned h is
 * acquired as a whole (every part).  -ENOENT, -EBUSY (already acquired),
 * -EINVAL (device-homed data or no local storage), -EIO. */
int bt_data_acquire(bt_runtime *rt, bt_handle h, int mode);
int bt_data_release(bt_runtime *rt, bt_handle h);

/* starpu_data_unregister: wait for the handle's tasks, copy the final
 * contents back to the registered host buffer (home_node 0), free the device
 * replica and forget h and its parts.  -ENOENT, -EBUSY (partitioned, or h is a
 * sub-handle), -EIO. */
int bt_data_unregister(bt_runtime *rt, bt_handle h);

/* starpu_malloc / starpu_free: page-locked host memory, so that
 * register/acquire/unregister transfers run at full link speed. */
int bt_malloc(void **out, size_t bytes);
int bt_free(void *ptr);

/* Error text for a negative errno returned by this library. */
const char *bt_strerror(int err);
/* Message of the last failing call on rt (empty string if none). */
const char *bt_last_error(bt_runtime *rt);

/* Counters since bt_init (or the last bt_stats_reset). */
typedef struct bt_stats {
  uint64_t tasks_submitted;   /* accepted bt_insert_task* tasks (all ranks' view) */
  uint64_t tasks_local;       /* of which executed on this rank */
  uint64_t items;             /* work items (a fused SCAL chain is one item) */
  uint64_t fused_tasks;       /* tasks merged into an earlier item */
  uint64_t edges;             /* dependency edges between items */
  uint64_t units;             /* work units (item chunks) run by the device */
  uint64_t epochs;            /* epochs launched */
  uint64_t upload_bytes;      /* DAG bytes copied host -> device */
  double host_build_ms;       /* time in the dependency builder (insert + pack) */
  double device_ms;           /* summed persistent-kernel time of completed epochs */
  double device_span_ms;      /* summed device time from the first launch after a wait to the end
                                 of that wait's work (overlapping launches counted once) */
  uint32_t grid;              /* persistent CTAs of the last launch */
  uint32_t block;             /* threads per CTA of the last launch */
  uint64_t kernel_launches;   /* this library's kernel launches (per epoch: set-up + scheduler) */
  uint64_t sched_launches;    /* of which scheduler-kernel launches (a stream launch runs several epochs);
                                 device_ms / sched_launches = average launch duration */
  uint64_t stream_closes;     /* stream launches ended early by the host (a later round needed a larger
                                 epoch buffer, or the run failed part-way) */
  uint64_t stream_resumes;    /* stream launches that closed themselves (no publication for 50 ms, e.g.
                                 under a launch-serialising tool) and were finished by their resume launch */
  uint64_t prio_epochs;       /* epochs run with the priority ready queue (upward-rank levels) */
  uint64_t h2d_data_bytes;    /* host-homed data uploaded (first reads; bt_data_release of an RW acquire) */
  uint64_t d2h_data_bytes;    /* host-homed data written back (eager write-backs, dirty ranges) */
  uint64_t cross_rank_copies; /* cross-rank reads that copied their operand (bt_comm_init) */
  uint64_t cross_rank_skips;  /* ... that found the pair's previous copy still current (no write since) */
} bt_stats;
int bt_stats_get(bt_runtime *rt, bt_stats *out);
int bt_stats_reset(bt_runtime *rt);

/* ---- analysis view (used by tests; works in host-only runtimes) -------- */
typedef struct bt_dag_view {
  uint64_t ntasks;            /* tasks in the snapshotted epoch (submission order) */
  uint64_t nitems;
  uint64_t nedges;
  const uint32_t *task_item;  /* [ntasks] item running the task, UINT32_MAX if not local */
  const uint32_t *task_pos;   /* [ntasks] position of the task inside its item's chain */
  const uint8_t *item_kind;   /* [nitems] BT_CL_* */
  const uint32_t *item_k;     /* [nitems] number of tasks in the item */
  const uint32_t *item_npred; /* [nitems] */
  const uint32_t *succ_off;   /* [nitems+1] CSR offsets */
  const uint32_t *succ;       /* [nedges] successor items */
  const uint8_t *item_flags;  /* [nitems] BT_DAG_WHOLE_PREDS: some predecessor's operand on the handle it
                                 was found through has another base address than the item's (partition-
                                 inherited state), so the item's work units wait for whole predecessors;
                                 otherwise unit c of an item of several units waits only for unit c of
                                 each same-length predecessor (chunk-wise release) */
} bt_dag_view;
enum { BT_DAG_WHOLE_PREDS = 1 };

/* Close the pending epoch WITHOUT executing it and expose its DAG (valid until
 * the next call on rt).  Only for BT_FLAG_HOST_ONLY runtimes (-EPERM else),
 * where a registered vector's host address stands in for its device replica
 * (operand base addresses; nothing is dereferenced). */
int bt_dag_snapshot(bt_runtime *rt, bt_dag_view *out);

/* Per-unit device timestamps of the last completed epoch (BT_FLAG_TIMESTAMPS):
 * for unit u, t[4u+0..3] = pop start, body start, body end, release end
 * (%globaltimer ns); item[u] = its item.  *n = number of units.  Pointers valid
 * until the next flush.  -ENODATA if no trace is available. */
int bt_trace(bt_runtime *rt, const uint64_t **t, const uint32_t **item, uint64_t *n);

/* ---- test hook --------------------------------------------------------- */
/* Hold the runtime's stream: work enqueued on it after this call (the next
 * epochs' kernels, the copies of cross-rank reads) starts only once the caller
 * stores a nonzero value into **flag_out, a word of mapped pinned host memory
 * owned by the runtime (valid until bt_shutdown).  Implemented as a stream
 * memory wait (cuStreamWaitValue32), else a one-thread gate kernel polling the
 * word (60 s watchdog).  Nothing else waits: other ranks' streams keep running,
 * which makes a missing cross-rank RAW/WAR ordering (bt_comm_init) observable
 * with all ranks on one GPU (tests/test_gpu.py::test_cross_rank_gated_*).
 * -EINVAL, -ENODEV (host-only runtime), -ENOMEM, -EIO. */
int bt_debug_gate(bt_runtime *rt, volatile uint32_t **flag_out);

#ifdef __cplusplus
}
#endif
#endif /* BTASK_H */
