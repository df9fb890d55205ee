// device_abi.h -- layouts shared by the host packer (runtime.cpp) and the
// persistent scheduler kernel (scheduler.cu).  Internal to libbtask.so.
#pragma once
#include <stddef.h>
#include <stdint.h>

namespace bt {

#if defined(__CUDACC__)
#define BT_HD __host__ __device__
#else
#define BT_HD
#endif

// Work-item kinds (equal to the public BT_CL_* codelet ids).
enum : uint32_t { K_SCAL = 1, K_AXPY = 2, K_COPY = 3 };

// DItem::meta: kind (bits 0-3) | K_SINGLE_PRED (bit 4) | priority level
// (bits 5-7, device_abi Bucket) | k (bits 8-18) | K_ITEM_DEPS (bit 19) |
// K_ONE_UNIT (bit 20) | successor count (bits 21-31).
constexpr uint32_t K_MASK = 0xFu;
// the item has exactly one predecessor, so the completion of that
// predecessor makes it ready without touching its pending counter
constexpr uint32_t K_SINGLE_PRED = 1u << 4;
constexpr uint32_t K_LEVEL_SHIFT = 5, K_LEVEL_MASK = 0x7u;
constexpr uint32_t K_K_SHIFT = 8, K_K_MASK = 0x7FFu;            // chained factors, 1..2047
// Chunk-wise release: chunk c of an item covers elements [c*chunk, (c+1)*chunk)
// of each operand, and a predecessor that reached the item through the same
// (sub)handle touched the same elements at the same offsets -- so chunk c of
// the item needs only chunk c of such a predecessor (same length), not all of
// it (SCAL/AXPY/COPY are element-wise).  K_ITEM_DEPS: some predecessor came
// through partition-inherited state (other offsets): wait for whole items.
constexpr uint32_t K_ITEM_DEPS = 1u << 19;
constexpr uint32_t K_ONE_UNIT = 1u << 20;   // the item is one work unit (n <= the epoch's chunk): no length load
constexpr uint32_t K_NSUCC_SHIFT = 21, K_NSUCC_ESC = 0x7FFu;   // 2047: the count is succ[succ], the list follows

// One work item of an epoch: a task, or a fused chain of SCAL tasks on the
// same (sub)handle.  32 bytes (two 16-byte words), read-only during the kernel:
//   word 0: x, y            word 1: n, meta, arg, succ
// Units per item = ceil(n / EpochArgs::chunk_elems) (computed, not stored).
struct alignas(16) DItem {
  uint64_t x;         // device address of operand 0 (float*)
  uint64_t y;         // device address of operand 1 (AXPY/COPY), else 0
  uint32_t n;         // elements of each operand (< 2^32: bt_vector_data_register)
  uint32_t meta;      // see above
  uint32_t arg;       // SCAL: k == 1: float bits of the factor; k > 1: offset of
                      // the k factors in EpochArgs::factors; AXPY: float bits of a
  uint32_t succ;      // one successor: its item id; more: offset of their ids in
                      // EpochArgs::succ (escaped count: succ[succ] = count, ids after)
  BT_HD uint32_t kind() const { return meta & K_MASK; }
  BT_HD uint32_t k() const { return (meta >> K_K_SHIFT) & K_K_MASK; }
  BT_HD uint32_t nsucc_field() const { return meta >> K_NSUCC_SHIFT; }
  BT_HD bool single_pred() const { return (meta & K_SINGLE_PRED) != 0; }
};
static_assert(sizeof(DItem) == 32, "DItem layout");
BT_HD inline uint32_t make_meta(uint32_t kind, bool single_pred, uint32_t k, uint64_t nsucc, bool item_deps = false,
                                bool one_unit = false) {
  return kind | (single_pred ? K_SINGLE_PRED : 0u) | (k << K_K_SHIFT) | (item_deps ? K_ITEM_DEPS : 0u) |
         (one_unit ? K_ONE_UNIT : 0u) |
         ((uint32_t)(nsucc < K_NSUCC_ESC ? nsucc : K_NSUCC_ESC) << K_NSUCC_SHIFT);
}
BT_HD inline uint32_t units_of(uint32_t n, uint64_t chunk_elems) {
  // (the common single-unit case without a division: chains of small items)
  return n <= chunk_elems ? 1u : (uint32_t)(((uint64_t)n + chunk_elems - 1) / chunk_elems);
}

// Epoch counters, in device memory, initialised by the host upload.
struct alignas(64) Counters {
  unsigned long long head;    // next ticket (queue position) to take
  unsigned long long tail;    // next free queue position
  unsigned int error;         // nonzero: a CTA detected a fault (see ERR_*)
  unsigned int abort;         // set with error: every CTA leaves its loop
  unsigned long long done;    // units completed and released
  unsigned long long trace_next;  // next trace record (BT_FLAG_TIMESTAMPS)
  unsigned int exited;        // CTAs that left the kernel (the last one reports to the host)
  unsigned int pad;
  unsigned long long spare[2];
};
static_assert(sizeof(Counters) == 64, "Counters layout");

enum : uint32_t { ERR_NONE = 0, ERR_BAD_KIND = 1, ERR_WATCHDOG = 2, ERR_BAD_UNIT = 3 };

// ---- priority ready queue (PAPER.md:91-96 HEFT, 1005-1018) --
// DAG epochs on the "sw" kernel order ready work by the item's upward rank
// (bytes on the longest path from the item to the end of the epoch, the
// item's own included): items are dealt to kMaxBuckets levels (DItem::meta
// level bits, higher = more urgent), and every level is a FIFO of its own.  A
// level's unit count is known on the host, so a level is a ticket queue like
// the single FIFO: a CTA holds at most one ticket per level (taken only when
// the level has unclaimed units, so no CTA waits on an empty level while others
// have work), runs the most urgent of its published tickets, and leaves when
// every level is exhausted.  No CAS anywhere.
// Level b's positions: t < ready -> queue[rbase + t] (initially ready units,
// uploaded), else queue[U0 + pbase + t - ready] (published at release; the
// region after the U0 initially ready units is EMPTY at launch).
constexpr int kMaxBuckets = 8;   // DItem::meta level bits
struct alignas(16) Bucket {
  unsigned long long head;   // next ticket
  unsigned long long tail;   // positions reserved by releases (starts at ready)
  uint32_t total;            // units of this level in the epoch
  uint32_t ready;            // initially ready units
  uint32_t rbase;            // first initially ready unit in queue[]
  uint32_t pbase;            // first published unit in queue[U0 + ...]
};
static_assert(sizeof(Bucket) == 32, "Bucket layout");

// A queue slot holds (item << 32) | chunk; EMPTY until published.
constexpr unsigned long long Q_EMPTY = ~0ull;

struct EpochArgs {
  const DItem *items;
  int32_t *pending;             // unfinished predecessors per item (single-unit items)
  int32_t *cpending;            // ... per unit (unit_base[item] + chunk) of items of several units with
                                // several predecessors (chunk-wise release); null if the epoch has none
  uint32_t *chunk_done;         // finished units per item
  const uint32_t *succ;
  const float *factors;
  unsigned long long *queue;    // total_units slots
  Counters *ctr;
  Counters *host_ctr;           // mapped pinned host memory: the last CTA copies *ctr here
  unsigned long long *trace;    // 4 timestamps per unit, or null
  uint32_t *trace_item;         // item per unit, or null
  const uint32_t *unit_base;    // first unit of each item (prefix of its units): index of its
                                // units' pending counters and trace records
  Bucket *bk;                   // priority levels (scheduler_kernel_swp), else null
  uint32_t nbuckets;
  uint32_t nready;              // U0: initially ready units (queue[0, U0))
  uint64_t total_units;
  uint64_t chunk_elems;         // elements per unit (multiple of 8)
  uint64_t watchdog_ns;         // spin limit before declaring ERR_WATCHDOG
  uint32_t nitems;
  unsigned *stream_abort;       // stream launch: the launch-wide abort flag (StreamCtl::abort), else null
};

// ---- direct launch: an epoch of a few hundred independent items (no edges)
// runs as one plain grid over its items, described in the kernel parameters:
// no queue, no counters, no blob upload (the paper's running example C1 and
// the fused C2 chain -- 256 items of k = 16 -- are such epochs) --------------
// Two sizes: a small parameter block for tiny epochs (the launch copies the
// whole block: C1's latency), a large one (kernel parameters may take up to
// 32,764 bytes since CUDA 12.1) for epochs of up to 512 items.
constexpr int kDirectItemsSmall = 16, kDirectFactorsSmall = 256;
constexpr int kDirectItems = 512;       // items per direct launch (at most)
constexpr int kDirectFactors = 1024;    // distinct chained factors per direct launch (at most)
// A group of items with the same kind, length, factors / scalar whose operands
// advance by one stride (C2's 256 tiles x 16 sweeps: ONE group): items
// first .. (the next group's first) - 1, item first + j at x + j * stride
// (y + j * stride).  Groups keep the launch's parameter block small.
struct DirectItem {
  uint64_t x, y, n;   // as DItem (the group's first item)
  uint32_t kind;      // K_SCAL / K_AXPY / K_COPY
  uint32_t k;         // SCAL: chained factors
  uint32_t arg;       // SCAL: offset of its factors in DirectArgs::factors; AXPY: float bits of a
  uint32_t first;     // index of the group's first item (groups in item order)
  uint64_t stride;    // bytes from one item's operands to the next one's
};
template <int NI, int NF>
struct DirectArgsT {
  uint32_t nitems;    // groups
  uint32_t chunk;     // elements per CTA (grid.x covers the largest item; grid.y = items)
  DirectItem items[NI];
  float factors[NF];
};
using DirectArgs = DirectArgsT<kDirectItems, kDirectFactors>;
using DirectArgsSmall = DirectArgsT<kDirectItemsSmall, kDirectFactorsSmall>;

// ---- stream launch (one persistent launch consumes a growing
// sequence of sub-epochs) ----------------------------------------------------
// The pipelined rounds of one SCAL run are sub-epochs of ONE launch of the
// "sw" kernel: the host builds, uploads and publishes sub-epoch r while the
// kernel already runs sub-epochs < r.  Sub-epochs are independent (disjoint
// handles; everything they depend on precedes the launch in stream order), so
// a CTA only needs to know which sub-epoch a queue ticket falls in: tickets
// are taken from one launch-wide counter and sub-epoch r owns tickets
// [base_r, base_r + total_units_r) with base_r = sum of the earlier subs'
// units.  The host publishes sub-epoch r by copying its EpochArgs into
// subs[r] and then r + 1 into `published` (two stream-ordered copies after
// the copy of its blob); the kernel reads subs[r] only after observing
// published > r with ld.acquire.
constexpr int kMaxSubs = 16;
constexpr int kMaxStreamGrid = 2048;   // CTAs of a stream launch (abandoned-ticket slots)
constexpr unsigned kStreamClosed = 1u << 31;
//
// Closing (launch-serialising tools, a stalled host): the host may be unable to
// publish while the launch runs -- under ncu, compute-sanitizer or
// CUDA_LAUNCH_BLOCKING=1 the launch call itself returns only when the kernel
// ends.  A CTA waiting for a publication counts itself in `state`; when EVERY
// CTA has waited longer than the quiescence limit, one of them closes the
// launch with a CAS (count == grid -> count | kStreamClosed).  A CTA leaving
// its wait decrements `state` and, if the returned value carries the closed
// bit, abandons too; the CAS and the decrements are RMWs of one word, so no
// CTA starts a sub-epoch the closer has given up.  Every CTA then holds one
// ticket of an unpublished sub-epoch; it appends it to abandoned[] and exits
// (its other slot drained), so the tickets taken are exactly those run plus
// those abandoned.  The run's RESUME launch (same kernel, enqueued after the
// last publication) exits at once unless the last CTA of the first launch set
// `resume`; then it runs the abandoned tickets first, then fresh ones.
struct alignas(64) StreamCtl {
  unsigned long long ticket;    // next launch-wide ticket
  unsigned published;           // sub-epochs whose args and blobs are in device memory
  unsigned abort;               // any sub-epoch's fault stops every CTA
  unsigned exited;              // CTAs that left the kernel
  unsigned nsub;                // sub-epochs of this launch (fixed at its start)
  unsigned state;               // CTAs waiting for a publication | kStreamClosed
  unsigned resume;              // the first launch closed: the resume launch runs the rest
  unsigned nabandoned;          // tickets abandoned at the close
  unsigned ab_take;             // ... taken again by the resume launch
  unsigned pad[6];
  EpochArgs subs[kMaxSubs];
  unsigned long long abandoned[kMaxStreamGrid];
};
static_assert(sizeof(StreamCtl) % 64 == 0 && offsetof(StreamCtl, subs) == 64, "StreamCtl layout");

}  // namespace bt
