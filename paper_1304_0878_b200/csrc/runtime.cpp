// runtime.cpp -- libbtask.so: the C ABI of include/btask.h.
//
// Host side of the task-stream executor: data registry,
// partitioning, asynchronous task submission with
// dependency inference (builder.hpp),
// epoch packing + upload, launch of the persistent scheduler kernel
// (scheduler.cu), wait / acquire / release / unregister (PAPER.md:213-214,
// 504-507) and owner-computes rank filtering.
#include <cuda_runtime.h>
#include <errno.h>
#if defined(__x86_64__)
#include <immintrin.h>
#endif
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <memory>
#include <tuple>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/btask.h"
#include "builder.hpp"
#include "comm.hpp"
#include "device_abi.h"
#include "pool.hpp"

namespace bt {
cudaError_t launch_epoch(const EpochArgs &args, int grid, cudaStream_t stream, int kernel);
cudaError_t launch_stream(StreamCtl *ctl, uint64_t watchdog_ns, uint64_t quiesce_ns, int grid, cudaStream_t stream,
                          bool prefetch, bool resume);
cudaError_t launch_direct(const DirectArgs &args, unsigned grid_x, unsigned nall, cudaStream_t stream);
cudaError_t scheduler_occupancy(int *blocks_per_sm, int *block);
cudaError_t scheduler_occupancy_wq(int *blocks_per_sm, int *block);
cudaError_t launch_stage(void *dst, const void *src_mapped, size_t bytes, unsigned long long *q_empty, size_t nq,
                         uint32_t *zero, size_t nz, cudaStream_t stream);
cudaError_t launch_gate(const volatile unsigned *flag_dev, uint64_t watchdog_ns, cudaStream_t stream);
int max_factors();
}  // namespace bt

using namespace bt;

namespace {

constexpr uint32_t kMaxChunkBytes = 256u << 10;     // adaptive chunking: upper bound
constexpr uint64_t kMinChunkElems = 16384;          // adaptive chunking: lower bound (64 KiB: a unit costs
                                                    // ~1 us of pop + release; C2 fused 62 -> 43 us, tools/c2_chunks.py)
constexpr uint32_t kUnitsPerCta = 16;               // adaptive chunking: target work units per CTA
constexpr uint32_t kDefaultMaxFused = 256;
constexpr uint32_t kDefaultParallelMin = 16384;
constexpr int kDefaultRounds = 4;
#ifndef BT_ROUNDS_UPLOADING
#define BT_ROUNDS_UPLOADING 8
#endif
constexpr int kRoundsUploading = BT_ROUNDS_UPLOADING;   // rounds for partitions of data still being uploaded
constexpr uint32_t kDefaultPipelineMin = 131072;
constexpr int kEpochRing = 12;                      // epoch buffers in flight (>= rounds + 2)
constexpr uint64_t kWatchdogNs = 20ull * 1000 * 1000 * 1000;   // 20 s
constexpr uint64_t kQuiesceNs = 50ull * 1000 * 1000;             // stream launch: close after 50 ms without a publication
constexpr size_t kParallelPack = 1024;              // items above which the pack runs on the pool
constexpr uint64_t kWarpUnitMax = 4096;             // units of at most this many elements use "wq"
constexpr uint64_t kPrefetchBelowK = 32;            // "sw" epochs with shorter average chains prefetch
constexpr uint64_t kUploadChunk = 64ull << 20;      // registrations >= this upload in chunks on a copy stream
constexpr size_t kStageBelow = 1u << 20;            // epoch blobs up to this size are pulled by the set-up kernel
constexpr uint64_t kDagChunkElems = 16384;          // work-unit cap (64 KiB) for epochs with dependencies

const char *codelet_name(int c) {
  switch (c) {
    case BT_CL_SCAL: return "vector_scal";
    case BT_CL_AXPY: return "axpy";
    case BT_CL_COPY: return "copy";
    default: return "unknown";
  }
}

double now_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

enum : uint32_t { F_LIVE = 1, F_PARTITIONED = 2, F_BLOCKED = 4 };

// Hot per-(sub)handle fields read on every insert (32 bytes).
struct SlotHot {
  uint32_t gen = 1;
  uint32_t flags = 0;
  int32_t rank = 0;
  uint32_t grp = 0;           // builder group of the slot's 64-slot block (round * P + lane)
  float *dptr = nullptr;      // device address of element 0 (null: no local storage)
  uint64_t nx = 0;
};

struct Slot {
  uint32_t parent = NONE;
  uint32_t child_index = 0;
  uint32_t nparts = 0;        // partitioned into nparts children if > 0
  uint32_t first_child = NONE;
  uint32_t root = NONE;       // top-level ancestor (itself for a top-level handle)
  uint64_t offset = 0;        // element offset inside the root
  void *hptr = nullptr;       // root only: registered pointer
  int home_node = 0;
  int acquired = 0;           // 0, BT_R or BT_RW (on the acquired handle itself)
  bool owns_dev = false;      // root only: runtime-allocated replica
  bool ipc_alloc = false;     // root only: replica from cudaMalloc (shareable with other ranks)
  uint64_t reg_key = 0;       // root only: registration ordinal (equal on all ranks)
  uint8_t prounds = 0;        // partitioned parent: rounds its parts were dealt to
  int8_t pgeo = 0;            // ... geometrically (round_of: 1 growing, 2 shrinking)
};

struct EpochBuf {
  char *hblob = nullptr;       // pinned + mapped
  char *hblob_dev = nullptr;   // its device-side address
  size_t hcap = 0;
  char *dblob = nullptr;
  size_t dcap = 0;
  cudaEvent_t start = nullptr, end = nullptr, done = nullptr;
  bool inflight = false;
  uint64_t seq = 0;           // launch order
  uint64_t units = 0;
  bool traced = false;
  bool timed = true;          // start/end bracket a launch (false: a later sub-epoch of a stream launch)
  bool held = false;          // a deferred stream launch's sub-epoch, not launched yet: never picked
  Counters *hctr = nullptr;     // mapped pinned: written by the kernel's last CTA
  Counters *hctr_dev = nullptr;
  size_t trace_off_h = 0;     // offset of the trace copy in hblob
};

// Host <-> device coherence of one host-homed registered vector (PAPER.md:
// 97-99 "transferring data between main memory and GPUs as needed").
//  * lazy upload ("W-first accesses skip upload"): nothing is
//    copied at registration; the first epoch that READS a range uploads it
//    (in 64 MiB pieces on a copy stream, each with an event the epoch waits
//    for), while a range whose first access is write-only (a COPY
//    destination) becomes valid on the device without any upload;
//  * write-back: when an epoch writes a range of the vector for the first
//    time since registration, that range is copied back to the host buffer
//    right after the epoch (on a second copy stream), so unregister finds the
//    host copy current.  A range written again is marked dirty; acquire /
//    unregister copy back exactly the dirty ranges they need.
struct UploadChunk {
  uint64_t lo, hi;            // device byte range
  cudaEvent_t ev;             // recorded after its H2D copy
};
// Disjoint half-open byte ranges, merged on insertion (a long-lived host-homed
// vector written by many epochs keeps a handful of ranges, not one per epoch).
struct RangeSet {
  std::map<uint64_t, uint64_t> m;   // lo -> hi
  bool overlaps(uint64_t lo, uint64_t hi) const {
    auto it = m.lower_bound(hi);    // first range starting at or after hi
    if (it == m.begin()) return false;
    --it;
    return it->second > lo;
  }
  void add(uint64_t lo, uint64_t hi) {
    auto it = m.upper_bound(lo);
    if (it != m.begin() && std::prev(it)->second >= lo) {
      --it;
      lo = it->first;
      hi = std::max(hi, it->second);
      it = m.erase(it);
    }
    while (it != m.end() && it->first <= hi) {
      hi = std::max(hi, it->second);
      it = m.erase(it);
    }
    m.emplace(lo, hi);
  }
  bool empty() const { return m.empty(); }
  // the parts of [lo, hi) in the set, appended to out; removed from the set if take
  void pieces(uint64_t lo, uint64_t hi, std::vector<std::pair<uint64_t, uint64_t>> &out, bool take) {
    auto it = m.upper_bound(lo);
    if (it != m.begin() && std::prev(it)->second > lo) --it;
    while (it != m.end() && it->first < hi) {
      const uint64_t rlo = it->first, rhi = it->second;
      const uint64_t a = std::max(lo, rlo), b = std::min(hi, rhi);
      out.emplace_back(a, b);
      if (!take) {
        ++it;
        continue;
      }
      it = m.erase(it);
      if (rlo < a) m.emplace(rlo, a);   // keys below `it`: the iterator stays valid
      if (b < rhi) {                    // b == hi: the last overlapping range
        m.emplace(b, rhi);
        break;
      }
    }
  }
  void remove(uint64_t lo, uint64_t hi) {
    std::vector<std::pair<uint64_t, uint64_t>> tmp;
    pieces(lo, hi, tmp, true);
  }
};

struct RootCache {
  uint64_t dlo = 0, dhi = 0;  // device byte range of the replica
  std::vector<UploadChunk> uploads;   // issued host -> device copies (events), until the next wait
  RangeSet pending;           // device bytes whose replica is not valid yet: the host holds the data
                              // (uploaded on the first read; a write-only first access skips it)
  RangeSet written;           // device byte ranges written by epochs
  RangeSet dirty;             // written again after their eager write-back: copied back at acquire/unregister
  RangeSet ewrite;            // scratch: ranges the epoch being flushed writes
  bool wb = false;            // eager write-backs issued
};

}  // namespace

struct bt_runtime {
  bt_config cfg;
  // BT_DEBUG_ERRORS: the last scheduling events, dumped with a device fault
  char evlog[64][96] = {};
  unsigned evn = 0;
  void ev(const char *fmt, ...) __attribute__((format(printf, 2, 3))) {
    static const bool on = getenv("BT_DEBUG_ERRORS") != nullptr;
    if (!on) return;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(evlog[evn++ % 64], 96, fmt, ap);
    va_end(ap);
  }
  void ev_dump() {
    for (unsigned i = evn > 64 ? evn - 64 : 0; i < evn; ++i) fprintf(stderr, "  ev %u: %s\n", i, evlog[i % 64]);
  }
  bool host_only = false;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sms = 0;
  int grid_max = 0;
  int block = 0;
  int grid_wq = 0, block_wq = 0;   // the warp-worker kernel
  int poisoned = 0;
  std::string last_error;

  std::vector<SlotHot> hot;
  // phase-1 key per slot: (gen << 32) | (grp << 1) | ok, ok = a local SCAL
  // target (live, not partitioned or blocked, has device storage, this rank);
  // rebuilt by scal_run_parallel when any SlotHot changed (key_dirty)
  std::vector<uint64_t> key;
  bool key_dirty = true;
  std::vector<Slot> slots;
  std::vector<DepState> deps;
  std::map<uint32_t, std::vector<uint32_t>> free_ranges;        // count -> starts
  std::map<uintptr_t, std::pair<uintptr_t, uint32_t>> ranges;   // start -> (end, root slot)
  std::unordered_map<uintptr_t, uint32_t> by_ptr;               // exact base -> root slot
  uint32_t live_roots = 0;

  Builder builder;
  std::unique_ptr<Pool> pool;
  std::vector<Lane> lanes;
  std::vector<vec<RunRec>> runs;                        // [chunk][round * P + lane]: runs of the stream
  std::vector<uint64_t> run_tasks;                      // [chunk][round * P + lane]: tasks in those runs
  int npool = 1;
  int nrounds = 1;        // bucket rounds (max over round policies)
  int rounds_default = 1; // rounds of a partition of device-resident data
  EpochBuf ep[kEpochRing];
  uint64_t ep_seq = 0;
  cudaStream_t rstream[2] = {nullptr, nullptr};   // round streams (pipelined SCAL runs)
  // stream launch (device_abi.h StreamCtl): the rounds of one
  // pipelined SCAL run as sub-epochs of one "sw" launch.  want: the run asks
  // for it (decided at its first flush); active: sub-epochs next..nsub-1 join
  // the running launch
  StreamCtl *sctl = nullptr;
  char *close_h = nullptr;   // pinned: published values 1..kMaxSubs, then a zero EpochArgs (close_stream)
  struct {
    bool want = false, active = false;
    unsigned nsub = 0, next = 0;
    bool prefetch = false;
    bool started = false;
    bool launched = false;   // the run's launch is enqueued
    bool defer = false;      // the launch is enqueued after the last publication
    uint64_t run_tasks = 0, cur_tasks = 0;   // local tasks of the run / of the sub-epoch being flushed
    uint64_t max_tasks = 0;                  // local tasks of the run's largest sub-epoch
    EpochBuf *bufs[kMaxSubs] = {};    // the sub-epochs' buffers (bufs[0]'s start/end time the launch)
  } sl;
  cudaEvent_t ev_pub0 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_round[2] = {nullptr, nullptr};
  cudaEvent_t span_start = nullptr, span_end = nullptr;
  bool span_open = false;
  cudaStream_t h2d = nullptr, d2h = nullptr;        // copy streams (chunked upload, write-back)
  std::unordered_map<uint32_t, RootCache> caches;   // host-homed roots with a replica
  std::vector<cudaEvent_t> ev_free;
  cudaEvent_t get_event() {
    if (!ev_free.empty()) {
      cudaEvent_t e = ev_free.back();
      ev_free.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    return e;
  }
  void put_event(cudaEvent_t e) { ev_free.push_back(e); }
  bt_stats stats{};
  std::unique_ptr<Comm> comm;   // cross-rank reads (bt_comm_init)
  // Shared copies across ranks (NEXT-4, "lazy MSI across ranks"): every rank
  // sees every task in submission order, so every rank can tell alike whether
  // data a reader copied before has been written since.  wver[root] counts
  // the tasks writing a part of the root (local or not); gver is bumped by
  // everything coarser (a parallel SCAL run, registration, partitioning, rank
  // changes, a host RW release -- collective calls under bt_comm_init).  A
  // cross-rank read whose (wver, gver) equal those of the pair's last transfer
  // of the same range skips the rendezvous on both sides.
  std::vector<uint64_t> wver;
  uint64_t gver = 1;
  std::map<std::tuple<uint64_t, uint64_t, uint64_t, int>, std::pair<uint64_t, uint64_t>> xcache;
  uint64_t reg_seq = 0;         // registrations so far (Slot::reg_key)

  // host-only snapshot storage
  std::vector<uint8_t> snap_kind;
  std::vector<uint32_t> snap_k, snap_npred, snap_off, snap_succ;
  std::vector<uint8_t> snap_flags;
  std::vector<uint32_t> snap_task_item, snap_task_pos;

  // last trace
  std::vector<uint64_t> trace_t;
  std::vector<uint32_t> trace_item;

  // bt_debug_gate flags (mapped pinned words, freed at shutdown)
  std::vector<uint32_t *> gates;

  // pack scratch
  std::vector<uint32_t> succ_off, cursor;
  size_t hcap_max = 0, dcap_max = 0;     // largest epoch buffers allocated so far

  template <class F>
  void par(F &&f) {
    std::function<void(int)> fn = f;
    pool->run(fn);
  }
};

namespace {

int fail(bt_runtime *rt, int err, const char *fmt, ...) {
  if (rt) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    rt->last_error = buf;
    static const bool dbg = getenv("BT_DEBUG_ERRORS") != nullptr;
    if (dbg) fprintf(stderr, "btask error %d: %s\n", err, buf);
  }
  return err;
}

int insert_fail(bt_runtime *rt, int codelet, int err, const char *detail) {
  return fail(rt, err, "failed to insert task `%s': %s (%s)", codelet_name(codelet), strerror(-err), detail);
}

int cuda_fail(bt_runtime *rt, cudaError_t e, const char *what) {
  rt->poisoned = -EIO;
  return fail(rt, -EIO, "%s: %s", what, cudaGetErrorString(e));
}

#define CUDA_TRY(rt, call)                                    \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return cuda_fail((rt), e_, #call); \
  } while (0)

inline bt_handle make_handle(const bt_runtime *rt, uint32_t s) {
  return ((uint64_t)rt->hot[s].gen << 32) | (uint64_t)(s + 1);
}

// Resolve a handle to a live slot, or NONE.
inline uint32_t resolve(const bt_runtime *rt, bt_handle h) {
  const uint64_t idx = (h & 0xFFFFFFFFull);
  if (idx == 0 || idx > rt->hot.size()) return NONE;
  const uint32_t s = (uint32_t)(idx - 1);
  const SlotHot &sh = rt->hot[s];
  if (!(sh.flags & F_LIVE) || sh.gen != (uint32_t)(h >> 32)) return NONE;
  return s;
}

uint32_t alloc_slots(bt_runtime *rt, uint32_t count) {
  auto it = rt->free_ranges.find(count);
  uint32_t s;
  if (it != rt->free_ranges.end() && !it->second.empty()) {
    s = it->second.back();
    it->second.pop_back();
  } else {
    s = (uint32_t)rt->hot.size();
    rt->key_dirty = true;
    rt->hot.resize(s + count);
    rt->slots.resize(s + count);
    rt->deps.resize(s + count);
  }
  for (uint32_t i = 0; i < count; ++i) {
    rt->key_dirty = true;
    SlotHot &h = rt->hot[s + i];
    const uint32_t gen = h.gen;
    h = SlotHot();
    h.gen = gen;
    h.flags = F_LIVE;
    const uint32_t k = (s + i) >> 6;    // 64-slot block -> lane k % P, round (k / P) % R
    h.grp = ((k / (uint32_t)rt->npool) % (uint32_t)rt->rounds_default) * (uint32_t)rt->npool + k % (uint32_t)rt->npool;
    rt->slots[s + i] = Slot();
    rt->deps[s + i] = DepState();
  }
  return s;
}

void free_slots(bt_runtime *rt, uint32_t s, uint32_t count) {
  for (uint32_t i = 0; i < count; ++i) {
    rt->key_dirty = true;
    SlotHot &h = rt->hot[s + i];
    h.flags = 0;
    if (++h.gen == 0) h.gen = 1;
    rt->deps[s + i] = DepState();
  }
  rt->free_ranges[count].push_back(s);
}

void set_blocked(bt_runtime *rt, uint32_t s, bool on) {
  std::vector<uint32_t> stack{s};
  while (!stack.empty()) {
    const uint32_t x = stack.back();
    stack.pop_back();
    rt->key_dirty = true;
    if (on) rt->hot[x].flags |= F_BLOCKED;
    else rt->hot[x].flags &= ~F_BLOCKED;
    const Slot &sl = rt->slots[x];
    for (uint32_t t = 0; t < sl.nparts; ++t) stack.push_back(sl.first_child + t);
  }
}

bool acquired_chain(const bt_runtime *rt, uint32_t s) {
  if (rt->hot[s].flags & F_BLOCKED) return true;
  // a descendant acquired also blocks partition/acquire of s
  std::vector<uint32_t> stack{s};
  while (!stack.empty()) {
    const uint32_t x = stack.back();
    stack.pop_back();
    if (rt->slots[x].acquired) return true;
    const Slot &sl = rt->slots[x];
    for (uint32_t t = 0; t < sl.nparts; ++t) stack.push_back(sl.first_child + t);
  }
  return false;
}

int check_live(bt_runtime *rt) {
  if (!rt) return -EINVAL;
  if (rt->poisoned) return fail(rt, rt->poisoned, "runtime poisoned by an earlier device error");
  return 0;
}

// ---------------------------------------------------------------- epochs --

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Epoch buffers grow to the largest size any ring slot has needed so far, so
// each slot allocates about once instead of growing step by step (pinned and
// device allocations cost milliseconds each).
int ensure_host(bt_runtime *rt, EpochBuf &e, size_t need) {
  if (e.hcap >= need) return 0;
  if (e.hblob) cudaFreeHost(e.hblob);
  e.hblob = nullptr;
  size_t cap = std::max({need, e.hcap + e.hcap / 2, rt->hcap_max});
  rt->hcap_max = cap;
  CUDA_TRY(rt, cudaHostAlloc((void **)&e.hblob, cap, cudaHostAllocPortable | cudaHostAllocMapped));
  CUDA_TRY(rt, cudaHostGetDevicePointer((void **)&e.hblob_dev, e.hblob, 0));
  e.hcap = cap;
  return 0;
}

int ensure_dev(bt_runtime *rt, EpochBuf &e, size_t need) {
  if (e.dcap >= need) return 0;
  // tests: BT_DEBUG_FAIL_DEV_ALLOC=n fails the n-th epoch allocation (1-based)
  static long fail_at = getenv("BT_DEBUG_FAIL_DEV_ALLOC") ? atol(getenv("BT_DEBUG_FAIL_DEV_ALLOC")) : 0;
  if (fail_at > 0 && --fail_at == 0) return fail(rt, -ENOMEM, "cannot allocate epoch memory (injected failure)");
  if (e.dblob) cudaFree(e.dblob);
  e.dblob = nullptr;
  size_t cap = std::max({need, e.dcap + e.dcap / 2, rt->dcap_max});
  rt->dcap_max = cap;
  cudaError_t err = cudaMalloc((void **)&e.dblob, cap);
  if (err != cudaSuccess) {
    cudaGetLastError();
    e.dcap = 0;
    return fail(rt, -ENOMEM, "cannot allocate %zu bytes of epoch memory: %s", cap, cudaGetErrorString(err));
  }
  e.dcap = cap;
  return 0;
}

// Wait for an in-flight epoch, account its time, check its error counter.
int retire(bt_runtime *rt, EpochBuf &e) {
  if (!e.inflight) return 0;
  cudaError_t err = cudaEventSynchronize(e.done);
  e.inflight = false;
  if (err != cudaSuccess) return cuda_fail(rt, err, "epoch completion");
  float ms = 0.f;
  if (e.timed && cudaEventElapsedTime(&ms, e.start, e.end) == cudaSuccess) rt->stats.device_ms += ms;
  const Counters *c = e.hctr;
  // a stream launch that closed (no publication for kQuiesceNs): its resume
  // launch ran the rest, until e.done
  if (e.timed && c->pad && cudaEventElapsedTime(&ms, e.end, e.done) == cudaSuccess) {
    rt->stats.device_ms += ms;
    rt->stats.stream_resumes += 1;
  }
  if (c->error != ERR_NONE) {
    rt->poisoned = -EIO;
    return fail(rt, -EIO, "device scheduler fault (code %u%s)", c->error,
                c->error == ERR_WATCHDOG ? ": watchdog, a unit was never released" : "");
  }
  if (c->done != e.units) {
    static const bool dbg = getenv("BT_DEBUG_ERRORS") != nullptr;
    if (dbg) {
      fprintf(stderr, "btask retire: buffer %d seq %llu units %llu done %llu error %u exited %u timed %d\n",
              (int)(&e - rt->ep), (unsigned long long)e.seq, (unsigned long long)e.units,
              (unsigned long long)c->done, c->error, c->exited, (int)e.timed);
      rt->ev_dump();
      if (rt->sctl) {
        unsigned char hdr[64];
        cudaError_t ce = cudaMemcpy(hdr, rt->sctl, 64, cudaMemcpyDeviceToHost);
        unsigned long long tk;
        unsigned w[4];
        memcpy(&tk, hdr, 8);
        memcpy(w, hdr + 8, 16);
        unsigned pd[4];
        memcpy(pd, hdr + 24, 16);
        fprintf(stderr, "  StreamCtl (%d): ticket %llu published %u abort %u exited %u nsub %u state %x resume %u "
                        "abandoned %u taken %u\n",
                (int)ce, tk, w[0], w[1], w[2], w[3], pd[0], pd[1], pd[2], pd[3]);
        for (unsigned q = 0; q < kMaxSubs && rt->sl.bufs[q]; ++q) {
          Counters c2;
          cudaMemcpy(&c2, rt->sl.bufs[q]->dblob, sizeof c2, cudaMemcpyDeviceToHost);
          fprintf(stderr, "  sub %u ctr: head %llu tail %llu error %u abort %u done %llu exited %u\n", q, c2.head,
                  c2.tail, c2.error, c2.abort, c2.done, c2.exited);
        }
      }
    }
    rt->poisoned = -EIO;
    return fail(rt, -EIO, "device scheduler ended early (%llu of %llu units)", (unsigned long long)c->done,
                (unsigned long long)e.units);
  }
  if (e.traced) {
    const uint64_t *t = reinterpret_cast<const uint64_t *>(e.hblob + e.trace_off_h);
    rt->trace_t.assign(t, t + 4 * e.units);
    const uint32_t *ti = reinterpret_cast<const uint32_t *>(e.hblob + e.trace_off_h + 32 * e.units);
    rt->trace_item.assign(ti, ti + e.units);
  }
  return 0;
}

// Upload device byte range [lo, hi) of host-homed root `root` from the
// registered host buffer on the H2D copy stream, in pieces of at most
// kUploadChunk, each with an event that epochs reading it wait for
// (RootCache::uploads).
int upload_range(bt_runtime *rt, uint32_t root, RootCache &c, uint64_t lo, uint64_t hi) {
  const char *host = static_cast<const char *>(rt->slots[root].hptr);
  for (uint64_t a = lo; a < hi; a += kUploadChunk) {
    const uint64_t len = std::min<uint64_t>(kUploadChunk, hi - a);
    CUDA_TRY(rt, cudaMemcpyAsync(reinterpret_cast<void *>(a), host + (a - c.dlo), len, cudaMemcpyHostToDevice, rt->h2d));
    UploadChunk u{a, a + len, rt->get_event()};
    CUDA_TRY(rt, cudaEventRecord(u.ev, rt->h2d));
    c.uploads.push_back(u);
    rt->stats.h2d_data_bytes += len;
  }
  return 0;
}

// Make device bytes [lo, hi) of a host-homed root valid: upload the parts still pending.
int ensure_device(bt_runtime *rt, uint32_t root, RootCache &c, uint64_t lo, uint64_t hi) {
  if (c.pending.empty()) return 0;
  std::vector<std::pair<uint64_t, uint64_t>> ps;
  c.pending.pieces(lo, hi, ps, true);
  for (const auto &pc : ps)
    if (int e = upload_range(rt, root, c, pc.first, pc.second)) return e;
  return 0;
}

// Host <-> device coherence of the epoch about to launch (items in topological
// order): every range an item reads is uploaded if still pending; a range whose
// first access is a COPY destination (write-only) just stops being pending;
// the ranges the epoch writes are collected per root (RootCache::ewrite) for
// the write-back after it.
int epoch_coherence(bt_runtime *rt) {
  struct Ref {
    uint64_t lo, hi;
    uint32_t root;
    RootCache *c;
  };
  std::vector<Ref> refs;
  for (auto &kv : rt->caches) {
    kv.second.ewrite.m.clear();
    refs.push_back(Ref{kv.second.dlo, kv.second.dhi, kv.first, &kv.second});
  }
  std::sort(refs.begin(), refs.end(), [](const Ref &a, const Ref &b) { return a.lo < b.lo; });
  auto find = [&](uint64_t a) -> Ref * {
    auto it = std::upper_bound(refs.begin(), refs.end(), a, [](uint64_t v, const Ref &r) { return v < r.lo; });
    if (it == refs.begin()) return nullptr;
    --it;
    return a < it->hi ? &*it : nullptr;
  };
  // ranges read while pending are collected (merged) and uploaded once, in
  // large copies, before the epoch; a write-only first access removes its range
  std::vector<RangeSet> load(refs.size());
  std::vector<std::pair<uint64_t, uint64_t>> ps;
  for (const HItem &it : rt->builder.items) {
    const uint64_t bytes = 4 * it.n;
    auto rd = [&](uint64_t a) {
      Ref *r = find(a);
      if (!r || r->c->pending.empty()) return;
      ps.clear();
      r->c->pending.pieces(a, a + bytes, ps, true);
      for (const auto &pc : ps) load[r - refs.data()].add(pc.first, pc.second);
    };
    auto wr = [&](uint64_t a, bool reads) {
      Ref *r = find(a);
      if (!r) return;
      if (reads) rd(a);
      else if (!r->c->pending.empty()) r->c->pending.remove(a, a + bytes);   // write-only first: no upload (R7)
      r->c->ewrite.add(a, a + bytes);
    };
    switch (it.kind) {
      case K_SCAL: wr(it.x, true); break;
      case K_AXPY: rd(it.x); wr(it.y, true); break;
      default: rd(it.x); wr(it.y, it.x == it.y); break;   // COPY x -> x reads x
    }
  }
  for (size_t i = 0; i < refs.size(); ++i)
    for (const auto &rg : load[i].m)
      if (int e = upload_range(rt, refs[i].root, *refs[i].c, rg.first, rg.second)) return e;
  return 0;
}

// Elements per work unit for this epoch: fixed (bt_config.chunk_bytes), or
// adaptive: about kUnitsPerCta units per persistent CTA, a power of two in
// [8 KiB, 256 KiB] -- small enough to balance the tail, large enough to
// amortise one pop + release per unit.
uint64_t chunk_elems_for(const bt_runtime *rt, uint64_t total_elems) {
  if (rt->cfg.chunk_bytes) return std::max<uint64_t>(8, (rt->cfg.chunk_bytes / 4) / 8 * 8);
  const uint64_t target = total_elems / ((uint64_t)std::max(1, rt->grid_max) * kUnitsPerCta);
  uint64_t c = kMinChunkElems;
  while (c * 2 <= target && c * 2 <= kMaxChunkBytes / 4) c *= 2;
  return c;
}

// Split [0, n) into the pool's ranges.
inline void range_of(size_t n, int P, int p, size_t &lo, size_t &hi) {
  lo = n * (size_t)p / (size_t)P;
  hi = n * (size_t)(p + 1) / (size_t)P;
}

// Launch-serialising tools (ncu, compute-sanitizer, CUDA_LAUNCH_BLOCKING=1)
// return from a launch only when the kernel ends: a stream launch enqueued
// before its last publication would wait for publications the blocked host
// cannot make (until it closes, kQuiesceNs later).  Under them, and with
// BT_STREAM_DEFER=1, the launch is enqueued after the last publication.
bool stream_defer() {
  static const bool d = [] {
    const char *lb = getenv("CUDA_LAUNCH_BLOCKING");
    if (getenv("BT_STREAM_NODEFER")) return false;   // tests: exercise the close + resume path
    // Nsight Compute's target environment (checked on the box: ncu 2025.2
    // sets NV_NSIGHT_INJECTION_* and NV_COMPUTE_PROFILER_PERFWORKS_DIR);
    // CUDA_INJECTION64_PATH: injection-based tools in general
    return getenv("BT_STREAM_DEFER") != nullptr || getenv("CUDA_INJECTION64_PATH") != nullptr ||
           getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") != nullptr ||
           getenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR") != nullptr || (lb && lb[0] == '1');
  }();
  return d;
}

uint64_t quiesce_ns() {
  static const uint64_t q = getenv("BT_QUIESCE_US") ? strtoull(getenv("BT_QUIESCE_US"), nullptr, 10) * 1000
                                                    : kQuiesceNs;
  return q;
}

// Enqueue the run's stream launch on rstream[0] (after sub-epoch 0's copies;
// deferred: after the last publication).
int enqueue_stream_launch(bt_runtime *rt) {
  cudaStream_t ls = rt->rstream[0];
  EpochBuf &e0 = *rt->sl.bufs[0];
  CUDA_TRY(rt, cudaEventRecord(e0.start, ls));
  rt->stats.grid = (uint32_t)rt->grid_max;
  rt->stats.block = (uint32_t)rt->block;
  rt->stats.kernel_launches += 1;
  rt->stats.sched_launches += 1;
  CUDA_TRY(rt, launch_stream(rt->sctl, kWatchdogNs, quiesce_ns(), rt->grid_max, ls, rt->sl.prefetch, false));
  CUDA_TRY(rt, cudaEventRecord(e0.end, ls));
  rt->sl.launched = true;
  return 0;
}

// Every sub-epoch of the run is published (or closed): order the launch
// stream after the last publication; a deferred launch is enqueued now,
// otherwise the RESUME launch (device_abi.h StreamCtl: it exits at once unless
// the running launch closed for want of publications, then runs the rest).
// The sub-epochs' buffers complete (done events) after that.
int finish_stream_run(bt_runtime *rt) {
  if (!rt->sl.bufs[0]) return 0;   // nothing enqueued for this run
  cudaStream_t ls = rt->rstream[0];
  CUDA_TRY(rt, cudaEventRecord(rt->ev_pub0, rt->rstream[1]));
  CUDA_TRY(rt, cudaStreamWaitEvent(ls, rt->ev_pub0, 0));
  if (!rt->sl.launched) {
    if (int rc = enqueue_stream_launch(rt)) return rc;
  } else {
    rt->stats.kernel_launches += 1;
    CUDA_TRY(rt, launch_stream(rt->sctl, kWatchdogNs, quiesce_ns(), rt->grid_max, ls, rt->sl.prefetch, true));
  }
  for (EpochBuf *b : rt->sl.bufs)
    if (b && b->held) {
      CUDA_TRY(rt, cudaEventRecord(b->done, ls));
      b->held = false;
    }
  // the run's join (scal_run_parallel) waits for ev_round[0]: after all of it
  CUDA_TRY(rt, cudaEventRecord(rt->ev_round[0], ls));
  return 0;
}

// End the running stream launch early: sub-epochs next..nsub-1 are published
// empty (zero EpochArgs: no units), so its CTAs finish.  Copies from a pinned
// table whose contents never change (published value q + 1 at index q, then a
// zero EpochArgs), so overlapping closes of successive launches cannot race.
int close_stream(bt_runtime *rt) {
  rt->ev("close stream launch at sub %u of %u", rt->sl.next, rt->sl.nsub);
  rt->stats.stream_closes += 1;
  if (rt->sl.bufs[0]) {   // else nothing of this run reached the device: no kernel reads *sctl
    const unsigned *pub = reinterpret_cast<const unsigned *>(rt->close_h);
    const char *zero_args = rt->close_h + 4 * kMaxSubs;
    cudaStream_t up = rt->rstream[1];
    for (unsigned q = rt->sl.next; q < rt->sl.nsub; ++q) {
      CUDA_TRY(rt, cudaMemcpyAsync(&rt->sctl->subs[q], zero_args, sizeof(EpochArgs), cudaMemcpyHostToDevice, up));
      CUDA_TRY(rt, cudaMemcpyAsync(&rt->sctl->published, &pub[q], 4, cudaMemcpyHostToDevice, up));
    }
  }
  rt->sl.next = rt->sl.nsub;
  rt->sl.active = false;
  return finish_stream_run(rt);
}

// Default pipelined rounds of device-resident partitions are geometric
// (bt_data_partition); BT_UNIFORM_ROUNDS=1 gives equal quarters (comparisons).
bool geometric_rounds() {
  static const bool uniform = getenv("BT_UNIFORM_ROUNDS") != nullptr;
  return !uniform;
}

// Round of part t of n dealt to `rounds` rounds: contiguous equal shares, or
// (4 rounds) geometric shares growing 1/16, 2/16, 4/16, 9/16 (geo = 1) or
// shrinking 9/16, 4/16, 2/16, 1/16 (geo = 2) -- see bt_data_partition.
uint32_t round_of(uint64_t t, uint64_t n, uint32_t rounds, int geo) {
  if (geo == 1) {
    const uint64_t q = t * 16 / n;
    return q < 1 ? 0 : q < 3 ? 1 : q < 7 ? 2 : 3;
  }
  if (geo == 2) {
    const uint64_t q = t * 16 / n;
    return q < 9 ? 0 : q < 13 ? 1 : q < 15 ? 2 : 3;
  }
  return (uint32_t)(t * rounds / n);
}

// A round of a pipelined SCAL run built by Builder::lane_count (direct
// rounds, builder.hpp): the lanes' handle runs in item order and the totals.
struct DirectRound {
  Lane *const *lanes;
  size_t nlanes;
  uint64_t N, E, F, elems, work, tasks;
};

int flush_epoch(bt_runtime *rt, cudaStream_t stream = nullptr, const DirectRound *dr = nullptr) {
  Builder &B = rt->builder;
  if (dr ? dr->N == 0 : B.items.empty()) {
    B.next_epoch();
    return 0;
  }
  if (!stream) stream = rt->stream;
  const double t0 = now_ms();
  // buffer: the lowest-numbered one that is idle or finished (so a program
  // touches -- and allocates -- only as many buffers as it keeps in flight),
  // else the oldest in flight (retire waits for it)
  EpochBuf *pick = nullptr, *oldest = nullptr;
  for (EpochBuf &c : rt->ep) {
    if (c.held) continue;
    const cudaError_t qe = c.inflight ? cudaEventQuery(c.done) : cudaSuccess;
    if (c.inflight) rt->ev("query buf %d seq %llu -> %d", (int)(&c - rt->ep), (unsigned long long)c.seq, (int)qe);
    if (!c.inflight || qe != cudaErrorNotReady) {
      pick = &c;
      break;
    }
    if (!oldest || c.seq < oldest->seq) oldest = &c;
  }
  EpochBuf &e = pick ? *pick : *oldest;
  rt->ev("pick buf %d (%s) seq %llu inflight %d", (int)(&e - rt->ep), pick ? "free" : "oldest",
         (unsigned long long)e.seq, (int)e.inflight);
  if (int r = retire(rt, e)) return r;

  const size_t N = dr ? dr->N : B.items.size();
  const size_t E = dr ? dr->E : B.edges.size();
  const bool big = !dr && N >= kParallelPack && rt->pool->size() > 1;
  const int P = big ? rt->pool->size() : 1;

  // work-unit size from the epoch's total elements (sampled for huge epochs;
  // exact for a direct round)
  uint64_t tot_elems = 0, tot_work = 0;
  if (dr) {
    tot_elems = dr->elems;
    tot_work = dr->work;
  } else {
    const size_t stride = std::max<size_t>(1, N / 4096);
    uint64_t sampled = 0, cnt = 0, sampled_work = 0;
    for (size_t i = 0; i < N; i += stride, ++cnt) {
      sampled += B.items[i].n;
      sampled_work += B.items[i].n * std::max<uint32_t>(1, B.items[i].kind == K_SCAL ? B.items[i].k : 1);
    }
    tot_elems = sampled / cnt * N;
    tot_work = sampled_work / cnt * N;
  }
  uint64_t est = tot_elems;
  // a stream launch's sub-epoch: units sized for the whole run (the launch
  // has no per-round tail to balance), equal in every sub-epoch
  if ((rt->sl.want || rt->sl.active) && rt->sl.cur_tasks) est = est * rt->sl.run_tasks / rt->sl.cur_tasks;
  uint64_t CE = chunk_elems_for(rt, est);
  // the last sub-epoch of a stream launch ends the launch: smaller units there
  // shorten its tail (BT_TAIL_SPLIT = divisor, experiments)
  static const uint64_t tail_split = getenv("BT_TAIL_SPLIT") ? strtoull(getenv("BT_TAIL_SPLIT"), nullptr, 10) : 1;
  if (rt->sl.active && rt->sl.next + 1 == rt->sl.nsub && tail_split > 1 && !rt->cfg.chunk_bytes)
    CE = std::max<uint64_t>(kMinChunkElems, CE / tail_split) / 8 * 8;
  // a DAG's ready width can be far below the item count (C3: ~16 ready 4 MiB
  // tasks): smaller units keep all SMs busy (measured: 64 KiB units 14.6 ms
  // vs 256 KiB 17.2 ms on C3, tools/c3_chunks.py)
  if (E > 0 && !rt->cfg.chunk_bytes) CE = std::min(CE, kDagChunkElems);

  // Pass A (per range): units, initially ready units, successors, factors
  // (a SCAL item whose factor list equals the previous item's reuses it).
  struct RangeAcc {
    uint64_t units = 0, ready = 0, succ = 0, fac = 0, esc = 0, needc = 0, single = 0;
    uint64_t wlo = ~0ull, whi = 0, alo = ~0ull, ahi = 0;   // written / all operand byte ranges
  };
  std::vector<RangeAcc> acc(P);
  rt->cursor.resize(N);   // per item: 1 = reuses the previous item's factor list
  auto passA = [&](int p) {
    size_t lo, hi;
    range_of(N, P, p, lo, hi);
    RangeAcc a;
    const HItem *prev = nullptr;
    for (size_t i = lo; i < hi; ++i) {
      const HItem &it = B.items[i];
      const uint64_t nc = it.n <= CE ? 1 : (it.n + CE - 1) / CE;   // (no division for small items)
      a.units += nc;
      if (it.npred == 0) a.ready += nc;
      if (nc > 1 && it.npred > 1) a.needc = 1;
      a.single += it.npred == 1;
      a.succ += it.nsucc + (it.nsucc >= K_NSUCC_ESC ? 1u : 0u);   // an escaped count precedes its list
      a.esc += it.nsucc >= K_NSUCC_ESC;
      const uint64_t bytes = 4 * it.n;
      const uint64_t w = it.kind == K_SCAL ? it.x : it.y;
      a.wlo = std::min(a.wlo, w);
      a.whi = std::max(a.whi, w + bytes);
      a.alo = std::min(a.alo, it.x);
      a.ahi = std::max(a.ahi, it.x + bytes);
      if (it.kind != K_SCAL) {
        a.alo = std::min(a.alo, it.y);
        a.ahi = std::max(a.ahi, it.y + bytes);
      }
      uint32_t reuse = 0;
      if (it.kind == K_SCAL && it.k > 1) {   // k == 1: the factor travels inline (DItem::arg)
        if (prev && prev->k == it.k && memcmp(B.factors(*prev), B.factors(it), 4ull * it.k) == 0) reuse = 1;
        else a.fac += it.k;
        prev = &it;
      }
      rt->cursor[i] = reuse;
    }
    acc[p] = a;
  };
  if (dr) {   // a direct round: units from the lanes' handle runs (every chain starts ready)
    const SlotHot *hot = rt->hot.data();
    rt->par([&](int l) {
      for (size_t i = (size_t)l; i < dr->nlanes; i += (size_t)rt->pool->size()) {
        Lane &L = *dr->lanes[i];
        uint64_t u = 0, r = 0;
        for (const RunH &h : L.hr) {
          const uint64_t nc = units_of((uint32_t)hot[h.slot].nx, CE);
          u += nc * h.items;
          r += nc;
        }
        L.d_units = u;
        L.d_ready = r;
      }
    });
    RangeAcc a;
    for (size_t i = 0; i < dr->nlanes; ++i) {
      dr->lanes[i]->qbase = a.ready;
      a.units += dr->lanes[i]->d_units;
      a.ready += dr->lanes[i]->d_ready;
    }
    a.succ = E;
    a.fac = dr->F;
    acc[0] = a;
  } else if (big) {
    rt->par(passA);
  } else {
    passA(0);
  }
  const double tA = now_ms();
  std::vector<RangeAcc> base(P);
  RangeAcc tot;
  for (int p = 0; p < P; ++p) {
    base[p] = tot;
    tot.units += acc[p].units;
    tot.ready += acc[p].ready;
    tot.succ += acc[p].succ;
    tot.esc += acc[p].esc;
    tot.needc |= acc[p].needc;
    tot.single += acc[p].single;
    tot.fac += acc[p].fac;
    tot.wlo = std::min(tot.wlo, acc[p].wlo);
    tot.whi = std::max(tot.whi, acc[p].whi);
    tot.alo = std::min(tot.alo, acc[p].alo);
    tot.ahi = std::max(tot.ahi, acc[p].ahi);
  }
  const uint64_t U = tot.units, U0 = tot.ready, F = tot.fac;
  const bool traced = (rt->cfg.flags & BT_FLAG_TIMESTAMPS) != 0;
  if (tot.succ != E + tot.esc) return fail(rt, -EIO, "internal: successor count mismatch");
  const uint64_t SL = tot.succ;   // successor-list words (edges + escaped counts)

  // scheduler variant ("Persistent scheduler kernels")
  static const char *kv = getenv("BT_KERNEL");   // "sw" / "rw" / "wq": experiments only
  // work per unit = elements x chained multiplies
  const uint64_t avg_work = tot_work / std::max<uint64_t>(1, U);
  // units of at most 16 KiB: one warp per unit ("wq", many units in flight)
  const uint64_t avg_elems = tot_elems / std::max<uint64_t>(1, U);
  // ... when the epoch is wide: a narrow one (few initially ready units, e.g.
  // a 1-wide dependency chain) is latency-bound, and the CTA-wide "rw" kernel
  // runs chains in its slots with the shortest dependency latency
  const bool wide = U0 * 4 >= (uint64_t)rt->grid_wq * 8;
  // units above 16 KiB: CTA-wide bodies with one scheduler warp ("sw"; DAG
  // epochs: the rule below); epochs of short chains (average k below the
  // FP32/HBM ridge) are HBM-bound and use the instance whose bodies prefetch
  // the next step's data
  const bool prefetch = avg_work < kPrefetchBelowK * avg_elems;
  int kernel = avg_elems <= kWarpUnitMax ? (wide && rt->grid_wq > 0 ? 2 : 1) : prefetch ? 3 : 0;
  // DAG epochs other than chains (fewer than half the items have a single
  // predecessor; tools/kernel_matrix.py, profiles/r02_kernel_matrix.jsonl):
  // "rw" when every slot of every CTA has a unit from the start (C3 with 4 MiB
  // buffers, 1,792 initially ready units: 12.6 vs 13.5 ms on "sw"; a 100k-task
  // DAG of 4 KiB buffers: 1.20 vs 1.36 ms, "wq" 2.1), else "sw" at any unit
  // size (C3 with 4 KiB - 1 MiB buffers, ~30 initially ready, 15 %
  // single-predecessor items: 3.25 vs 4.3 ms at 16 KiB -- "rw" holds up to
  // four ready units per CTA while other CTAs idle).  Chains keep the rule
  // above: "rw" runs narrow ones in its slots (3-5x faster than "sw" at 1 to
  // 256 chains of 4 KiB), "wq" wide ones (C4: 1.4 vs 2.5 ms on "rw"), "sw"
  // large units (C2 unfused: 0.25 vs 0.28 ms on "rw").
  if (E > 0 && !dr && tot.single * 2 < N)
    kernel = U0 >= 2ull * (uint64_t)rt->grid_max ? 1 : prefetch ? 3 : 0;
  // BT_FLAG_PRIORITY: the priority levels live in the "sw" bodies ("swp"), so
  // a runtime that asks for them keeps its DAG epochs there
  if (E > 0 && !dr && (rt->cfg.flags & BT_FLAG_PRIORITY) && kernel == 1) kernel = prefetch ? 3 : 0;
  if (kv) kernel = kv[0] == 'w' ? 2 : kv[0] == 'r' ? 1 : prefetch ? 3 : 0;
  if (rt->cfg.flags & BT_FLAG_KERNEL_SW) kernel = prefetch ? 3 : 0;
  if (rt->cfg.flags & BT_FLAG_KERNEL_RW) kernel = 1;
  if ((rt->cfg.flags & BT_FLAG_KERNEL_WQ) && rt->grid_wq > 0) kernel = 2;
  // stream launch: the run's first sub-epoch decides whether its rounds join
  // one launch ("sw" kernels only; no tracing, no host-homed write-backs)
  if (rt->sl.want) {
    rt->sl.want = false;
    rt->sl.active = (kernel == 0 || kernel == 3) && !traced && rt->caches.empty() &&
                    !(rt->cfg.flags & BT_FLAG_SYNC_EPOCH) && rt->sctl && rt->sl.nsub >= 2;
    rt->sl.next = 0;
    rt->sl.launched = false;
    rt->sl.prefetch = kernel == 3;
    rt->sl.started = rt->sl.active;
    rt->sl.defer = stream_defer();
  }
  bool sub = rt->sl.active;
  // priority ready queue (device_abi.h Bucket): DAG epochs on
  // the "sw" bodies order ready work by upward rank
  static const int prio_levels = getenv("BT_PRIO_LEVELS") ? std::max(1, std::min(kMaxBuckets, atoi(getenv("BT_PRIO_LEVELS"))))
                                                          : kMaxBuckets;
  const int NB = !dr && E > 0 && (kernel == 0 || kernel == 3) && !sub && !traced && (rt->cfg.flags & BT_FLAG_PRIORITY)
                     ? prio_levels : 0;
  // device layout: ctr | items | pending[N] | (cpending[U]) | succ | factors | unit_base[N] | buckets[NB] | queue[U] |
  // chunk_done[N] | trace
  const size_t o_ctr = 0;
  const size_t o_items = 64;
  const size_t o_pend = align_up(o_items + sizeof(DItem) * N, 16);
  const size_t o_cpend = align_up(o_pend + 4 * N, 16);   // per unit, only if some item needs it (chunk-wise)
  const size_t o_succ = align_up(o_cpend + (tot.needc ? 4 * U : 0), 16);
  const size_t o_fac = align_up(o_succ + 4 * SL, 16);
  // unit_base: the index of an item's per-unit counters / trace records; not
  // uploaded when nothing reads it (4 bytes per item: 4 MB in a 1M-item round)
  const bool need_ubase = traced || tot.needc;
  const size_t o_ubase = align_up(o_fac + 4 * F, 16);
  const size_t o_bk = align_up(o_ubase + (need_ubase ? 4 * N : 0), 32);
  const size_t o_queue = align_up(o_bk + sizeof(Bucket) * NB, 16);
  const size_t upload = o_queue + 8 * U0;
  const size_t o_cdone = align_up(o_queue + 8 * U, 16);
  const size_t o_trace = align_up(o_cdone + 4 * N, 16);
  const size_t dneed = o_trace + (traced ? 36 * U : 0);
  const size_t o_readback = align_up(upload, 64);
  const size_t o_trace_h = o_readback + 64;
  // sub-epoch of a stream launch: the whole blob through chunk_done goes up by
  // one copy (no set-up kernel), followed by its EpochArgs and the new
  // `published` count, staged after the blob: [StreamCtl header | args | count]
  const size_t o_sx_h = align_up(std::max(o_trace_h + (traced ? 36 * U : 0), o_cdone + 4 * N), 64);
  const size_t o_args_h = o_sx_h + 64;
  const size_t o_pub_h = align_up(o_args_h + sizeof(EpochArgs), 16);
  // A sub-epoch that joins a RUNNING launch must not allocate: cudaMalloc /
  // cudaHostAlloc / cudaFree are implicit synchronisation points and would
  // wait for the launch, which waits for this very publication.  Such a
  // sub-epoch closes the launch instead (the remaining sub-epochs are
  // published empty, so it ends) and runs as an ordinary epoch.
  if (sub && rt->sl.next > 0 && (e.hcap < o_pub_h + 16 || e.dcap < dneed)) {
    if (int r = close_stream(rt)) return r;
    sub = false;
  }
  const size_t hneed = sub ? o_pub_h + 16 : align_up(o_trace_h + (traced ? 36 * U : 0), 16);
  if (sub && rt->sl.next == 0) {
    // before the launch: grow every reusable epoch buffer to 1.25 x this
    // sub-epoch's needs scaled to the run's largest sub-epoch (by tasks), so
    // the later sub-epochs find room without allocating
    const double grow = 1.25 * (double)std::max(rt->sl.max_tasks, rt->sl.cur_tasks) /
                        (double)std::max<uint64_t>(1, rt->sl.cur_tasks);
    const size_t want_h = (size_t)(grow * (double)hneed) + 4096, want_d = (size_t)(grow * (double)dneed) + 4096;
    for (EpochBuf &c : rt->ep) {
      if (&c == &e || c.held || (c.hcap >= want_h && c.dcap >= want_d)) continue;
      if (c.inflight && cudaEventQuery(c.done) == cudaErrorNotReady) continue;
      if (int r = retire(rt, c)) return r;
      if (int r = ensure_host(rt, c, want_h)) return r;
      if (int r = ensure_dev(rt, c, want_d)) return r;
    }
  }
  if (int r = ensure_host(rt, e, hneed)) return r;
  if (int r = ensure_dev(rt, e, dneed)) return r;

  char *h = e.hblob;
  Counters *ctr = reinterpret_cast<Counters *>(h + o_ctr);
  memset(ctr, 0, sizeof(Counters));
  ctr->head = 0;
  ctr->tail = U0;
  DItem *di = reinterpret_cast<DItem *>(h + o_items);
  int32_t *pend = reinterpret_cast<int32_t *>(h + o_pend);
  int32_t *cpend = tot.needc ? reinterpret_cast<int32_t *>(h + o_cpend) : nullptr;
  uint32_t *succ = reinterpret_cast<uint32_t *>(h + o_succ);
  float *fac = reinterpret_cast<float *>(h + o_fac);
  unsigned long long *q = reinterpret_cast<unsigned long long *>(h + o_queue);
  uint32_t *ubase = need_ubase ? reinterpret_cast<uint32_t *>(h + o_ubase) : nullptr;
  rt->succ_off.resize(N);

  // Pass B (per range): fill items, counters, factors, initial ready queue.
  auto passB = [&](int p) {
    size_t lo, hi;
    range_of(N, P, p, lo, hi);
    uint64_t qi = base[p].ready, so = base[p].succ, fo = base[p].fac, ub = base[p].units;
    uint32_t prev_fo = 0;
    for (size_t i = lo; i < hi; ++i) {
      const HItem &it = B.items[i];
      DItem d;   // built here, stored whole (two 16-byte stores into the upload blob)
      d.x = it.x;
      d.y = it.y;
      d.n = (uint32_t)it.n;
      d.meta = make_meta(it.kind, it.npred == 1, it.k, it.nsucc, it.item_deps, it.n <= CE);
      if (it.kind == K_SCAL && it.k == 1) {
        memcpy(&d.arg, B.factors(it), 4);
      } else if (it.kind == K_SCAL) {
        if (!rt->cursor[i]) {
          memcpy(fac + fo, B.factors(it), 4ull * it.k);
          prev_fo = (uint32_t)fo;
          fo += it.k;
        }
        d.arg = prev_fo;
      } else {
        d.arg = it.arg;
      }
      const uint64_t nc = it.n <= CE ? 1 : (it.n + CE - 1) / CE;   // (no division for small items)
      if (ubase) ubase[i] = (uint32_t)ub;
      d.succ = (uint32_t)so;
      if (it.nsucc >= K_NSUCC_ESC) {   // the count in front of the list
        succ[so] = it.nsucc;
        ++so;
      }
      rt->succ_off[i] = (uint32_t)so;
      so += it.nsucc;
      pend[i] = (int32_t)it.npred;
      if (cpend && nc > 1)   // every chunk waits for every predecessor (chunk-wise ones release it alone)
        for (uint64_t c = 0; c < nc; ++c) cpend[ub + c] = (int32_t)it.npred;
      ub += nc;
      di[i] = d;
      if (it.npred == 0)
        for (uint64_t c = 0; c < nc; ++c) q[qi++] = ((unsigned long long)i << 32) | c;
    }
  };
  if (dr) {
    // direct round: the lanes write their descriptors and initially ready
    // units (every chain's first item) in parallel
    const SlotHot *hot = rt->hot.data();
    rt->par([&](int l) {
      for (size_t i = (size_t)l; i < dr->nlanes; i += (size_t)rt->pool->size())
        B.lane_write(
            *dr->lanes[i], CE, fac, q,
            [hot](uint32_t sl) { return std::pair<uint64_t, uint64_t>(reinterpret_cast<uint64_t>(hot[sl].dptr), hot[sl].nx); },
            [di](uint32_t id2) -> DItem & { return di[id2]; });
    });
  } else if (big) {
    rt->par(passB);
  } else {
    passB(0);
  }
  const double tB = now_ms();
  // CSR scatter (successor order within a list: edge creation order when
  // sequential; any order is valid).  An item with a single successor holds
  // the successor's id itself in DItem::succ_off (one dependent load less on
  // the device's release path: chains).
  if (dr) {
    // chains only: every successor is stored inline (lane_write)
  } else if (big) {
    uint32_t *cur = rt->succ_off.data();
    rt->par([&](int p) {
      size_t lo, hi;
      range_of(E, P, p, lo, hi);
      for (size_t j = lo; j < hi; ++j) {
        const uint64_t ed = B.edges[j];
        const uint32_t src = (uint32_t)(ed >> 32);
        if (di[src].nsucc_field() == 1) {
          di[src].succ = (uint32_t)ed;
          continue;
        }
        const uint32_t pos = __atomic_fetch_add(&cur[src], 1u, __ATOMIC_RELAXED);
        succ[pos] = (uint32_t)ed;
      }
    });
  } else {
    for (uint64_t ed : B.edges) {
      const uint32_t src = (uint32_t)(ed >> 32);
      if (di[src].nsucc_field() == 1) di[src].succ = (uint32_t)ed;
      else succ[rt->succ_off[src]++] = (uint32_t)ed;
    }
  }

  // priority levels: upward rank = the item's bytes plus the largest rank of
  // its successors (the longest remaining path, in HBM bytes; HEFT's rank_u on
  // identical processors), computed in reverse item order
  // (items are numbered in a topological order: every edge goes from a lower
  // to a higher id, checked); uniform levels over [0, max rank]
  int nb_used = 0;
  if (NB > 0) {
    bool topo = true;
    std::vector<uint64_t> rank(N);
    uint64_t maxr = 0;
    for (size_t i = N; i-- > 0 && topo;) {
      const DItem &it = di[i];
      const uint32_t kd = it.kind();
      uint64_t best = 0;
      const uint32_t f = it.nsucc_field();
      const uint32_t ns = f == K_NSUCC_ESC ? succ[it.succ] : f, off = f == K_NSUCC_ESC ? it.succ + 1 : it.succ;
      for (uint32_t j = 0; j < ns; ++j) {
        const uint32_t sj = ns == 1 ? off : succ[off + j];
        if (sj <= i || sj >= N) {
          topo = false;
          break;
        }
        best = std::max(best, rank[sj]);
      }
      rank[i] = best + it.n * (kd == K_AXPY ? 12u : 8u);
      maxr = std::max(maxr, rank[i]);
    }
    if (topo) {
      nb_used = NB;
      Bucket *bkh = reinterpret_cast<Bucket *>(h + o_bk);
      uint64_t tot[kMaxBuckets] = {}, rdy[kMaxBuckets] = {};
      for (size_t i = 0; i < N; ++i) {
        const uint32_t l = (uint32_t)std::min<uint64_t>(NB - 1, (unsigned __int128)rank[i] * NB / (maxr + 1));
        di[i].meta |= l << K_LEVEL_SHIFT;
        const uint32_t nci = units_of(di[i].n, CE);
        tot[l] += nci;
        if (B.items[i].npred == 0) rdy[l] += nci;
      }
      uint64_t rb = 0, pb = 0, cur[kMaxBuckets];
      for (int l = 0; l < NB; ++l) {
        bkh[l] = Bucket{0, rdy[l], (uint32_t)tot[l], (uint32_t)rdy[l], (uint32_t)rb, (uint32_t)pb};
        cur[l] = rb;
        rb += rdy[l];
        pb += tot[l] - rdy[l];
      }
      for (size_t i = 0; i < N; ++i)   // the initially ready units, grouped by level
        if (B.items[i].npred == 0) {
          const uint32_t l = (di[i].meta >> K_LEVEL_SHIFT) & K_LEVEL_MASK;
          const uint32_t nci = units_of(di[i].n, CE);
          for (uint32_t c = 0; c < nci; ++c) q[cur[l]++] = ((unsigned long long)i << 32) | c;
        }
    }
  }
  rt->stats.prio_epochs += nb_used > 0;

  char *d = e.dblob;
  const double tC = now_ms();
  if (!e.hctr) {
    CUDA_TRY(rt, cudaHostAlloc((void **)&e.hctr, sizeof(Counters), cudaHostAllocMapped | cudaHostAllocPortable));
    CUDA_TRY(rt, cudaHostGetDevicePointer((void **)&e.hctr_dev, e.hctr, 0));
  }
  memset(e.hctr, 0, sizeof(Counters));
  EpochArgs a{};
  a.items = reinterpret_cast<const DItem *>(d + o_items);
  a.pending = reinterpret_cast<int32_t *>(d + o_pend);
  a.cpending = tot.needc ? reinterpret_cast<int32_t *>(d + o_cpend) : nullptr;
  a.chunk_done = reinterpret_cast<uint32_t *>(d + o_cdone);
  a.succ = reinterpret_cast<const uint32_t *>(d + o_succ);
  a.factors = reinterpret_cast<const float *>(d + o_fac);
  a.queue = reinterpret_cast<unsigned long long *>(d + o_queue);
  a.ctr = reinterpret_cast<Counters *>(d + o_ctr);
  a.host_ctr = e.hctr_dev;
  a.trace = traced ? reinterpret_cast<unsigned long long *>(d + o_trace) : nullptr;
  a.trace_item = traced ? reinterpret_cast<uint32_t *>(d + o_trace + 32 * U) : nullptr;
  a.unit_base = need_ubase ? reinterpret_cast<const uint32_t *>(d + o_ubase) : nullptr;
  a.bk = nb_used ? reinterpret_cast<Bucket *>(d + o_bk) : nullptr;
  a.nbuckets = (uint32_t)nb_used;
  a.nready = (uint32_t)U0;
  a.total_units = U;
  a.chunk_elems = CE;
  a.watchdog_ns = kWatchdogNs;
  a.nitems = (uint32_t)N;
  a.stream_abort = sub ? &rt->sctl->abort : nullptr;
  auto account = [&]() {
    e.inflight = true;
    e.seq = ++rt->ep_seq;
    e.units = U;
    e.traced = traced;
    e.trace_off_h = o_trace_h;
    rt->stats.items += N;
    rt->stats.edges += E;
    rt->stats.units += U;
    rt->stats.epochs += 1;
    rt->stats.upload_bytes += upload;
    rt->stats.fused_tasks += dr ? dr->tasks - N : B.fused;
    B.next_epoch();
    rt->stats.host_build_ms += now_ms() - t0;
  };
  if (sub) {
    // ---- sub-epoch r of the run's stream launch (device_abi.h StreamCtl) ----
    const unsigned r = rt->sl.next;
    rt->ev("sub %u/%u buf %d seq %llu U %llu U0 %llu N %zu", r, rt->sl.nsub, (int)(&e - rt->ep),
           (unsigned long long)rt->ep_seq + 1, (unsigned long long)U, (unsigned long long)U0, N);
    cudaStream_t ls = rt->rstream[0];                    // the launch
    cudaStream_t up = r == 0 ? ls : rt->rstream[1];      // this sub-epoch's copies
    if (!rt->span_open) {
      CUDA_TRY(rt, cudaEventRecord(rt->span_start, ls));
      rt->span_open = true;
    }
    // tests: a host that publishes late (BT_DEBUG_PUBLISH_DELAY_US before every
    // sub-epoch after the first) makes the running launch close and resume
    static const long pub_delay_us = getenv("BT_DEBUG_PUBLISH_DELAY_US") ? atol(getenv("BT_DEBUG_PUBLISH_DELAY_US")) : 0;
    if (r > 0 && pub_delay_us > 0) std::this_thread::sleep_for(std::chrono::microseconds(pub_delay_us));
    // the launch is already running (r > 0): no set-up kernel, so the queue's
    // unpublished slots read EMPTY and the chunk counters zero in the blob
    for (uint64_t i = U0; i < U; ++i) q[i] = Q_EMPTY;
    memset(h + o_cdone, 0, 4 * N);
    memcpy(h + o_args_h, &a, sizeof a);
    *reinterpret_cast<uint32_t *>(h + o_pub_h) = r + 1;
    if (r == 0) {   // launch-wide header: ticket = published = abort = exited = 0, nsub
      memset(h + o_sx_h, 0, 64);
      *reinterpret_cast<uint32_t *>(h + o_sx_h + offsetof(StreamCtl, nsub)) = rt->sl.nsub;
      CUDA_TRY(rt, cudaMemcpyAsync(rt->sctl, h + o_sx_h, 64, cudaMemcpyHostToDevice, up));
    }
    CUDA_TRY(rt, cudaMemcpyAsync(d, h, o_cdone + 4 * N, cudaMemcpyHostToDevice, up));
    CUDA_TRY(rt, cudaMemcpyAsync(&rt->sctl->subs[r], h + o_args_h, sizeof(EpochArgs), cudaMemcpyHostToDevice, up));
    CUDA_TRY(rt, cudaMemcpyAsync(&rt->sctl->published, h + o_pub_h, 4, cudaMemcpyHostToDevice, up));
    if (r == 0) {   // later sub-epochs' copies follow the header reset
      CUDA_TRY(rt, cudaEventRecord(rt->ev_pub0, ls));
      CUDA_TRY(rt, cudaStreamWaitEvent(rt->rstream[1], rt->ev_pub0, 0));
    }
    rt->sl.bufs[r] = &e;
    if (r == 0 && !rt->sl.defer)
      if (int rc = enqueue_stream_launch(rt)) return rc;
    // held (not reusable) until the run's last launch is enqueued
    // (finish_stream_run records its done event after it)
    e.held = true;
    e.timed = r == 0;
    const bool last = ++rt->sl.next == rt->sl.nsub;
    if (last) rt->sl.active = false;
    account();
    if (last)
      if (int rc = finish_stream_run(rt)) return rc;
    static const bool dbg_t = getenv("BT_DEBUG_TIMING") != nullptr;
    if (dbg_t)
      fprintf(stderr, "flush sub %u N=%zu U=%llu: passA %.3f passB %.3f csr %.3f copies+launch %.3f ms\n", r, N,
              (unsigned long long)U, tA - t0, tB - tA, tC - tB, now_ms() - tC);
    return 0;
  }
  e.timed = true;
  // a tiny epoch of independent items: one direct launch, no blob (DirectArgs)
  static const bool no_direct = getenv("BT_NO_DIRECT") != nullptr;   // comparisons
  uint64_t max_n = 0;
  bool direct = !dr && E == 0 && N <= (size_t)kDirectItems && !traced && !no_direct &&
                !(rt->cfg.flags & (BT_FLAG_KERNEL_SW | BT_FLAG_KERNEL_RW | BT_FLAG_KERNEL_WQ));
  // distinct factor lists (consecutive equal lists shared, as in pass B)
  uint64_t dfac = 0;
  for (size_t i = 0; direct && i < N; ++i) {
    const HItem &it = B.items[i];
    max_n = std::max<uint64_t>(max_n, it.n);
    if (it.kind == K_SCAL && (it.k == 1 || !rt->cursor[i])) dfac += it.k;
  }
  direct = direct && max_n > 0 && dfac <= (uint64_t)kDirectFactors;
  if (!rt->span_open) {
    CUDA_TRY(rt, cudaEventRecord(rt->span_start, stream));
    rt->span_open = true;
  }
  // the set-up kernel copies whole 16-byte words: the word holding the last
  // initially-ready unit may extend into queue[U0], which must read EMPTY
  // (it also writes EMPTY there; both writes agree)
  if (U > U0) q[U0] = Q_EMPTY;
  // small blobs (and any blob while chunked uploads occupy the copy engine)
  // are pulled by the set-up kernel from mapped memory; large ones by a memcpy
  bool uploads_pending = false;
  for (auto &kv2 : rt->caches) uploads_pending |= !kv2.second.uploads.empty();
  const bool sm_copy = uploads_pending || upload <= kStageBelow;
  if (!direct) {
    if (!sm_copy) CUDA_TRY(rt, cudaMemcpyAsync(d, h, upload, cudaMemcpyHostToDevice, stream));
    rt->stats.kernel_launches += 2;   // the set-up kernel below and the scheduler kernel
    CUDA_TRY(rt, launch_stage(d, sm_copy ? e.hblob_dev : nullptr, upload,
                              reinterpret_cast<unsigned long long *>(d + o_queue) + U0, U - U0,
                              reinterpret_cast<uint32_t *>(d + o_cdone), N, stream));
  } else {
    rt->stats.kernel_launches += 1;
  }

  const int grid = (int)std::min<uint64_t>((uint64_t)rt->grid_max, U);

  // host-homed data: upload what this epoch reads first, skip write-only
  // first accesses, collect what it writes
  if (!rt->caches.empty())
    if (int r = epoch_coherence(rt)) return r;
  // host-homed data this epoch touches must have arrived (chunked uploads)
  for (auto &kv2 : rt->caches) {
    RootCache &c = kv2.second;
    if (c.uploads.empty() || tot.ahi <= c.dlo || tot.alo >= c.dhi) continue;
    for (const UploadChunk &u : c.uploads)
      if (u.lo < tot.ahi && tot.alo < u.hi) CUDA_TRY(rt, cudaStreamWaitEvent(stream, u.ev, 0));
  }
  CUDA_TRY(rt, cudaEventRecord(e.start, stream));
  const int kgrid = kernel == 2 ? (int)std::min<uint64_t>((uint64_t)rt->grid_wq, (U + 7) / 8) : grid;
  rt->stats.grid = (uint32_t)kgrid;
  rt->stats.sched_launches += 1;
  rt->stats.block = kernel == 2 ? (uint32_t)rt->block_wq : (uint32_t)rt->block;
  rt->ev("epoch buf %d seq %llu U %llu kernel %d grid %d stream %p direct %d", (int)(&e - rt->ep),
         (unsigned long long)rt->ep_seq + 1, (unsigned long long)U, kernel, kgrid, (void *)stream, (int)direct);
  if (direct) {
    DirectArgs da{};
    da.chunk = 16384;
    uint32_t fo = 0, prev_fo = 0, ng = 0;
    for (size_t i = 0; i < N; ++i) {
      const HItem &it = B.items[i];
      DirectItem di2{};
      di2.x = it.x;
      di2.y = it.y;
      di2.n = it.n;
      di2.kind = it.kind;
      di2.k = it.k;
      di2.first = (uint32_t)i;
      if (it.kind == K_SCAL) {
        if (it.k == 1 || !rt->cursor[i]) {   // rt->cursor[i] == 1: same list as the previous k > 1 item
          if (it.k == 1 && ng && da.items[ng - 1].kind == K_SCAL && da.items[ng - 1].k == 1 &&
              memcmp(&da.factors[da.items[ng - 1].arg], B.factors(it), 4) == 0) {
            di2.arg = da.items[ng - 1].arg;   // the same single factor: joinable with the previous group
          } else {
            memcpy(&da.factors[fo], B.factors(it), 4ull * it.k);
            if (it.k > 1) prev_fo = fo;
            di2.arg = fo;
            fo += it.k;
          }
        } else {
          di2.arg = prev_fo;
        }
      } else {
        di2.arg = it.arg;
      }
      // join the previous group: same kind, length, factors / scalar, operands
      // one constant stride on (the first join fixes the stride)
      if (ng) {
        DirectItem &g = da.items[ng - 1];
        const uint64_t cnt = i - g.first;   // items in g so far
        const uint64_t dx = it.x - g.x, dy = it.y - g.y;
        const bool same = g.kind == di2.kind && g.k == di2.k && g.arg == di2.arg && g.n == di2.n;
        const bool stride_ok = dx % cnt == 0 && (cnt == 1 || dx / cnt == g.stride) &&
                               (it.kind == K_SCAL || dy == dx) && it.x > g.x;
        if (same && stride_ok) {
          g.stride = dx / cnt;
          continue;
        }
      }
      da.items[ng++] = di2;
    }
    da.nitems = ng;
    rt->stats.grid = (uint32_t)((max_n + da.chunk - 1) / da.chunk);
    rt->stats.block = 256;
    CUDA_TRY(rt, launch_direct(da, (unsigned)((max_n + da.chunk - 1) / da.chunk), (unsigned)N, stream));
  } else {
    CUDA_TRY(rt, launch_epoch(a, kgrid, stream, kernel));
  }
  CUDA_TRY(rt, cudaEventRecord(e.end, stream));
  // write-back of host-homed ranges written for the first time since registration
  // (the parts written before are marked dirty instead: copied back at
  // acquire / unregister, after everything that writes them)
  bool wb_waited = false;
  for (auto &kv2 : rt->caches) {
    RootCache &c = kv2.second;
    for (const auto &w : c.ewrite.m) {
      std::vector<std::pair<uint64_t, uint64_t>> old;
      c.written.pieces(w.first, w.second, old, false);
      for (const auto &o : old) c.dirty.add(o.first, o.second);
      uint64_t a = w.first;
      old.emplace_back(w.second, w.second);
      for (const auto &o : old) {   // the gaps between old pieces: first writes
        if (a < o.first) {
          if (!wb_waited) {
            CUDA_TRY(rt, cudaStreamWaitEvent(rt->d2h, e.end, 0));
            wb_waited = true;
          }
          char *host = static_cast<char *>(rt->slots[kv2.first].hptr) + (a - c.dlo);
          CUDA_TRY(rt, cudaMemcpyAsync(host, reinterpret_cast<const void *>(a), o.first - a, cudaMemcpyDeviceToHost,
                                       rt->d2h));
          rt->stats.d2h_data_bytes += o.first - a;
          c.wb = true;
        }
        a = std::max(a, o.second);
      }
      c.written.add(w.first, w.second);
    }
    c.ewrite.m.clear();
  }
  if (traced) CUDA_TRY(rt, cudaMemcpyAsync(h + o_trace_h, d + o_trace, 36 * U, cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(rt, cudaEventRecord(e.done, stream));
  account();
  if (direct) e.units = 0;   // no completion counters: retire checks done == 0
  static const bool dbg = getenv("BT_DEBUG_TIMING") != nullptr;
  if (dbg)
    fprintf(stderr, "flush_epoch N=%zu E=%zu U=%llu upload=%zu B: passA %.3f passB %.3f csr %.3f launch %.3f ms\n", N, E,
            (unsigned long long)U, upload, tA - t0, tB - tA, tC - tB, now_ms() - tC);
  if (rt->cfg.flags & BT_FLAG_SYNC_EPOCH) return retire(rt, e);
  return 0;
}

double g_wait_return_ms = 0;   // BT_DEBUG_TIMING: host time the last wait_all returned

int wait_all(bt_runtime *rt) {
  static const bool dbg = getenv("BT_DEBUG_TIMING") != nullptr;
  const double w0 = dbg ? now_ms() : 0;
  if (int r = flush_epoch(rt)) return r;
  if (rt->span_open) CUDA_TRY(rt, cudaEventRecord(rt->span_end, rt->stream));
  // retire in launch order (older first)
  for (;;) {
    EpochBuf *next = nullptr;
    for (auto &e : rt->ep)
      if (e.inflight && (!next || e.seq < next->seq)) next = &e;
    if (!next) break;
    if (int r = retire(rt, *next)) return r;
  }
  const double w1 = dbg ? now_ms() : 0;
  CUDA_TRY(rt, cudaStreamSynchronize(rt->stream));
  const double w2 = dbg ? now_ms() : 0;
  for (auto &kv2 : rt->caches) {   // every epoch that needed an upload chunk has run
    for (const UploadChunk &u : kv2.second.uploads) {
      CUDA_TRY(rt, cudaEventSynchronize(u.ev));
      rt->put_event(u.ev);
    }
    kv2.second.uploads.clear();
  }
  if (rt->span_open) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, rt->span_start, rt->span_end) == cudaSuccess) rt->stats.device_span_ms += ms;
    rt->span_open = false;
  }
  if (dbg) {
    g_wait_return_ms = now_ms();
    fprintf(stderr, "wait_all: retire %.3f ms, stream sync %.3f ms, rest %.3f ms\n", w1 - w0, w2 - w1,
            g_wait_return_ms - w2);
  }
  return 0;
}

}  // namespace

// ================================================================ C ABI ====

extern "C" {

int bt_config_init(bt_config *cfg) {
  if (!cfg) return -EINVAL;
  memset(cfg, 0, sizeof *cfg);
  cfg->abi_version = BT_ABI_VERSION;
  cfg->device = -1;
  cfg->rank = 0;
  cfg->nranks = 1;
  return 0;
}

int bt_init(const bt_config *cfg_in, bt_runtime **out) {
  if (!out) return -EINVAL;
  *out = nullptr;
  bt_config cfg;
  if (cfg_in) cfg = *cfg_in;
  else bt_config_init(&cfg);
  if (cfg.abi_version != BT_ABI_VERSION) return -EINVAL;
  if (cfg.nranks < 1 || cfg.rank < 0 || cfg.rank >= cfg.nranks) return -EINVAL;
  if (cfg.max_fused == 0) cfg.max_fused = kDefaultMaxFused;
  if (cfg.max_fused > (uint32_t)max_factors()) return -EINVAL;
  if (cfg.chunk_bytes != 0 && cfg.chunk_bytes < 32) return -EINVAL;
  if (cfg.host_threads < 0) return -EINVAL;
  if (cfg.parallel_min == 0) cfg.parallel_min = kDefaultParallelMin;
  if (cfg.pipeline_rounds == 0) cfg.pipeline_rounds = kDefaultRounds;
  if (cfg.pipeline_rounds < 1 || cfg.pipeline_rounds > kEpochRing - 2) return -EINVAL;
  if (__builtin_popcount(cfg.flags & (BT_FLAG_KERNEL_SW | BT_FLAG_KERNEL_RW | BT_FLAG_KERNEL_WQ)) > 1) return -EINVAL;
  if (cfg.pipeline_min == 0) cfg.pipeline_min = kDefaultPipelineMin;

  bt_runtime *rt = new (std::nothrow) bt_runtime();
  if (!rt) return -ENOMEM;
  rt->cfg = cfg;
  rt->host_only = (cfg.flags & BT_FLAG_HOST_ONLY) != 0;
  rt->builder.fusion = (cfg.flags & BT_FLAG_NO_FUSION) == 0;
  rt->builder.max_fused = cfg.max_fused;
  rt->builder.record_tasks = rt->host_only && getenv("BT_HOST_NORECORD") == nullptr;   // (env: host benchmarks)
  int threads = cfg.host_threads;
  if (threads == 0) {
    // leave two cores to the CUDA driver / caller threads (measured: 14 of 16 beats 16 of 16)
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    threads = (int)std::min<unsigned>(16, hw > 4 ? hw - 2 : hw);
  }
  rt->pool.reset(new Pool(threads));

  rt->npool = threads;
  rt->rounds_default = cfg.pipeline_rounds;
  rt->nrounds = std::max(cfg.pipeline_rounds, cfg.pipeline_rounds > 1 ? kRoundsUploading : 1);
  rt->lanes.resize((size_t)threads * rt->nrounds);                  // [(round - first round of the launch) * P + lane]
  rt->runs.resize((size_t)threads * threads * rt->nrounds);         // [chunk][round * P + lane]
  rt->run_tasks.assign(rt->runs.size(), 0);

  if (!rt->host_only) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      delete rt;
      return -ENODEV;
    }
    int dev = cfg.device;
    if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    if (dev >= ndev || cudaSetDevice(dev) != cudaSuccess) {
      cudaGetLastError();
      delete rt;
      return -ENODEV;
    }
    rt->device = dev;
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess || p.major < 10) {
      cudaGetLastError();
      delete rt;
      return -ENODEV;   // sm_100a kernels only
    }
    rt->sms = p.multiProcessorCount;
    int occ = 0, block = 0;
    if (scheduler_occupancy(&occ, &block) != cudaSuccess || occ < 1) {
      cudaGetLastError();
      delete rt;
      return -ENODEV;
    }
    if (cfg.ctas_per_sm > 0) occ = std::min(occ, cfg.ctas_per_sm);
    rt->grid_max = occ * rt->sms;
    rt->block = block;
    rt->stats.block = (uint32_t)block;
    int occ_wq = 0, block_wq = 0;
    if (scheduler_occupancy_wq(&occ_wq, &block_wq) != cudaSuccess || occ_wq < 1) {
      cudaGetLastError();
      occ_wq = 0;
    }
    if (cfg.ctas_per_sm > 0) occ_wq = std::min(occ_wq, cfg.ctas_per_sm);
    rt->grid_wq = occ_wq * rt->sms;
    rt->block_wq = block_wq;
    if (cfg.stream) {
      rt->stream = (cudaStream_t)cfg.stream;
    } else {
      if (cudaStreamCreateWithFlags(&rt->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete rt;
        return -ENOMEM;
      }
      rt->own_stream = true;
    }
    for (auto &e : rt->ep) {
      if (cudaEventCreate(&e.start) != cudaSuccess || cudaEventCreate(&e.end) != cudaSuccess ||
          cudaEventCreate(&e.done) != cudaSuccess) {
        delete rt;
        return -ENOMEM;
      }
    }
    if (cudaEventCreate(&rt->span_start) != cudaSuccess || cudaEventCreate(&rt->span_end) != cudaSuccess ||
        cudaEventCreateWithFlags(&rt->ev_fork, cudaEventDisableTiming) != cudaSuccess) {
      delete rt;
      return -ENOMEM;
    }
    if (cudaStreamCreateWithFlags(&rt->h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&rt->d2h, cudaStreamNonBlocking) != cudaSuccess) {
      delete rt;
      return -ENOMEM;
    }
    for (int i = 0; i < 2; ++i)
      if (cudaStreamCreateWithFlags(&rt->rstream[i], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&rt->ev_round[i], cudaEventDisableTiming) != cudaSuccess) {
        delete rt;
        return -ENOMEM;
      }
    if (!(cfg.flags & BT_FLAG_NO_STREAM) && rt->grid_max <= kMaxStreamGrid &&
        (cudaMalloc((void **)&rt->sctl, sizeof(StreamCtl)) != cudaSuccess ||
         cudaEventCreateWithFlags(&rt->ev_pub0, cudaEventDisableTiming) != cudaSuccess ||
         cudaHostAlloc((void **)&rt->close_h, 4 * kMaxSubs + sizeof(EpochArgs), cudaHostAllocPortable) !=
             cudaSuccess)) {
      cudaGetLastError();
      if (rt->sctl) cudaFree(rt->sctl);
      rt->sctl = nullptr;   // pipelined runs then launch once per round
    }
    if (rt->sctl) {
      for (unsigned q = 0; q < (unsigned)kMaxSubs; ++q) reinterpret_cast<unsigned *>(rt->close_h)[q] = q + 1;
      memset(rt->close_h + 4 * kMaxSubs, 0, sizeof(EpochArgs));
    }
    // every epoch buffer's mapped completion record, allocated here: a
    // sub-epoch joining a running stream launch must not allocate (flush_epoch)
    for (auto &e : rt->ep) {
      if (cudaHostAlloc((void **)&e.hctr, sizeof(Counters), cudaHostAllocMapped | cudaHostAllocPortable) !=
              cudaSuccess ||
          cudaHostGetDevicePointer((void **)&e.hctr_dev, e.hctr, 0) != cudaSuccess) {
        delete rt;
        return -ENOMEM;
      }
    }
    // keep freed replicas in the pool (register/unregister loops reuse them)
    cudaMemPool_t mp;
    if (cudaDeviceGetDefaultMemPool(&mp, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  } else {
    rt->grid_max = 148 * 4;   // only used by the chunk policy
  }
  *out = rt;
  return 0;
}

int bt_shutdown(bt_runtime *rt) {
  if (!rt) return -EINVAL;
  if (rt->live_roots) return fail(rt, -EBUSY, "%u handles still registered", rt->live_roots);
  if (!rt->host_only) {
    cudaSetDevice(rt->device);
    if (!rt->poisoned) wait_all(rt);
    cudaStreamSynchronize(rt->stream);
    for (auto &e : rt->ep) {
      if (e.hblob) cudaFreeHost(e.hblob);
      if (e.hctr) cudaFreeHost(e.hctr);
      if (e.dblob) cudaFree(e.dblob);
      if (e.start) cudaEventDestroy(e.start);
      if (e.end) cudaEventDestroy(e.end);
      if (e.done) cudaEventDestroy(e.done);
    }
    for (int i = 0; i < 2; ++i) {
      if (rt->rstream[i]) cudaStreamDestroy(rt->rstream[i]);
      if (rt->ev_round[i]) cudaEventDestroy(rt->ev_round[i]);
    }
    if (rt->ev_fork) cudaEventDestroy(rt->ev_fork);
    if (rt->ev_pub0) cudaEventDestroy(rt->ev_pub0);
    if (rt->sctl) cudaFree(rt->sctl);
    if (rt->close_h) cudaFreeHost(rt->close_h);
    for (cudaEvent_t ev : rt->ev_free) cudaEventDestroy(ev);
    for (uint32_t *g : rt->gates) cudaFreeHost(g);
    if (rt->h2d) cudaStreamDestroy(rt->h2d);
    if (rt->d2h) cudaStreamDestroy(rt->d2h);
    if (rt->span_start) cudaEventDestroy(rt->span_start);
    if (rt->span_end) cudaEventDestroy(rt->span_end);
    rt->comm.reset();
    if (rt->own_stream) cudaStreamDestroy(rt->stream);
  }
  delete rt;
  return 0;
}

int bt_vector_data_register(bt_runtime *rt, bt_handle *out, int home_node, void *ptr, size_t nx,
                            size_t elemsize) {
  if (int r = check_live(rt)) return r;
  if (!out) return fail(rt, -EINVAL, "null output handle");
  *out = 0;
  if (nx == 0 || elemsize != 4) return fail(rt, -EINVAL, "only float32 vectors (elemsize 4, nx > 0) are supported");
  if (nx > 0xFFFFFFFFull) return fail(rt, -EINVAL, "at most 2^32 - 1 elements per vector (16 GiB)");
  if (home_node != 0 && home_node != 1) return fail(rt, -EINVAL, "home_node must be 0 (host) or 1 (device)");
  if (home_node == 1 && !ptr) return fail(rt, -EINVAL, "device-homed data needs a pointer");
  if (home_node == 1 && rt->host_only) return fail(rt, -ENODEV, "host-only runtime");
  if (ptr && (reinterpret_cast<uintptr_t>(ptr) & 3u)) return fail(rt, -EINVAL, "pointer not 4-byte aligned");
  const uintptr_t lo = reinterpret_cast<uintptr_t>(ptr), hi = lo + nx * elemsize;
  if (ptr) {
    auto it = rt->ranges.upper_bound(lo);
    if (it != rt->ranges.end() && it->first < hi) return fail(rt, -EEXIST, "overlaps a registered buffer");
    if (it != rt->ranges.begin()) {
      --it;
      if (it->second.first > lo) return fail(rt, -EEXIST, "overlaps a registered buffer");
    }
  }
  if (home_node == 1) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess || at.type != cudaMemoryTypeDevice ||
        at.device != rt->device) {
      cudaGetLastError();
      return fail(rt, -EINVAL, "home_node 1 needs device memory of the runtime's GPU");
    }
  }
  float *dptr = nullptr;
  bool owns = false;
  // host-only (analysis) runtimes: the host address stands in for the replica,
  // so operand base addresses in the DAG are distinct per range (never
  // dereferenced: nothing executes)
  if (rt->host_only && ptr) dptr = static_cast<float *>(ptr);
  if (!rt->host_only && ptr) {
    cudaSetDevice(rt->device);
    if (home_node == 1) {
      dptr = static_cast<float *>(ptr);
    } else {
      // with cross-rank reads enabled the replica must be shareable (CUDA IPC
      // cannot export stream-ordered pool allocations)
      cudaError_t e = rt->comm ? cudaMalloc((void **)&dptr, nx * 4) : cudaMallocAsync((void **)&dptr, nx * 4, rt->stream);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(rt, -ENOMEM, "cannot allocate the device replica (%zu bytes)", nx * 4);
      }
      owns = true;
    }
  }
  const uint32_t s = alloc_slots(rt, 1);
  rt->key_dirty = true;
  SlotHot &sh = rt->hot[s];
  Slot &sl = rt->slots[s];
  sl.root = s;
  sh.dptr = dptr;
  sh.nx = nx;
  sl.hptr = ptr;
  sl.home_node = home_node;
  sh.rank = ptr ? rt->cfg.rank : -1;
  sl.owns_dev = owns;
  sl.ipc_alloc = owns && rt->comm;
  sl.reg_key = ++rt->reg_seq;
  if (ptr) {
    rt->ranges[lo] = {hi, s};
    rt->by_ptr[lo] = s;
  }
  if (owns) {   // host-homed replica: coherence state; the data stays on the host until first read
    RootCache &c = rt->caches[s];
    c = RootCache();
    c.dlo = reinterpret_cast<uint64_t>(dptr);
    c.dhi = c.dlo + nx * 4;
    c.pending.add(c.dlo, c.dhi);
    cudaEvent_t ev_alloc = rt->get_event();
    CUDA_TRY(rt, cudaEventRecord(ev_alloc, rt->stream));        // uploads follow the (stream-ordered) allocation
    CUDA_TRY(rt, cudaStreamWaitEvent(rt->h2d, ev_alloc, 0));
    rt->put_event(ev_alloc);
  }
  ++rt->live_roots;
  *out = make_handle(rt, s);
  return 0;
}

int bt_data_lookup(bt_runtime *rt, const void *ptr, bt_handle *out) {
  if (!rt || !out) return -EINVAL;
  *out = 0;
  auto it = rt->by_ptr.find(reinterpret_cast<uintptr_t>(ptr));
  if (it == rt->by_ptr.end()) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  *out = make_handle(rt, it->second);
  return 0;
}

int bt_data_partition(bt_runtime *rt, bt_handle h, uint32_t nparts) {
  if (int r = check_live(rt)) return r;
  ++rt->gver;
  uint32_t s = resolve(rt, h);
  if (s == NONE) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  if (rt->slots[s].nparts) return fail(rt, -EBUSY, "handle already partitioned");
  if (acquired_chain(rt, s)) return fail(rt, -EBUSY, "handle is acquired");
  if (nparts == 0 || nparts > rt->hot[s].nx) return fail(rt, -EINVAL, "bad number of parts");
  const uint32_t c0 = alloc_slots(rt, nparts);   // may reallocate the slot arrays
  rt->key_dirty = true;
  SlotHot &ph = rt->hot[s];
  Slot &p = rt->slots[s];
  const uint64_t base = ph.nx / nparts, extra = ph.nx % nparts;
  // data still arriving by chunked upload: finer rounds, so computation and
  // write-back follow the upload more closely (the e2e path is PCIe-bound)
  uint32_t rounds = (uint32_t)rt->rounds_default;
  {
    auto it = rt->caches.find(p.root);
    if (it != rt->caches.end() && (!it->second.uploads.empty() || !it->second.pending.empty()) && rounds > 1)
      rounds = (uint32_t)rt->nrounds;
  }
  for (uint32_t t = 0; t < nparts; ++t) {
    rt->key_dirty = true;
    SlotHot &ch = rt->hot[c0 + t];
    Slot &c = rt->slots[c0 + t];
    const uint64_t off = t * base + std::min<uint64_t>(t, extra);
    c.parent = s;
    c.child_index = t;
    c.root = p.root;
    c.offset = p.offset + off;
    ch.nx = base + (t < extra ? 1 : 0);
    ch.dptr = ph.dptr ? ph.dptr + off : nullptr;
    ch.rank = ph.rank;
    // pipelined rounds take contiguous quarters of the parts (so round r
    // needs only its own upload chunks and writes back one contiguous range);
    // lanes still own whole 64-slot blocks
    // device-resident data, fusion on: geometric rounds 1/16, 2/16, 4/16,
    // 9/16 of the parts, so the device starts after building 1/16 of a run;
    // each later round is built while the previous one runs (fused chains
    // make the device the slower side: C5 step 2.51 -> 2.40-2.45 ms).
    // Unfused runs are host-bound (C4: ~4 ns of build per task on 14
    // threads vs ~1 ns of device time), where a large last round would
    // leave the device the whole 9/16 after the host is done; shrinking rounds
    // (9/16 ... 1/16, round_of geo = 2) measured worse too (C4 unfused 4.9 ->
    // 6.3 ms: a 560k-item round builds slower per item): equal rounds.
    // (Parts owned by several ranks are re-dealt per rank: scal_run_parallel.)
    const int geo = rounds == 4 && geometric_rounds() && rt->builder.fusion ? 1 : 0;
    const uint32_t round = round_of(t, nparts, rounds, geo);
    p.prounds = (uint8_t)rounds;
    p.pgeo = (int8_t)geo;
    ch.grp = round * (uint32_t)rt->npool + ((c0 + t) >> 6) % (uint32_t)rt->npool;
  }
  p.nparts = nparts;
  p.first_child = c0;
  ph.flags |= F_PARTITIONED;
  rt->builder.partition_state(rt->deps[s], &rt->deps[c0], nparts);
  return 0;
}

int bt_data_get_sub_data(bt_runtime *rt, bt_handle h, uint32_t i, bt_handle *out) {
  if (!rt || !out) return -EINVAL;
  *out = 0;
  uint32_t s = resolve(rt, h);
  if (s == NONE) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  const Slot &p = rt->slots[s];
  if (!p.nparts || i >= p.nparts) return fail(rt, -EINVAL, "no part %u", i);
  *out = make_handle(rt, p.first_child + i);
  return 0;
}

int bt_data_get_children(bt_runtime *rt, bt_handle h, bt_handle *out, uint32_t nparts) {
  if (!rt || !out) return -EINVAL;
  uint32_t s = resolve(rt, h);
  if (s == NONE) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  const Slot &p = rt->slots[s];
  if (!p.nparts || nparts != p.nparts) return fail(rt, -EINVAL, "handle has %u parts, not %u", p.nparts, nparts);
  for (uint32_t i = 0; i < nparts; ++i) out[i] = make_handle(rt, p.first_child + i);
  return 0;
}

int bt_data_unpartition(bt_runtime *rt, bt_handle h) {
  if (int r = check_live(rt)) return r;
  ++rt->gver;
  uint32_t s = resolve(rt, h);
  if (s == NONE) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  Slot &p = rt->slots[s];
  if (!p.nparts) return fail(rt, -EINVAL, "handle is not partitioned");
  for (uint32_t t = 0; t < p.nparts; ++t) {
    const Slot &c = rt->slots[p.first_child + t];
    if (c.nparts) return fail(rt, -EBUSY, "part %u is itself partitioned", t);
    if (c.acquired) return fail(rt, -EBUSY, "part %u is acquired", t);
  }
  rt->builder.unpartition_state(rt->deps[s], &rt->deps[p.first_child], p.nparts);
  free_slots(rt, p.first_child, p.nparts);
  p.nparts = 0;
  p.first_child = NONE;
  rt->key_dirty = true;
  rt->hot[s].flags &= ~F_PARTITIONED;
  return 0;
}

int bt_data_set_rank(bt_runtime *rt, bt_handle h, int rank) {
  if (int r = check_live(rt)) return r;
  ++rt->gver;
  uint32_t s = resolve(rt, h);
  if (s == NONE) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  if (rank < 0 || rank >= rt->cfg.nranks) return fail(rt, -EINVAL, "rank %d out of range", rank);
  std::vector<uint32_t> stack{s};   // the handle and all its parts (recursively)
  while (!stack.empty()) {
    uint32_t x = stack.back();
    stack.pop_back();
    rt->key_dirty = true;
    rt->hot[x].rank = rank;
    const Slot &sl = rt->slots[x];
    for (uint32_t t = 0; t < sl.nparts; ++t) stack.push_back(sl.first_child + t);
  }
  return 0;
}

int bt_comm_init(bt_runtime *rt, const char *name) {
  if (int r = check_live(rt)) return r;
  if (rt->host_only) return fail(rt, -ENODEV, "host-only runtime: nothing executes");
  if (rt->comm) return fail(rt, -EBUSY, "bt_comm_init already called");
  if (rt->cfg.nranks < 2) return fail(rt, -EINVAL, "cross-rank reads need nranks >= 2");
  cudaSetDevice(rt->device);
  Comm *c = nullptr;
  std::string err;
  if (int r = Comm::create(name, rt->cfg.rank, rt->cfg.nranks, rt->device, &c, &err))
    return fail(rt, r, "bt_comm_init: %s", err.c_str());
  rt->comm.reset(c);
  return 0;
}

int bt_data_distribute_block(bt_runtime *rt, bt_handle h) {
  if (int r = check_live(rt)) return r;
  uint32_t s = resolve(rt, h);
  if (s == NONE) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  const Slot p = rt->slots[s];
  if (!p.nparts) return fail(rt, -EINVAL, "handle is not partitioned");
  for (uint32_t t = 0; t < p.nparts; ++t) {
    const int r = (int)(((uint64_t)t * (uint64_t)rt->cfg.nranks) / p.nparts);
    if (int e = bt_data_set_rank(rt, make_handle(rt, p.first_child + t), r)) return e;
  }
  return 0;
}

}  // extern "C"

namespace {

// Validate one operand; returns slot or a negative errno.
inline int64_t operand(bt_runtime *rt, int codelet, bt_handle h) {
  const uint32_t s = resolve(rt, h);
  if (s == NONE) {
    fail(rt, -ENOENT, "attempt to use unregistered pointer (task `%s')", codelet_name(codelet));
    return -ENOENT;
  }
  const uint32_t f = rt->hot[s].flags;
  if (f & F_PARTITIONED) return insert_fail(rt, codelet, -EBUSY, "handle is partitioned");
  if (f & F_BLOCKED) return insert_fail(rt, codelet, -EBUSY, "handle is acquired");
  return s;
}

// Order `stream` after the chunked uploads covering device bytes [lo, hi).
int wait_uploads(bt_runtime *rt, cudaStream_t stream, uint64_t lo, uint64_t hi) {
  for (auto &kv : rt->caches) {
    RootCache &c = kv.second;
    if (c.uploads.empty() || hi <= c.dlo || lo >= c.dhi) continue;
    for (const UploadChunk &u : c.uploads)
      if (u.lo < hi && lo < u.hi) CUDA_TRY(rt, cudaStreamWaitEvent(stream, u.ev, 0));
  }
  return 0;
}

// One side of a cross-rank read of slot x (comm.hpp): the owner publishes
// it for `peer` (send), the reader copies it into its own replica (recv).
// Everything submitted earlier is flushed first, so the copy is ordered after
// the owner's earlier writers and the reader's earlier readers of the replica.
int cross_rank_read(bt_runtime *rt, uint32_t x, int peer, bool send) {
  // the device protocol's stream operations are ordered after everything
  // already enqueued: flush the pending epoch only if it touches x (owner: x's
  // writers must precede the signal; reader: the replica's readers must
  // precede the copy).  Later work follows in stream order either way.
  if (!rt->comm->device_protocol() || rt->deps[x].epoch == rt->builder.epoch)
    if (int r = flush_epoch(rt)) return r;
  const Slot &xs = rt->slots[x];
  const uint32_t root = xs.root;
  float *const dptr = rt->hot[x].dptr;
  const uint64_t bytes = rt->hot[x].nx * 4;
  const uint64_t lo = reinterpret_cast<uint64_t>(dptr);
  auto ci = rt->caches.find(root);
  if (ci != rt->caches.end()) {
    if (send) {   // the peer reads this range of our replica: valid on the device first
      if (int r = ensure_device(rt, root, ci->second, lo, lo + bytes)) return r;
    } else {      // overwritten by the copy (a non-owner's replica holds the last value received)
      ci->second.pending.remove(lo, lo + bytes);
    }
  }
  if (int r = wait_uploads(rt, rt->stream, lo, lo + bytes)) return r;   // initial data in the replica
  std::string err;
  const int r = send ? rt->comm->send(rt->stream, peer, rt->slots[root].reg_key, rt->hot[root].dptr,
                                      rt->hot[root].nx * 4, &err)
                     : rt->comm->recv(rt->stream, peer, rt->slots[root].reg_key, (xs.offset - rt->slots[root].offset) * 4,
                                      dptr, bytes, &err);
  if (r) {
    rt->poisoned = -EIO;   // the ranks' streams are no longer in a known order
    return fail(rt, r, "cross-rank read: %s", err.c_str());
  }
  return 0;
}

// A task writes a part of slot s's root (every rank, local task or not).
inline void note_write(bt_runtime *rt, uint32_t s) {
  if (!rt->comm) return;
  const uint32_t r = rt->slots[s].root;
  if (rt->wver.size() <= r) rt->wver.resize(r + 1, 0);
  ++rt->wver[r];
}

int submit(bt_runtime *rt, int codelet, float scalar, bt_handle h0, bt_handle h1) {
  if (rt->poisoned) return fail(rt, rt->poisoned, "runtime poisoned by an earlier device error");
  int64_t s0 = operand(rt, codelet, h0);
  if (s0 < 0) return (int)s0;
  if (codelet == BT_CL_SCAL) note_write(rt, (uint32_t)s0);
  if (codelet == BT_CL_SCAL) {
    const SlotHot &x = rt->hot[s0];
    if (x.rank != rt->cfg.rank) {
      if (x.rank < 0) return insert_fail(rt, codelet, -EINVAL, "data has no home rank");
      rt->builder.add_remote();
      ++rt->stats.tasks_submitted;
      return 0;
    }
    if (!x.dptr && !rt->host_only) return insert_fail(rt, codelet, -EINVAL, "no local storage");
    uint32_t fb;
    memcpy(&fb, &scalar, 4);
    rt->builder.add_scal(rt->deps[s0], (uint32_t)s0, reinterpret_cast<uint64_t>(x.dptr), x.nx, fb);
  } else {
    int64_t s1 = operand(rt, codelet, h1);
    if (s1 < 0) return (int)s1;
    const SlotHot &x = rt->hot[s0];
    const SlotHot &y = rt->hot[s1];
    if (x.nx != y.nx) return insert_fail(rt, codelet, -EINVAL, "operand lengths differ");
    if (x.rank != y.rank) {
      if (x.rank < 0 || y.rank < 0) return insert_fail(rt, codelet, -EINVAL, "data has no home rank");
      if (!rt->comm)
        return insert_fail(rt, codelet, -EXDEV, "operands live on different ranks (see bt_comm_init)");
      // cross-rank read (comm.hpp): the task runs on y's owner, which first
      // copies x from x's owner; both meet here in submission order
      const int me = rt->cfg.rank;
      if (me == x.rank || me == y.rank) {
        if (!x.dptr || (me == y.rank && !y.dptr)) return insert_fail(rt, codelet, -EINVAL, "no local storage");
        // the pair's last transfer of this range is still current: skip (both sides)
        const Slot &xs = rt->slots[s0];
        const uint32_t root = xs.root;
        const int reader = y.rank;
        const auto key = std::make_tuple(rt->slots[root].reg_key, (uint64_t)(xs.offset - rt->slots[root].offset),
                                         (uint64_t)x.nx, reader);
        const std::pair<uint64_t, uint64_t> ver(root < rt->wver.size() ? rt->wver[root] : (uint64_t)0, rt->gver);
        auto it = rt->xcache.find(key);
        if (it != rt->xcache.end() && it->second == ver) {
          ++rt->stats.cross_rank_skips;
        } else {
          if (int r = cross_rank_read(rt, (uint32_t)s0, me == x.rank ? y.rank : x.rank, me == x.rank)) return r;
          rt->xcache[key] = ver;
          ++rt->stats.cross_rank_copies;
        }
      }
    }
    note_write(rt, (uint32_t)s1);
    if (y.rank != rt->cfg.rank) {
      if (y.rank < 0) return insert_fail(rt, codelet, -EINVAL, "data has no home rank");
      rt->builder.add_remote();
      ++rt->stats.tasks_submitted;
      return 0;
    }
    if ((!x.dptr || !y.dptr) && !rt->host_only) return insert_fail(rt, codelet, -EINVAL, "no local storage");
    uint32_t ab = 0;
    if (codelet == BT_CL_AXPY) memcpy(&ab, &scalar, 4);
    rt->builder.add_task((uint32_t)codelet, &rt->deps[s0], (uint32_t)s0, (uint32_t)BT_R, &rt->deps[s1],
                         (uint32_t)s1, (uint32_t)(codelet == BT_CL_AXPY ? BT_RW : BT_W),
                         reinterpret_cast<uint64_t>(x.dptr), reinterpret_cast<uint64_t>(y.dptr), x.nx, ab);
  }
  ++rt->stats.tasks_submitted;
  ++rt->stats.tasks_local;
  if (rt->cfg.epoch_tasks && rt->builder.ntasks >= rt->cfg.epoch_tasks && !rt->host_only) return flush_epoch(rt);
  return 0;
}

// A run of SCAL tasks [i0, i1) built on the pool.  Handles are grouped in
// blocks of 64 consecutive slots (768 bytes of DepState, so lanes never share
// a cache line); block k belongs to lane k % P; the round of a slot is fixed
// at allocation (SlotHot::grp): contiguous quarters of a partition's parts.
//   phase 1 (per chunk of the stream): validate, bucket by (round, lane);
//   phase 2 (per round, per lane): stable per-handle sort, runs -> items;
//   merge:  renumber the lanes' items into the epoch.
// Pipelined (R > 1, GPU runtime, long run): each round is flushed as its own
// epoch on one of two round streams as soon as it is built, so the device
// runs round r while the host builds round r+1 (rounds touch disjoint
// handles; a fork/join of events orders them after earlier work and before
// later work on the runtime's stream).  Returns 1 (nothing changed) if any
// task of the run would fail, so that the caller replays it sequentially and
// stops at the first error exactly like bt_insert_task; 0 when the whole run
// is submitted; a negative errno when submission failed after the run began
// to change state (items merged, rounds flushed): the runtime is then
// poisoned (-EIO from every later call), never replayed.
constexpr uint64_t kRemoteKey = 0xFFFFFFFEull;   // phase-1 key (low word) of another rank's SCAL target

// Phase 1 of scal_run_parallel, 8 tasks per step (AVX-512, selected at run
// time): 1 if all 8 are SCAL tasks whose slot key equals (their handle's
// generation | low) -- they continue the open run of group low >> 1 --, 2 if
// all 8 are valid SCALs on another rank's tiles, 0 otherwise (the caller then
// takes them one by one).  Slot indices are range-checked before the gather.
#if defined(__x86_64__)
__attribute__((target("avx512f,avx512vl"))) int block8(const bt_handle *h, const int32_t *c, const uint64_t *kt,
                                                       uint64_t nslots, uint64_t low) {
  const __m512i hv = _mm512_loadu_si512(h);
  const __m256i cv = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(c));
  const __mmask8 okc = _mm256_cmpeq_epi32_mask(cv, _mm256_set1_epi32(BT_CL_SCAL));
  const __m512i lo32 = _mm512_set1_epi64(0xFFFFFFFFll);
  const __m512i s = _mm512_sub_epi64(_mm512_and_si512(hv, lo32), _mm512_set1_epi64(1));
  const __mmask8 oks = _mm512_cmplt_epu64_mask(s, _mm512_set1_epi64((long long)nslots));
  if ((__mmask8)(okc & oks) != 0xFF) return 0;
  const __m512i k = _mm512_i64gather_epi64(s, reinterpret_cast<const long long *>(kt), 8);
  const __m512i gen = _mm512_andnot_si512(lo32, hv);
  if (low && _mm512_cmpeq_epi64_mask(k, _mm512_or_si512(gen, _mm512_set1_epi64((long long)low))) == 0xFF) return 1;
  if (_mm512_cmpeq_epi64_mask(k, _mm512_or_si512(gen, _mm512_set1_epi64((long long)kRemoteKey))) == 0xFF) return 2;
  return 0;
}
bool phase1_simd() {
  static const bool ok = getenv("BT_NO_SIMD") == nullptr && __builtin_cpu_supports("avx512f") &&
                         __builtin_cpu_supports("avx512vl");
  return ok;
}
#else
int block8(const bt_handle *, const int32_t *, const uint64_t *, uint64_t, uint64_t) { return 0; }
bool phase1_simd() { return false; }
#endif

int scal_run_parallel(bt_runtime *rt, const int32_t *codelets, const float *scalars, const bt_handle *h0, size_t i0,
                      size_t i1) {
  ++rt->gver;   // the run writes many roots: every shared copy across ranks is invalid
  const int P = rt->pool->size();
  const size_t n = i1 - i0;
  Builder &B = rt->builder;
  const bool pipelined = !rt->host_only && rt->cfg.pipeline_rounds > 1 && n >= rt->cfg.pipeline_min;
  const int R = rt->nrounds;              // groups are fixed per slot (SlotHot::grp); a
  const uint32_t G = (uint32_t)(P * R);   // non-pipelined run builds all rounds, then merges
  const int myrank = rt->cfg.rank;
  const bool host_only = rt->host_only;
  std::vector<int> bad(P, 0);
  std::vector<uint64_t> remote(P, 0);
  const size_t nslots = rt->hot.size();
  const SlotHot *hot = rt->hot.data();
  static const bool dbg = getenv("BT_DEBUG_TIMING") != nullptr;
  // task indices are epoch-relative; a pipelined run starts a fresh epoch
  // (a failure here changed nothing of the run: returned as is)
  if (pipelined && !B.items.empty())
    if (int r = flush_epoch(rt)) return r < 0 ? r : -EIO;
  const uint64_t tbase = B.ntasks;
  const bool record = B.record_tasks;
  double tp0 = now_ms();
  if (dbg && g_wait_return_ms > 0) fprintf(stderr, "scal_run_parallel: %.3f ms after the last wait returned\n", tp0 - g_wait_return_ms);
  if (rt->key_dirty || rt->key.size() != nslots) {
    rt->key.resize(nslots);
    uint64_t *key = rt->key.data();
    auto fill = [&](int c) {
      size_t lo, hi;
      range_of(nslots, nslots >= 65536 ? P : 1, c, lo, hi);
      for (size_t x = lo; x < hi; ++x) {
        const SlotHot &sh = hot[x];
        const bool ok = (sh.flags & (F_LIVE | F_PARTITIONED | F_BLOCKED)) == F_LIVE && (sh.dptr || host_only) &&
                        sh.rank == myrank;
        // another rank's valid SCAL target (owner-computes: skipped here) has
        // its own key, so phase 1 skips it without reading SlotHot
        const bool remote = !ok && (sh.flags & (F_LIVE | F_PARTITIONED | F_BLOCKED)) == F_LIVE && sh.rank != myrank &&
                            sh.rank >= 0;
        key[x] = ((uint64_t)sh.gen << 32) |
                 (remote ? kRemoteKey : ((uint64_t)(sh.grp & 0x7FFFFFFFu) << 1) | (ok ? 1u : 0u));
      }
    };
    if (nslots >= 65536) rt->par(fill);
    else fill(0);
    // a partition whose parts are spread over ranks (owner-computes): deal
    // THIS rank's parts to the rounds, so its share of a run still pipelines
    for (size_t x = 0; x < nslots; ++x) {
      const Slot &ps = rt->slots[x];
      if (!ps.nparts || !ps.prounds || !(hot[x].flags & F_LIVE)) continue;
      const uint32_t c0 = ps.first_child, n = ps.nparts;
      uint64_t L = 0;
      for (uint32_t t = 0; t < n; ++t) L += hot[c0 + t].rank == myrank;
      if (L == 0 || L == n) continue;
      uint64_t j = 0;
      for (uint32_t t = 0; t < n; ++t) {
        if (hot[c0 + t].rank != myrank) continue;
        const uint32_t grp = round_of(j++, L, ps.prounds, ps.pgeo) * (uint32_t)P + ((c0 + t) >> 6) % (uint32_t)P;
        key[c0 + t] = (key[c0 + t] & ~0xFFFFFFFEull) | ((uint64_t)(grp & 0x7FFFFFFFu) << 1);
      }
    }
    rt->key_dirty = false;
  }
  const uint64_t *kt = rt->key.data();
  std::vector<double> tstart(P), tend(P), tloop(P);
  rt->par([&](int c) {
    if (dbg) tstart[c] = now_ms();
    size_t lo, hi;
    range_of(n, P, c, lo, hi);
    // this chunk's run lists, moved to the stack while filling (no false
    // sharing of vector headers between threads); phase 1 writes only run
    // records (one per change of group along the stream), not the tasks:
    // the lanes read their tasks' handles and factors from the caller's
    // arrays in phase 2, so phase 1 (which every launch waits for) reads
    // codelets + handles once and writes almost nothing
    std::vector<vec<RunRec>> mine(G);
    std::vector<uint64_t> cnt(G, 0);
    for (uint32_t g = 0; g < G; ++g) {
      mine[g].swap(rt->runs[(size_t)c * G + g]);
      mine[g].clear();
    }
    struct Restore {
      std::vector<vec<RunRec>> &m;
      std::vector<uint64_t> &cnt;
      bt_runtime *rt;
      int c;
      uint32_t G;
      ~Restore() {
        for (uint32_t g = 0; g < G; ++g) {
          m[g].swap(rt->runs[(size_t)c * G + g]);
          rt->run_tasks[(size_t)c * G + g] = cnt[g];
        }
      }
    } restore{mine, cnt, rt, c, G};
    uint64_t rem = 0;
    uint32_t cur = NONE;      // group of the open run
    size_t run0 = lo;         // its first task
    auto close_run = [&](size_t j) {
      if (cur == NONE) return;
      mine[cur].push_back(RunRec{(uint32_t)run0, (uint32_t)(j - run0)});
      cnt[cur] += j - run0;
      cur = NONE;
    };
    if (dbg) tloop[c] = now_ms();
    // one task: false if the run must be rejected
    auto step = [&](size_t j) -> bool {
      const bt_handle h = h0[i0 + j];
      const uint32_t s = (uint32_t)(h & 0xFFFFFFFFull) - 1u;   // handle index 0 wraps to UINT32_MAX
      if (__builtin_expect(codelets[i0 + j] != BT_CL_SCAL || s >= nslots, 0)) return false;
      const uint64_t k = kt[s];
      if (__builtin_expect(((k >> 32) != (h >> 32)) | !(k & 1u), 0)) {
        if (k == ((h & 0xFFFFFFFF00000000ull) | kRemoteKey)) {   // another rank's tile: skipped
          close_run(j);
          ++rem;
          return true;
        }
        // not a local SCAL target: a stale handle or a bad state (the run
        // fails), or another rank's tile (skipped)
        const SlotHot &sh = hot[s];
        if (sh.gen != (uint32_t)(h >> 32) || (sh.flags & (F_LIVE | F_PARTITIONED | F_BLOCKED)) != F_LIVE ||
            (!sh.dptr && !host_only) || sh.rank == myrank || sh.rank < 0)
          return false;
        close_run(j);
        ++rem;
        return true;
      }
      const uint32_t g = (uint32_t)k >> 1;
      if (g != cur) {
        close_run(j);
        cur = g;
        run0 = j;
      }
      return true;
    };
    size_t j = lo;
    if (phase1_simd()) {
      // 8 tasks at a time while they continue the open run (or are all
      // another rank's); any other block of 8 goes through step()
      for (; j + 8 <= hi;) {
        const int r = block8(h0 + i0 + j, codelets + i0 + j, kt, nslots,
                             cur == NONE ? 0ull : ((uint64_t)cur << 1) | 1u);
        if (r == 1) {
          j += 8;
          continue;
        }
        if (r == 2) {
          close_run(j);
          rem += 8;
          j += 8;
          continue;
        }
        for (const size_t e = j + 8; j < e; ++j)
          if (!step(j)) {
            bad[c] = 1;
            return;
          }
      }
    }
    for (; j < hi; ++j)
      if (!step(j)) {
        bad[c] = 1;
        return;
      }
    close_run(hi);
    remote[c] = rem;
    if (dbg) tend[c] = now_ms();
  });
  if (dbg) {
    double s0 = 1e30, s1 = 0, l1 = 0, e1 = 0, lmax = 0;
    for (int c = 0; c < P; ++c) {
      s0 = std::min(s0, tstart[c]);
      s1 = std::max(s1, tstart[c]);
      l1 = std::max(l1, tloop[c]);
      e1 = std::max(e1, tend[c]);
      lmax = std::max(lmax, tend[c] - tloop[c]);
    }
    fprintf(stderr, "phase1: first start +%.3f, last start +%.3f, last loop start +%.3f, last end +%.3f, max loop %.3f ms\n",
            s0 - tp0, s1 - tp0, l1 - tp0, e1 - tp0, lmax);
  }
  for (int c = 0; c < P; ++c)
    if (bad[c]) {
      if (dbg) fprintf(stderr, "scal_run_parallel: chunk %d rejected, sequential replay\n", c);
      return 1;
    }
  if (B.record_tasks) {
    B.task_item.resize(tbase + n, NONE);
    B.task_pos.resize(tbase + n, 0);
  }
  uint64_t rem = 0;
  for (int c = 0; c < P; ++c) rem += remote[c];
  rt->stats.tasks_submitted += n;
  rt->stats.tasks_local += n - rem;
  // from here on the dependency states change: a failure poisons the runtime
  struct PoisonOnFail {
    bt_runtime *rt;
    bool ok = false;
    ~PoisonOnFail() {
      if (!ok && !rt->poisoned) {
        rt->poisoned = -EIO;
        fail(rt, -EIO, "SCAL run failed part-way (%s): runtime poisoned", rt->last_error.c_str());
      }
    }
  } poison_on_fail{rt};
  if (pipelined) {
    CUDA_TRY(rt, cudaEventRecord(rt->ev_fork, rt->stream));
    for (int i = 0; i < 2; ++i) CUDA_TRY(rt, cudaStreamWaitEvent(rt->rstream[i], rt->ev_fork, 0));
  }
  DepState *deps = rt->deps.data();
  const double tp1 = now_ms();
  double t_p2 = 0, t_merge = 0, t_flush = 0;
  std::vector<double> t_launch;
  // lane l owns slot blocks k with k % P == l (in every round); dense local
  // index over the lane's blocks: (k / P) * 64 + (s & 63)
  const uint32_t nlocal = (uint32_t)((((nslots + 63) >> 6) + P - 1) / P) * 64;
  // (k / P) * 64 per 64-slot block k, so the per-task local index needs no division
  std::vector<uint32_t> blk_local((nslots + 63) >> 6);
  for (size_t k = 0; k < blk_local.size(); ++k) blk_local[k] = (uint32_t)(k / (size_t)P) * 64;
  std::vector<size_t> round_size(R, 0);
  size_t local = 0;
  for (int c = 0; c < P; ++c)
    for (int r = 0; r < R; ++r)
      for (int l = 0; l < P; ++l) round_size[r] += rt->run_tasks[(size_t)c * G + (size_t)r * P + l];
  for (int r = 0; r < R; ++r) local += round_size[r];
  // launches: adjacent rounds are merged so that each launch carries at least
  // pipeline_min / 2 local tasks (a short run -- e.g. one rank's shard -- is
  // launch-overhead bound with many small launches); [bound[j], bound[j+1])
  // are the rounds of launch j.  Empty rounds belong to another round policy.
  std::vector<int> bound{0};
  if (pipelined) {
    // a round that joins a stream launch costs ~20 us of host flush, a
    // separate launch much more: with stream launches possible, rounds of at
    // least pipeline_min / 8 tasks stay separate (an N = 8 rank's shard of C5
    // starts after 1/16 of it is built instead of 7/16)
    const bool streamable = rt->sctl && rt->caches.empty() && !(rt->cfg.flags & BT_FLAG_TIMESTAMPS);
    const size_t per = std::max<size_t>(1, rt->cfg.pipeline_min / (streamable ? 8 : 2));
    int nonempty = 0;
    for (int r = 0; r < R; ++r) nonempty += round_size[r] != 0;
    const size_t want = std::max<size_t>(1, std::min<size_t>((size_t)nonempty, local / per));
    size_t cum = 0;
    size_t j = 0;
    int idx = 0;
    for (int r = 0; r < R; ++r) {
      // every nonempty round its own launch when they are few enough, else
      // rounds merged into `want` launches of balanced task counts
      const size_t jr = (size_t)nonempty <= want ? (size_t)(round_size[r] ? idx++ : std::max(idx - 1, 0))
                        : local ? std::min(want - 1, cum * want / local)
                                : 0;   // launch of round r
      if (jr != j && round_size[r]) {
        bound.push_back(r);
        j = jr;
      }
      cum += round_size[r];
    }
  }
  bound.push_back(R);
  const int launches = (int)bound.size() - 1;
  // the rounds' epochs join one stream launch (if the first one's kernel
  // choice allows it: flush_epoch); sl is reset however this run ends
  struct SlReset {
    bt_runtime *rt;
    ~SlReset() {
      static const bool dbg = getenv("BT_DEBUG_ERRORS") != nullptr;
      if (dbg && rt->sl.started && rt->sl.next != rt->sl.nsub)
        fprintf(stderr, "btask: stream launch published %u of %u sub-epochs\n", rt->sl.next, rt->sl.nsub);
      // a run that failed part-way: end its launch (no CTA waits for the watchdog)
      if (rt->sl.started && rt->sl.next < rt->sl.nsub) close_stream(rt);
      rt->sl.started = rt->sl.launched = false;
      rt->sl.want = rt->sl.active = false;
      rt->sl.run_tasks = rt->sl.cur_tasks = 0;
      for (EpochBuf *&b : rt->sl.bufs) {   // a run that failed before its deferred launch
        if (b) b->held = false;
        b = nullptr;
      }
    }
  } sl_reset{rt};
  if (pipelined && rt->sctl) {
    unsigned nsub = 0;
    rt->sl.max_tasks = 0;
    for (int rr = 0; rr < launches; ++rr) {
      size_t sz = 0;
      for (int r = bound[rr]; r < bound[rr + 1]; ++r) sz += round_size[r];
      nsub += sz != 0;
      rt->sl.max_tasks = std::max<uint64_t>(rt->sl.max_tasks, sz);
    }
    rt->sl.want = nsub >= 2 && nsub <= (unsigned)kMaxSubs;
    rt->sl.active = false;
    rt->sl.nsub = nsub;
    rt->sl.run_tasks = local;
  }
  // direct rounds (Builder::lane_count / lane_write): pipelined rounds of
  // device-resident data go from the sorted tasks straight to the device
  // descriptors (no items, edges, merge or pack pass); BT_NO_DIRECT_ROUNDS=1
  // builds them through lane_runs as before (comparisons)
  static const bool no_direct_rounds = getenv("BT_NO_DIRECT_ROUNDS") != nullptr;
  const bool direct_rounds = pipelined && !no_direct_rounds && rt->caches.empty() && !record &&
                             !(rt->cfg.flags & BT_FLAG_TIMESTAMPS);
  std::vector<Lane *> dlanes;
  for (int rr = 0; rr < launches; ++rr) {
    const int rlo = bound[rr], rhi = bound[rr + 1];
    size_t sz = 0;
    for (int r = rlo; r < rhi; ++r) sz += round_size[r];
    if (pipelined && sz == 0) continue;
    const double ta = now_ms();
    if (direct_rounds) {
      rt->par([&](int l) {
        for (int r = rlo; r < rhi; ++r) {
          const uint32_t g = (uint32_t)(r * P + l);
          Lane &L = rt->lanes[(size_t)(r - rlo) * P + l];
          // the lane's tasks, straight from the caller's arrays (the run records of phase 1)
          auto src = [&](auto &&visit) {
            for (int c = 0; c < P; ++c)
              for (const RunRec &run : rt->runs[(size_t)c * G + g]) {
                const bt_handle *hh = h0 + i0 + run.start;
                const uint32_t *ff = reinterpret_cast<const uint32_t *>(scalars + i0 + run.start);
                for (uint32_t j = 0; j < run.len; ++j) visit((uint32_t)(hh[j] & 0xFFFFFFFFull) - 1u, ff[j]);
              }
          };
          B.lane_count(
              L, src, nlocal, [bl = blk_local.data()](uint32_t s) { return bl[s >> 6] + (s & 63); },
              [up = (uint32_t)P, ul = (uint32_t)l](uint32_t loc) { return ((loc >> 6) * up + ul) * 64 + (loc & 63); },
              [hot](uint32_t s) {
                return std::pair<uint64_t, uint64_t>(reinterpret_cast<uint64_t>(hot[s].dptr), hot[s].nx);
              });
        }
      });
      const double tb = now_ms();
      // item order: round, then lane; each lane object's bases
      dlanes.clear();
      DirectRound dr{nullptr, 0, 0, 0, 0, 0, 0, 0};
      for (int r = rlo; r < rhi; ++r)
        for (int l = 0; l < P; ++l) {
          Lane *L = &rt->lanes[(size_t)(r - rlo) * P + l];
          if (L->hr.empty()) continue;
          L->ibase = dr.N;
          L->fbase = dr.F;
          dr.N += L->d_items;
          dr.E += L->d_items - L->hr.size();
          dr.F += L->d_fac;
          dr.elems += L->d_elems;
          dr.work += L->d_work;
          dr.tasks += L->d_tasks;
          dlanes.push_back(L);
        }
      dr.lanes = dlanes.data();
      dr.nlanes = dlanes.size();
      B.ntasks = tbase + n;   // the round's epoch accounts the run
      rt->sl.cur_tasks = sz;
      cudaStream_t st = rt->rstream[rr & 1];
      const double tc = now_ms();
      if (int e = flush_epoch(rt, st, &dr)) return e;
      CUDA_TRY(rt, cudaEventRecord(rt->ev_round[rr & 1], st));
      if (dbg) t_launch.push_back(now_ms() - tp0);
      t_p2 += tb - ta;
      t_flush += now_ms() - tc;
      continue;
    }
    rt->par([&](int l) {
      // this lane builds its groups of every round of the launch in one go
      for (int r = rlo; r < rhi; ++r) {
        const uint32_t g = (uint32_t)(r * P + l);
        Lane &L = rt->lanes[(size_t)(r - rlo) * P + l];
        // gather this group's tasks from the batch, in stream order
        size_t m = 0;
        for (int c = 0; c < P; ++c) m += rt->run_tasks[(size_t)c * G + g];
        L.gather.resize(m);
        if (record) L.gtask.resize(m);
        LaneEntry *ge = L.gather.data();
        uint32_t *gt = L.gtask.data();
        size_t q = 0;
        for (int c = 0; c < P; ++c)
          for (const RunRec &run : rt->runs[(size_t)c * G + g]) {
            const bt_handle *hh = h0 + i0 + run.start;
            const float *ff = scalars + i0 + run.start;
            for (uint32_t j = 0; j < run.len; ++j) {
              ge[q + j].slot = (uint32_t)(hh[j] & 0xFFFFFFFFull) - 1u;
              memcpy(&ge[q + j].fbits, &ff[j], 4);
            }
            if (record)
              for (uint32_t j = 0; j < run.len; ++j) gt[q + j] = (uint32_t)(tbase + run.start + j);
            q += run.len;
          }
        const LaneEntry *ptrs[1] = {ge};
        const uint32_t *tptr[1] = {record ? gt : nullptr};
        const size_t cnts[1] = {m};
        B.lane_runs(
            L, ptrs, tptr, cnts, 1, deps, nlocal,
            [bl = blk_local.data()](uint32_t s) { return bl[s >> 6] + (s & 63); },
            [up = (uint32_t)P, ul = (uint32_t)l](uint32_t loc) { return ((loc >> 6) * up + ul) * 64 + (loc & 63); },
            [hot](uint32_t s) {
              return std::pair<uint64_t, uint64_t>(reinterpret_cast<uint64_t>(hot[s].dptr), hot[s].nx);
            });
      }
    });
    const double tb = now_ms();
    B.merge(rt->lanes, P * (rhi - rlo), deps, [&](const std::function<void(int)> &f) { rt->pool->run(f); }, P);
    const double tc = now_ms();
    if (pipelined) {
      B.ntasks = tbase + n;   // the round's epoch accounts the run (its items carry the tasks)
      rt->sl.cur_tasks = sz;
      cudaStream_t st = rt->rstream[rr & 1];
      if (int e = flush_epoch(rt, st)) return e;
      CUDA_TRY(rt, cudaEventRecord(rt->ev_round[rr & 1], st));
      if (dbg) t_launch.push_back(now_ms() - tp0);
    }
    t_p2 += tb - ta;
    t_merge += tc - tb;
    t_flush += now_ms() - tc;
  }
  if (pipelined) {
    for (int i = 0; i < std::min(launches, 2); ++i) CUDA_TRY(rt, cudaStreamWaitEvent(rt->stream, rt->ev_round[i], 0));
  } else {
    B.ntasks = tbase + n;
  }
  if (dbg)
    fprintf(stderr,
            "scal_run_parallel n=%zu P=%d R=%d phase1 %.3f ms phase2 %.3f ms merge %.3f ms flush %.3f ms\n", n, P, R,
            tp1 - tp0, t_p2, t_merge, t_flush);
  if (dbg)
    for (size_t j = 0; j < t_launch.size(); ++j) fprintf(stderr, "  launch %zu issued at %.3f ms\n", j, t_launch[j]);
  poison_on_fail.ok = true;
  return 0;
}

}  // namespace

extern "C" {

int bt_insert_task(bt_runtime *rt, int codelet, const void *cl_args, size_t cl_args_size, const bt_handle *handles,
                   const int *modes, unsigned nbuffers) {
  if (int r = check_live(rt)) return r;
  float scalar = 0.f;
  switch (codelet) {
    case BT_CL_SCAL:
      if (nbuffers != 1 || !handles || !modes || modes[0] != BT_RW)
        return insert_fail(rt, codelet, -EINVAL, "vector_scal takes one RW buffer");
      if (cl_args_size != 4 || !cl_args) return insert_fail(rt, codelet, -EINVAL, "vector_scal takes one float");
      memcpy(&scalar, cl_args, 4);
      return submit(rt, codelet, scalar, handles[0], 0);
    case BT_CL_AXPY:
      if (nbuffers != 2 || !handles || !modes || modes[0] != BT_R || modes[1] != BT_RW)
        return insert_fail(rt, codelet, -EINVAL, "axpy takes buffers (R, RW)");
      if (cl_args_size != 4 || !cl_args) return insert_fail(rt, codelet, -EINVAL, "axpy takes one float");
      memcpy(&scalar, cl_args, 4);
      return submit(rt, codelet, scalar, handles[0], handles[1]);
    case BT_CL_COPY:
      if (nbuffers != 2 || !handles || !modes || modes[0] != BT_R || modes[1] != BT_W)
        return insert_fail(rt, codelet, -EINVAL, "copy takes buffers (R, W)");
      if (cl_args_size != 0) return insert_fail(rt, codelet, -EINVAL, "copy takes no scalar");
      return submit(rt, codelet, 0.f, handles[0], handles[1]);
    default:
      return fail(rt, -EINVAL, "failed to insert task: unknown codelet %d", codelet);
  }
}

int bt_insert_task_batch(bt_runtime *rt, size_t ntasks, const int32_t *codelets, const float *scalars,
                         const bt_handle *h0, const bt_handle *h1, size_t *nsubmitted) {
  if (nsubmitted) *nsubmitted = 0;
  if (int r = check_live(rt)) return r;
  if (ntasks && (!codelets || !scalars || !h0)) return fail(rt, -EINVAL, "null batch array");
  const double t0 = now_ms();
  size_t i = 0;
  int rc = 0;
  const size_t pmin = rt->cfg.parallel_min;
  // common case first: the whole batch is one long valid SCAL run
  // (scal_run_parallel: 1 = rejected, nothing changed -> per-task path below;
  // negative = failed part-way -> the error, nothing counted as submitted)
  if (ntasks >= pmin) {
    const int pr = scal_run_parallel(rt, codelets, scalars, h0, 0, ntasks);
    if (pr < 0) {
      rt->stats.host_build_ms += now_ms() - t0;
      return pr;
    }
    if (pr == 0) {
      i = ntasks;
      if (rt->cfg.epoch_tasks && rt->builder.ntasks >= rt->cfg.epoch_tasks && !rt->host_only) rc = flush_epoch(rt);
    }
  }
  while (i < ntasks && rc == 0) {
    if (codelets[i] == BT_CL_SCAL) {
      size_t j = i;
      while (j < ntasks && codelets[j] == BT_CL_SCAL) ++j;
      if (j - i >= pmin && j - i < ntasks) {
        const int pr = scal_run_parallel(rt, codelets, scalars, h0, i, j);
        if (pr < 0) {
          rc = pr;
          break;
        }
        if (pr == 0) {
          i = j;
          if (rt->cfg.epoch_tasks && rt->builder.ntasks >= rt->cfg.epoch_tasks && !rt->host_only)
            rc = flush_epoch(rt);
          continue;
        }
      }
      for (; i < j; ++i) {      // short run, or a task of the run fails: sequential
        rc = submit(rt, BT_CL_SCAL, scalars[i], h0[i], 0);
        if (rc) break;
      }
      continue;
    }
    const int c = codelets[i];
    if (c != BT_CL_SCAL && ((c != BT_CL_AXPY && c != BT_CL_COPY) || !h1)) {
      rc = fail(rt, -EINVAL, "failed to insert task: bad codelet %d or missing operand array", c);
      break;
    }
    rc = submit(rt, c, scalars[i], h0[i], c == BT_CL_SCAL ? 0 : h1[i]);
    if (rc) break;
    ++i;
  }
  rt->stats.host_build_ms += now_ms() - t0;
  if (nsubmitted) *nsubmitted = i;
  return rc;
}

int bt_flush(bt_runtime *rt) {
  if (int r = check_live(rt)) return r;
  if (rt->host_only) return fail(rt, -ENODEV, "host-only runtime: nothing executes");
  cudaSetDevice(rt->device);
  return flush_epoch(rt);
}

int bt_task_wait_for_all(bt_runtime *rt) {
  if (int r = check_live(rt)) return r;
  if (rt->host_only) return fail(rt, -ENODEV, "host-only runtime: nothing executes");
  cudaSetDevice(rt->device);
  return wait_all(rt);
}

}  // extern "C"

namespace {
// Make the host copy of device bytes [lo, hi) of host-homed root `root`
// current (caller has run wait_all): untouched since registration -> nothing;
// every write covered by an eager write-back -> wait for those copies;
// otherwise copy the range back after them (same copy stream).
int sync_to_host(bt_runtime *rt, uint32_t root, uint64_t lo, uint64_t hi) {
  auto it = rt->caches.find(root);
  if (it == rt->caches.end()) return 0;
  RootCache &c = it->second;
  const bool touched = c.written.overlaps(lo, hi);
  std::vector<std::pair<uint64_t, uint64_t>> ps;
  c.dirty.pieces(lo, hi, ps, true);   // written again since their eager write-back
  for (const auto &pc : ps) {
    char *host = static_cast<char *>(rt->slots[root].hptr) + (pc.first - c.dlo);
    CUDA_TRY(rt, cudaMemcpyAsync(host, reinterpret_cast<const void *>(pc.first), pc.second - pc.first,
                                 cudaMemcpyDeviceToHost, rt->d2h));
    rt->stats.d2h_data_bytes += pc.second - pc.first;
  }
  if (touched || c.wb) CUDA_TRY(rt, cudaStreamSynchronize(rt->d2h));
  return 0;
}
}  // namespace

extern "C" {

int bt_data_acquire(bt_runtime *rt, bt_handle h, int mode) {
  if (int r = check_live(rt)) return r;
  uint32_t s = resolve(rt, h);
  if (s == NONE) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  if (mode != BT_R && mode != BT_RW) return fail(rt, -EINVAL, "acquire mode must be R or RW");
  if (acquired_chain(rt, s)) return fail(rt, -EBUSY, "already acquired");
  const Slot &sl = rt->slots[s];
  const SlotHot &sh = rt->hot[s];
  const Slot &root = rt->slots[sl.root];
  if (root.home_node != 0 || !root.hptr) return fail(rt, -EINVAL, "no host copy to acquire into");
  if (rt->host_only) return fail(rt, -ENODEV, "host-only runtime");
  if (sh.rank != rt->cfg.rank || !sh.dptr) return fail(rt, -EINVAL, "data not stored on this rank");
  cudaSetDevice(rt->device);
  if (int r = wait_all(rt)) return r;
  const uint64_t lo = reinterpret_cast<uint64_t>(sh.dptr);
  if (int r = sync_to_host(rt, sl.root, lo, lo + sh.nx * 4)) return r;
  rt->slots[s].acquired = mode;
  set_blocked(rt, s, true);
  return 0;
}

int bt_data_release(bt_runtime *rt, bt_handle h) {
  if (int r = check_live(rt)) return r;
  ++rt->gver;   // host writes (RW): collective under bt_comm_init (btask.h)
  uint32_t s = resolve(rt, h);
  if (s == NONE) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  Slot &sl = rt->slots[s];
  if (!sl.acquired) return fail(rt, -EINVAL, "handle is not acquired");
  if (sl.acquired == BT_RW) {
    const Slot &root = rt->slots[sl.root];
    const SlotHot &sh = rt->hot[s];
    cudaSetDevice(rt->device);
    CUDA_TRY(rt, cudaMemcpyAsync(sh.dptr, static_cast<float *>(root.hptr) + sl.offset, sh.nx * 4,
                                 cudaMemcpyHostToDevice, rt->stream));
    rt->stats.h2d_data_bytes += sh.nx * 4;
    auto it = rt->caches.find(sl.root);
    if (it != rt->caches.end()) {
      const uint64_t lo = reinterpret_cast<uint64_t>(sh.dptr);
      it->second.pending.remove(lo, lo + sh.nx * 4);
      it->second.dirty.remove(lo, lo + sh.nx * 4);   // the device copy now equals the host's
    }
    // host writes under RW acquire: later tasks see them (stream order)
    CUDA_TRY(rt, cudaStreamSynchronize(rt->stream));
  }
  sl.acquired = 0;
  set_blocked(rt, s, false);
  return 0;
}

int bt_data_unregister(bt_runtime *rt, bt_handle h) {
  if (int r = check_live(rt)) return r;
  ++rt->gver;
  uint32_t s = resolve(rt, h);
  if (s == NONE) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  Slot &sl = rt->slots[s];
  rt->key_dirty = true;
  SlotHot &sh = rt->hot[s];
  if (sl.parent != NONE) return fail(rt, -EBUSY, "cannot unregister a sub-handle");
  if (sl.nparts) return fail(rt, -EBUSY, "unpartition before unregistering");
  if (sl.acquired) return fail(rt, -EBUSY, "release before unregistering");
  if (!rt->host_only) {
    cudaSetDevice(rt->device);
    if (int r = wait_all(rt)) return r;
    if (sl.home_node == 0 && sl.hptr && sh.dptr) {
      const uint64_t lo = reinterpret_cast<uint64_t>(sh.dptr);
      if (int r = sync_to_host(rt, s, lo, lo + sh.nx * 4)) return r;
    }
    rt->caches.erase(s);
    if (sl.owns_dev && sl.ipc_alloc) {
      CUDA_TRY(rt, cudaStreamSynchronize(rt->stream));
      CUDA_TRY(rt, cudaFree(sh.dptr));
    } else if (sl.owns_dev) {
      CUDA_TRY(rt, cudaFreeAsync(sh.dptr, rt->stream));
    }
  }
  if (sl.hptr) {
    rt->ranges.erase(reinterpret_cast<uintptr_t>(sl.hptr));
    rt->by_ptr.erase(reinterpret_cast<uintptr_t>(sl.hptr));
  }
  free_slots(rt, s, 1);
  --rt->live_roots;
  return 0;
}

int bt_malloc(void **out, size_t bytes) {
  if (!out) return -EINVAL;
  *out = nullptr;
  if (cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    return -ENOMEM;
  }
  return 0;
}

int bt_free(void *ptr) {
  if (!ptr) return 0;
  return cudaFreeHost(ptr) == cudaSuccess ? 0 : -EINVAL;
}

const char *bt_strerror(int err) { return strerror(err < 0 ? -err : err); }

const char *bt_last_error(bt_runtime *rt) { return rt ? rt->last_error.c_str() : ""; }

int bt_stats_get(bt_runtime *rt, bt_stats *out) {
  if (!rt || !out) return -EINVAL;
  *out = rt->stats;
  return 0;
}

int bt_stats_reset(bt_runtime *rt) {
  if (!rt) return -EINVAL;
  const uint32_t g = rt->stats.grid, b = rt->stats.block;
  rt->stats = bt_stats{};
  rt->stats.grid = g;
  rt->stats.block = b;
  return 0;
}

int bt_dag_snapshot(bt_runtime *rt, bt_dag_view *out) {
  if (!rt || !out) return -EINVAL;
  if (!rt->host_only) return fail(rt, -EPERM, "bt_dag_snapshot needs a BT_FLAG_HOST_ONLY runtime");
  Builder &B = rt->builder;
  const size_t N = B.items.size();
  rt->snap_kind.resize(N);
  rt->snap_k.resize(N);
  rt->snap_npred.resize(N);
  rt->snap_flags.resize(N);
  rt->snap_off.resize(N + 1);
  rt->snap_succ.resize(B.edges.size());
  uint32_t acc = 0;
  for (size_t i = 0; i < N; ++i) {
    rt->snap_off[i] = acc;
    acc += B.items[i].nsucc;
    rt->snap_kind[i] = (uint8_t)B.items[i].kind;
    rt->snap_k[i] = B.items[i].k;
    rt->snap_npred[i] = B.items[i].npred;
    rt->snap_flags[i] = B.items[i].item_deps ? (uint8_t)BT_DAG_WHOLE_PREDS : (uint8_t)0;
  }
  rt->snap_off[N] = acc;
  rt->cursor.assign(rt->snap_off.begin(), rt->snap_off.end() - 1);
  for (uint64_t ed : B.edges) rt->snap_succ[rt->cursor[ed >> 32]++] = (uint32_t)ed;
  rt->snap_task_item = B.task_item;
  rt->snap_task_pos = B.task_pos;
  out->ntasks = B.ntasks;
  out->nitems = N;
  out->nedges = B.edges.size();
  out->task_item = rt->snap_task_item.data();
  out->task_pos = rt->snap_task_pos.data();
  out->item_kind = rt->snap_kind.data();
  out->item_k = rt->snap_k.data();
  out->item_npred = rt->snap_npred.data();
  out->succ_off = rt->snap_off.data();
  out->succ = rt->snap_succ.data();
  out->item_flags = rt->snap_flags.data();
  rt->stats.items += N;
  rt->stats.edges += B.edges.size();
  rt->stats.fused_tasks += B.fused;
  B.next_epoch();
  return 0;
}

// Test hook (btask.h): hold rt->stream until the caller sets a mapped flag.
// A stream memory wait occupies no SM; the gate kernel (fallback) one thread.
int bt_debug_gate(bt_runtime *rt, volatile uint32_t **flag_out) {
  if (int r = check_live(rt)) return r;
  if (!flag_out) return fail(rt, -EINVAL, "null flag pointer");
  if (rt->host_only) return fail(rt, -ENODEV, "host-only runtime: nothing executes");
  cudaSetDevice(rt->device);
  uint32_t *flag = nullptr;
  if (cudaHostAlloc((void **)&flag, 64, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return fail(rt, -ENOMEM, "cannot allocate the gate flag");
  }
  rt->gates.push_back(flag);
  __atomic_store_n(flag, 0u, __ATOMIC_SEQ_CST);
  uint32_t *dflag = nullptr;
  CUDA_TRY(rt, cudaHostGetDevicePointer((void **)&dflag, flag, 0));
  // CUresult cuStreamWaitValue32(CUstream, CUdeviceptr, cuuint32_t, unsigned flags); GEQ = 0
  using WaitValue32 = int (*)(cudaStream_t, unsigned long long, uint32_t, unsigned);
  static WaitValue32 wait_value = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (getenv("BT_GATE_KERNEL") || cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      fn = nullptr;
    }
    return reinterpret_cast<WaitValue32>(fn);
  }();
  if (!wait_value || wait_value(rt->stream, reinterpret_cast<unsigned long long>(dflag), 1u, 0u) != 0) {
    cudaGetLastError();
    CUDA_TRY(rt, launch_gate(dflag, 60ull * 1000 * 1000 * 1000, rt->stream));
    ++rt->stats.kernel_launches;
  }
  *flag_out = flag;
  return 0;
}

int bt_trace(bt_runtime *rt, const uint64_t **t, const uint32_t **item, uint64_t *n) {
  if (!rt || !t || !item || !n) return -EINVAL;
  if (rt->trace_item.empty()) return -ENODATA;
  *t = rt->trace_t.data();
  *item = rt->trace_item.data();
  *n = rt->trace_item.size();
  return 0;
}

}  // extern "C"
