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
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/btask.h"
#include "builder.hpp"
#include "device_abi.h"

namespace bt {
cudaError_t launch_epoch(const EpochArgs &args, int grid, cudaStream_t stream);
cudaError_t scheduler_occupancy(int *blocks_per_sm, int *block);
int max_factors();
}  // namespace bt

using namespace bt;

namespace {

constexpr uint32_t kDefaultChunkBytes = 256u << 10;
constexpr uint32_t kDefaultMaxFused = 256;
constexpr uint64_t kWatchdogNs = 20ull * 1000 * 1000 * 1000;   // 20 s

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

struct Slot {
  uint32_t gen = 1;
  bool live = false;
  uint32_t parent = NONE;
  uint32_t child_index = 0;
  uint32_t nparts = 0;        // partitioned into nparts children if > 0
  uint32_t first_child = NONE;
  uint32_t root = NONE;       // top-level ancestor (itself for a top-level handle)
  float *dptr = nullptr;      // device address of element 0 (null: no local storage)
  uint64_t nx = 0;
  uint64_t offset = 0;        // element offset inside the root
  void *hptr = nullptr;       // root only: registered pointer
  int home_node = 0;
  int rank = 0;
  int acquired = 0;           // 0, BT_R or BT_RW
  bool owns_dev = false;      // root only: runtime-allocated replica
};

struct EpochBuf {
  char *hblob = nullptr;
  size_t hcap = 0;
  char *dblob = nullptr;
  size_t dcap = 0;
  cudaEvent_t start = nullptr, end = nullptr, done = nullptr;
  bool inflight = false;
  uint64_t units = 0;
  bool traced = false;
  size_t ctr_readback = 0;    // offset of the Counters readback in hblob
  size_t trace_off_h = 0;     // offset of the trace copy in hblob
};

}  // namespace

struct bt_runtime {
  bt_config cfg;
  bool host_only = false;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sms = 0;
  int grid_max = 0;
  int block = 0;
  uint64_t chunk_elems = 0;
  int poisoned = 0;
  std::string last_error;

  std::vector<Slot> slots;
  std::vector<DepState> deps;
  std::map<uint32_t, std::vector<uint32_t>> free_ranges;   // count -> starts
  std::map<uintptr_t, std::pair<uintptr_t, uint32_t>> ranges;  // start -> (end, root slot)
  std::unordered_map<uintptr_t, uint32_t> by_ptr;          // exact base -> root slot
  uint32_t live_roots = 0;

  Builder builder;
  EpochBuf ep[2];
  int ep_cur = 0;
  bt_stats stats{};

  // host-only snapshot storage
  std::vector<uint8_t> snap_kind;
  std::vector<uint32_t> snap_k, snap_npred, snap_off, snap_succ;
  std::vector<uint32_t> snap_task_item, snap_task_pos;

  // last trace
  std::vector<uint64_t> trace_t;
  std::vector<uint32_t> trace_item;

  // pack scratch
  std::vector<uint32_t> cursor, node_off, csr_off;
  std::vector<uint8_t> node_written;
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

#define CUDA_TRY(rt, call)                                   \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) return cuda_fail((rt), e_, #call); \
  } while (0)

inline bt_handle make_handle(const bt_runtime *rt, uint32_t s) {
  return ((uint64_t)rt->slots[s].gen << 32) | (uint64_t)(s + 1);
}

// Resolve a handle to a live slot, or NONE.
inline uint32_t resolve(const bt_runtime *rt, bt_handle h) {
  const uint64_t idx = (h & 0xFFFFFFFFull);
  if (idx == 0 || idx > rt->slots.size()) return NONE;
  const uint32_t s = (uint32_t)(idx - 1);
  const Slot &sl = rt->slots[s];
  if (!sl.live || sl.gen != (uint32_t)(h >> 32)) return NONE;
  return s;
}

uint32_t alloc_slots(bt_runtime *rt, uint32_t count) {
  auto it = rt->free_ranges.find(count);
  uint32_t s;
  if (it != rt->free_ranges.end() && !it->second.empty()) {
    s = it->second.back();
    it->second.pop_back();
  } else {
    s = (uint32_t)rt->slots.size();
    rt->slots.resize(s + count);
    rt->deps.resize(s + count);
  }
  for (uint32_t i = 0; i < count; ++i) {
    Slot &sl = rt->slots[s + i];
    const uint32_t gen = sl.gen;
    sl = Slot();
    sl.gen = gen;
    sl.live = true;
    rt->deps[s + i].epoch = NONE;
  }
  return s;
}

void free_slots(bt_runtime *rt, uint32_t s, uint32_t count) {
  for (uint32_t i = 0; i < count; ++i) {
    Slot &sl = rt->slots[s + i];
    sl.live = false;
    ++sl.gen;
    if (sl.gen == 0) sl.gen = 1;
    rt->deps[s + i] = DepState();
  }
  rt->free_ranges[count].push_back(s);
}

bool acquired_chain(const bt_runtime *rt, uint32_t s) {
  for (uint32_t p = s; p != NONE; p = rt->slots[p].parent)
    if (rt->slots[p].acquired) return true;
  return false;
}

int check_live(bt_runtime *rt) {
  if (!rt) return -EINVAL;
  if (rt->poisoned) return fail(rt, rt->poisoned, "runtime poisoned by an earlier device error");
  return 0;
}

// ---------------------------------------------------------------- epochs --

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

int ensure_host(bt_runtime *rt, EpochBuf &e, size_t need) {
  if (e.hcap >= need) return 0;
  if (e.hblob) cudaFreeHost(e.hblob);
  e.hblob = nullptr;
  size_t cap = std::max(need, e.hcap + e.hcap / 2);
  CUDA_TRY(rt, cudaHostAlloc((void **)&e.hblob, cap, cudaHostAllocPortable));
  e.hcap = cap;
  return 0;
}

int ensure_dev(bt_runtime *rt, EpochBuf &e, size_t need) {
  if (e.dcap >= need) return 0;
  if (e.dblob) cudaFree(e.dblob);
  e.dblob = nullptr;
  size_t cap = std::max(need, e.dcap + e.dcap / 2);
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
  if (cudaEventElapsedTime(&ms, e.start, e.end) == cudaSuccess) rt->stats.device_ms += ms;
  const Counters *c = reinterpret_cast<const Counters *>(e.hblob + e.ctr_readback);
  if (c->error != ERR_NONE) {
    rt->poisoned = -EIO;
    return fail(rt, -EIO, "device scheduler fault (code %u%s)", c->error,
                c->error == ERR_WATCHDOG ? ": watchdog, a unit was never released" : "");
  }
  if (c->head < e.units) {
    rt->poisoned = -EIO;
    return fail(rt, -EIO, "device scheduler ended early (%llu of %llu units)", (unsigned long long)c->head,
                (unsigned long long)e.units);
  }
  if (e.traced) {
    rt->trace_t.assign(reinterpret_cast<const uint64_t *>(e.hblob + e.trace_off_h),
                       reinterpret_cast<const uint64_t *>(e.hblob + e.trace_off_h) + 4 * e.units);
    const uint32_t *ti = reinterpret_cast<const uint32_t *>(e.hblob + e.trace_off_h + 32 * e.units);
    rt->trace_item.assign(ti, ti + e.units);
  }
  return 0;
}

// CSR of successors + offsets, from the builder's edge list (creation order).
void build_csr(bt_runtime *rt, std::vector<uint32_t> &off, uint32_t *succ) {
  const auto &items = rt->builder.items;
  const size_t n = items.size();
  off.resize(n + 1);
  uint32_t acc = 0;
  for (size_t i = 0; i < n; ++i) {
    off[i] = acc;
    acc += items[i].nsucc;
  }
  off[n] = acc;
  rt->cursor.assign(off.begin(), off.end() - 1);
  for (uint64_t e : rt->builder.edges) succ[rt->cursor[e >> 32]++] = (uint32_t)e;
}

int flush_epoch(bt_runtime *rt) {
  Builder &B = rt->builder;
  if (B.items.empty()) {
    B.next_epoch();
    return 0;
  }
  const double t0 = now_ms();
  EpochBuf &e = rt->ep[rt->ep_cur];
  rt->ep_cur ^= 1;
  if (int r = retire(rt, e)) return r;

  const size_t N = B.items.size();
  const size_t E = B.edges.size();
  const uint64_t CE = rt->chunk_elems;
  // factor lists: one materialised copy per distinct trie node used by an item
  rt->node_off.assign(B.nodes.size(), NONE);
  size_t F = 0;
  for (const HItem &it : B.items)
    if (it.kind == K_SCAL && rt->node_off[it.arg] == NONE) {
      rt->node_off[it.arg] = (uint32_t)F;
      F += it.k;
    }
  uint64_t U = 0, U0 = 0;
  for (const HItem &it : B.items) {
    const uint64_t nc = (it.n + CE - 1) / CE;
    U += nc;
    if (it.npred == 0) U0 += nc;
  }
  // device layout: ctr | items | pending | succ | factors | queue[U] | chunk_done[N] | trace
  const size_t o_ctr = 0;
  const size_t o_items = 64;
  const size_t o_pend = align_up(o_items + 48 * N, 16);
  const size_t o_succ = align_up(o_pend + 4 * N, 16);
  const size_t o_fac = align_up(o_succ + 4 * E, 16);
  const size_t o_queue = align_up(o_fac + 4 * F, 16);
  const size_t upload = o_queue + 8 * U0;
  const size_t o_cdone = align_up(o_queue + 8 * U, 16);
  const size_t o_trace = align_up(o_cdone + 4 * N, 16);
  const bool traced = (rt->cfg.flags & BT_FLAG_TIMESTAMPS) != 0;
  const size_t dneed = o_trace + (traced ? 36 * U : 0);
  const size_t o_readback = align_up(upload, 64);
  const size_t o_trace_h = o_readback + 64;
  const size_t hneed = o_trace_h + (traced ? 36 * U : 0);
  if (int r = ensure_host(rt, e, hneed)) return r;
  if (int r = ensure_dev(rt, e, dneed)) return r;

  char *h = e.hblob;
  Counters *ctr = reinterpret_cast<Counters *>(h + o_ctr);
  memset(ctr, 0, sizeof(Counters));
  ctr->head = 0;
  ctr->tail = U0;
  DItem *di = reinterpret_cast<DItem *>(h + o_items);
  int32_t *pend = reinterpret_cast<int32_t *>(h + o_pend);
  uint32_t *succ = reinterpret_cast<uint32_t *>(h + o_succ);
  float *fac = reinterpret_cast<float *>(h + o_fac);
  unsigned long long *q = reinterpret_cast<unsigned long long *>(h + o_queue);

  std::vector<uint32_t> &offs = rt->csr_off;
  build_csr(rt, offs, succ);
  // factor lists: each used trie node is written once, walking to the root
  rt->node_written.assign(B.nodes.size(), 0);
  for (const HItem &it : B.items) {
    if (it.kind != K_SCAL || rt->node_written[it.arg]) continue;
    rt->node_written[it.arg] = 1;
    float *dst = fac + rt->node_off[it.arg];
    uint32_t node = it.arg;
    for (int64_t j = (int64_t)it.k - 1; j >= 0; --j) {
      const TrieNode &nd = B.nodes[node];
      memcpy(dst + j, &nd.fbits, 4);
      node = nd.parent;
    }
  }
  uint64_t qi = 0;
  for (size_t i = 0; i < N; ++i) {
    const HItem &it = B.items[i];
    DItem &d = di[i];
    d.x = it.x;
    d.y = it.y;
    d.n = it.n;
    d.kind = it.kind;
    d.k = it.k;
    d.arg = it.kind == K_SCAL ? rt->node_off[it.arg] : it.arg;
    const uint64_t nc = (it.n + CE - 1) / CE;
    d.nchunks = (uint32_t)nc;
    d.succ_off = offs[i];
    d.nsucc = it.nsucc;
    pend[i] = (int32_t)it.npred;
    if (it.npred == 0)
      for (uint64_t c = 0; c < nc; ++c) q[qi++] = ((unsigned long long)i << 32) | c;
  }

  char *d = e.dblob;
  CUDA_TRY(rt, cudaMemcpyAsync(d, h, upload, cudaMemcpyHostToDevice, rt->stream));
  if (U > U0) CUDA_TRY(rt, cudaMemsetAsync(d + o_queue + 8 * U0, 0xFF, 8 * (U - U0), rt->stream));
  CUDA_TRY(rt, cudaMemsetAsync(d + o_cdone, 0, 4 * N, rt->stream));

  EpochArgs a{};
  a.items = reinterpret_cast<const DItem *>(d + o_items);
  a.pending = reinterpret_cast<int32_t *>(d + o_pend);
  a.chunk_done = reinterpret_cast<uint32_t *>(d + o_cdone);
  a.succ = reinterpret_cast<const uint32_t *>(d + o_succ);
  a.factors = reinterpret_cast<const float *>(d + o_fac);
  a.queue = reinterpret_cast<unsigned long long *>(d + o_queue);
  a.ctr = reinterpret_cast<Counters *>(d + o_ctr);
  a.trace = traced ? reinterpret_cast<unsigned long long *>(d + o_trace) : nullptr;
  a.trace_item = traced ? reinterpret_cast<uint32_t *>(d + o_trace + 32 * U) : nullptr;
  a.total_units = U;
  a.chunk_elems = CE;
  a.watchdog_ns = kWatchdogNs;
  a.nitems = (uint32_t)N;
  const int grid = (int)std::min<uint64_t>((uint64_t)rt->grid_max, U);

  CUDA_TRY(rt, cudaEventRecord(e.start, rt->stream));
  CUDA_TRY(rt, launch_epoch(a, grid, rt->stream));
  CUDA_TRY(rt, cudaEventRecord(e.end, rt->stream));
  CUDA_TRY(rt, cudaMemcpyAsync(h + o_readback, d + o_ctr, 64, cudaMemcpyDeviceToHost, rt->stream));
  if (traced) CUDA_TRY(rt, cudaMemcpyAsync(h + o_trace_h, d + o_trace, 36 * U, cudaMemcpyDeviceToHost, rt->stream));
  CUDA_TRY(rt, cudaEventRecord(e.done, rt->stream));
  e.inflight = true;
  e.units = U;
  e.traced = traced;
  e.ctr_readback = o_readback;
  e.trace_off_h = o_trace_h;

  rt->stats.items += N;
  rt->stats.edges += E;
  rt->stats.units += U;
  rt->stats.epochs += 1;
  rt->stats.upload_bytes += upload;
  rt->stats.fused_tasks += B.fused;
  rt->stats.grid = (uint32_t)grid;
  B.next_epoch();
  rt->stats.host_build_ms += now_ms() - t0;
  if (rt->cfg.flags & BT_FLAG_SYNC_EPOCH) return retire(rt, e);
  return 0;
}

int wait_all(bt_runtime *rt) {
  if (int r = flush_epoch(rt)) return r;
  // retire in launch order (older first)
  EpochBuf &older = rt->ep[rt->ep_cur];
  EpochBuf &newer = rt->ep[rt->ep_cur ^ 1];
  if (int r = retire(rt, older)) return r;
  if (int r = retire(rt, newer)) return r;
  CUDA_TRY(rt, cudaStreamSynchronize(rt->stream));
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
  if (cfg.chunk_bytes == 0) cfg.chunk_bytes = kDefaultChunkBytes;
  if (cfg.chunk_bytes < 32) return -EINVAL;

  bt_runtime *rt = new (std::nothrow) bt_runtime();
  if (!rt) return -ENOMEM;
  rt->cfg = cfg;
  rt->host_only = (cfg.flags & BT_FLAG_HOST_ONLY) != 0;
  rt->builder.fusion = (cfg.flags & BT_FLAG_NO_FUSION) == 0;
  rt->builder.max_fused = cfg.max_fused;
  rt->builder.record_tasks = rt->host_only;
  rt->chunk_elems = std::max<uint64_t>(8, (cfg.chunk_bytes / 4) / 8 * 8);

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
    // keep freed replicas in the pool (register/unregister loops reuse them)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
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
      if (e.dblob) cudaFree(e.dblob);
      if (e.start) cudaEventDestroy(e.start);
      if (e.end) cudaEventDestroy(e.end);
      if (e.done) cudaEventDestroy(e.done);
    }
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
  if (!rt->host_only && ptr) {
    cudaSetDevice(rt->device);
    if (home_node == 1) {
      dptr = static_cast<float *>(ptr);
    } else {
      cudaError_t e = cudaMallocAsync((void **)&dptr, nx * 4, rt->stream);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(rt, -ENOMEM, "cannot allocate the device replica (%zu bytes)", nx * 4);
      }
      owns = true;
      e = cudaMemcpyAsync(dptr, ptr, nx * 4, cudaMemcpyHostToDevice, rt->stream);
      if (e != cudaSuccess) {
        cudaFreeAsync(dptr, rt->stream);
        return cuda_fail(rt, e, "register upload");
      }
    }
  }
  const uint32_t s = alloc_slots(rt, 1);
  Slot &sl = rt->slots[s];
  sl.root = s;
  sl.dptr = dptr;
  sl.nx = nx;
  sl.hptr = ptr;
  sl.home_node = home_node;
  sl.rank = ptr ? rt->cfg.rank : -1;
  sl.owns_dev = owns;
  if (ptr) {
    rt->ranges[lo] = {hi, s};
    rt->by_ptr[lo] = s;
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
  uint32_t s = resolve(rt, h);
  if (s == NONE) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  if (rt->slots[s].nparts) return fail(rt, -EBUSY, "handle already partitioned");
  if (acquired_chain(rt, s)) return fail(rt, -EBUSY, "handle is acquired");
  if (nparts == 0 || nparts > rt->slots[s].nx) return fail(rt, -EINVAL, "bad number of parts");
  const uint32_t c0 = alloc_slots(rt, nparts);   // may reallocate slots/deps
  Slot &p = rt->slots[s];
  const uint64_t base = p.nx / nparts, extra = p.nx % nparts;
  for (uint32_t t = 0; t < nparts; ++t) {
    Slot &c = rt->slots[c0 + t];
    const uint64_t off = t * base + std::min<uint64_t>(t, extra);
    c.parent = s;
    c.child_index = t;
    c.root = p.root;
    c.offset = p.offset + off;
    c.nx = base + (t < extra ? 1 : 0);
    c.dptr = p.dptr ? p.dptr + off : nullptr;
    c.rank = p.rank;
  }
  p.nparts = nparts;
  p.first_child = c0;
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

int bt_data_unpartition(bt_runtime *rt, bt_handle h) {
  if (int r = check_live(rt)) return r;
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
  return 0;
}

int bt_data_set_rank(bt_runtime *rt, bt_handle h, int rank) {
  if (int r = check_live(rt)) return r;
  uint32_t s = resolve(rt, h);
  if (s == NONE) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  if (rank < 0 || rank >= rt->cfg.nranks) return fail(rt, -EINVAL, "rank %d out of range", rank);
  // the handle and all its parts (recursively)
  std::vector<uint32_t> stack{s};
  while (!stack.empty()) {
    uint32_t x = stack.back();
    stack.pop_back();
    rt->slots[x].rank = rank;
    const Slot &sl = rt->slots[x];
    for (uint32_t t = 0; t < sl.nparts; ++t) stack.push_back(sl.first_child + t);
  }
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
  const Slot &sl = rt->slots[s];
  if (sl.nparts) return insert_fail(rt, codelet, -EBUSY, "handle is partitioned");
  if (acquired_chain(rt, s)) return insert_fail(rt, codelet, -EBUSY, "handle is acquired");
  return s;
}

int submit(bt_runtime *rt, int codelet, float scalar, bt_handle h0, bt_handle h1) {
  int64_t s0 = operand(rt, codelet, h0);
  if (s0 < 0) return (int)s0;
  if (codelet == BT_CL_SCAL) {
    const Slot &x = rt->slots[s0];
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
    const Slot &x = rt->slots[s0];
    const Slot &y = rt->slots[s1];
    if (x.nx != y.nx) return insert_fail(rt, codelet, -EINVAL, "operand lengths differ");
    if (x.rank != y.rank) {
      if (x.rank < 0 || y.rank < 0) return insert_fail(rt, codelet, -EINVAL, "data has no home rank");
      return insert_fail(rt, codelet, -EXDEV, "operands live on different ranks");
    }
    if (y.rank != rt->cfg.rank) {
      if (y.rank < 0) return insert_fail(rt, codelet, -EINVAL, "data has no home rank");
      rt->builder.add_remote();
      ++rt->stats.tasks_submitted;
      return 0;
    }
    if ((!x.dptr || !y.dptr) && !rt->host_only) return insert_fail(rt, codelet, -EINVAL, "no local storage");
    uint32_t ab = 0;
    if (codelet == BT_CL_AXPY) memcpy(&ab, &scalar, 4);
    Access a0{(uint32_t)s0, (uint32_t)BT_R};
    Access a1{(uint32_t)s1, (uint32_t)(codelet == BT_CL_AXPY ? BT_RW : BT_W)};
    DepState *d0 = &rt->deps[s0];
    DepState *d1 = &rt->deps[s1];
    rt->builder.add_task((uint32_t)codelet, d0, a0, d1, a1, reinterpret_cast<uint64_t>(x.dptr),
                         reinterpret_cast<uint64_t>(y.dptr), x.nx, ab);
  }
  ++rt->stats.tasks_submitted;
  ++rt->stats.tasks_local;
  if (rt->cfg.epoch_tasks && rt->builder.ntasks >= rt->cfg.epoch_tasks && !rt->host_only) return flush_epoch(rt);
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
  for (; i < ntasks; ++i) {
    const int c = codelets[i];
    if (c != BT_CL_SCAL) {
      if ((c != BT_CL_AXPY && c != BT_CL_COPY) || !h1) {
        rc = fail(rt, -EINVAL, "failed to insert task: bad codelet %d or missing operand array", c);
        break;
      }
    }
    rc = submit(rt, c, scalars[i], h0[i], c == BT_CL_SCAL ? 0 : h1[i]);
    if (rc) break;
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

int bt_data_acquire(bt_runtime *rt, bt_handle h, int mode) {
  if (int r = check_live(rt)) return r;
  uint32_t s = resolve(rt, h);
  if (s == NONE) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  if (mode != BT_R && mode != BT_RW) return fail(rt, -EINVAL, "acquire mode must be R or RW");
  if (acquired_chain(rt, s)) return fail(rt, -EBUSY, "already acquired");
  Slot &sl = rt->slots[s];
  const Slot &root = rt->slots[sl.root];
  if (root.home_node != 0 || !root.hptr) return fail(rt, -EINVAL, "no host copy to acquire into");
  if (rt->host_only) return fail(rt, -ENODEV, "host-only runtime");
  if (sl.rank != rt->cfg.rank || !sl.dptr) return fail(rt, -EINVAL, "data not stored on this rank");
  cudaSetDevice(rt->device);
  if (int r = wait_all(rt)) return r;
  CUDA_TRY(rt, cudaMemcpyAsync(static_cast<float *>(root.hptr) + sl.offset, sl.dptr, sl.nx * 4,
                               cudaMemcpyDeviceToHost, rt->stream));
  CUDA_TRY(rt, cudaStreamSynchronize(rt->stream));
  rt->slots[s].acquired = mode;
  return 0;
}

int bt_data_release(bt_runtime *rt, bt_handle h) {
  if (int r = check_live(rt)) return r;
  uint32_t s = resolve(rt, h);
  if (s == NONE) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  Slot &sl = rt->slots[s];
  if (!sl.acquired) return fail(rt, -EINVAL, "handle is not acquired");
  if (sl.acquired == BT_RW) {
    const Slot &root = rt->slots[sl.root];
    cudaSetDevice(rt->device);
    CUDA_TRY(rt, cudaMemcpyAsync(sl.dptr, static_cast<float *>(root.hptr) + sl.offset, sl.nx * 4,
                                 cudaMemcpyHostToDevice, rt->stream));
    // host writes under RW acquire: later tasks must see them (stream order)
    CUDA_TRY(rt, cudaStreamSynchronize(rt->stream));
  }
  sl.acquired = 0;
  return 0;
}

int bt_data_unregister(bt_runtime *rt, bt_handle h) {
  if (int r = check_live(rt)) return r;
  uint32_t s = resolve(rt, h);
  if (s == NONE) return fail(rt, -ENOENT, "attempt to use unregistered pointer");
  Slot &sl = rt->slots[s];
  if (sl.parent != NONE) return fail(rt, -EBUSY, "cannot unregister a sub-handle");
  if (sl.nparts) return fail(rt, -EBUSY, "unpartition before unregistering");
  if (!rt->host_only) {
    cudaSetDevice(rt->device);
    if (int r = wait_all(rt)) return r;
    if (sl.home_node == 0 && sl.hptr && sl.dptr) {
      CUDA_TRY(rt, cudaMemcpyAsync(sl.hptr, sl.dptr, sl.nx * 4, cudaMemcpyDeviceToHost, rt->stream));
      CUDA_TRY(rt, cudaStreamSynchronize(rt->stream));
    }
    if (sl.owns_dev) CUDA_TRY(rt, cudaFreeAsync(sl.dptr, rt->stream));
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
  rt->snap_succ.resize(B.edges.size());
  build_csr(rt, rt->snap_off, rt->snap_succ.data());
  for (size_t i = 0; i < N; ++i) {
    rt->snap_kind[i] = (uint8_t)B.items[i].kind;
    rt->snap_k[i] = B.items[i].k;
    rt->snap_npred[i] = B.items[i].npred;
  }
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
  rt->stats.items += N;
  rt->stats.edges += B.edges.size();
  rt->stats.fused_tasks += B.fused;
  B.next_epoch();
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
