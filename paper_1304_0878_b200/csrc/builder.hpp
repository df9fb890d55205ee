// builder.hpp -- host dependency builder: submission order -> epoch DAG.
//
// "These access modes, along with the sequence of task
// invocations, allows StarPU to determine at run-time the dependency graph of
// tasks."  Rule (reading R5), per leaf (sub)handle:
//   state = { writers: tasks whose writes are the latest,
//             readers: tasks that read since then }
//   access with R : depend on every writer                      (RAW)
//   access with W : depend on every writer and every reader     (WAW, WAR)
//                   then writers = {T}, readers = {}
//   access R only : readers += {T}
// Partition copies the parent's state into every part; unpartition sets the
// parent's state to the union of its parts' states (reading R9) -- no barrier
// task is needed and tiles stay independent.
//
// Vertical fusion (BASELINE north_star: "a fused pass over consecutive inout
// scalings of the same tile"): a SCAL(RW) whose only predecessor would be the
// current single writer W of its handle, where W is a SCAL item of this epoch
// on the same handle with no successor yet, is appended to W's factor list
// instead of becoming a new item.  The factors stay in submission order; the
// device applies them one rounding at a time.
//
// Two insertion paths produce identical DAGs up to item numbering:
//  * sequential (any codelet): add_scal / add_task;
//  * parallel lanes for long runs of SCAL tasks: a SCAL touches one handle,
//    so the stream decomposes by handle.  Lane p owns the handles of slot
//    blocks (slot >> 6) % P == p, sorts its tasks by handle (stable) and
//    turns each handle's run into lane-local items ("tagged" ids, bit 31);
//    merge() renumbers them into the global item array.
#pragma once
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <memory>
#include <utility>
#include <vector>

#include "device_abi.h"

namespace bt {

// std::allocator that default-initialises (no zero fill on resize): the
// builder resizes multi-megabyte arrays whose every element it overwrites.
template <class T>
struct NoInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = NoInitAlloc<U>;
  };
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U> &) {}
  template <class U>
  void construct(U *p) noexcept {
    ::new (static_cast<void *>(p)) U;
  }
  template <class U, class... A>
  void construct(U *p, A &&...a) {
    ::new (static_cast<void *>(p)) U(std::forward<A>(a)...);
  }
};
template <class T>
using vec = std::vector<T, NoInitAlloc<T>>;

constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr uint32_t TAG = 0x80000000u;     // lane-local item id / lane-local factor offset
constexpr uint32_t STAMP_NONE = 0x7FFFFFFFu;   // HItem::stamp of no task

// Per leaf (sub)handle.  12 bytes; multi-writer / reader sets live in exts.
struct DepState {
  uint32_t epoch = NONE;   // states of older epochs are empty
  uint32_t writer = NONE;  // single latest writer (common case)
  uint32_t ext = NONE;     // index into Builder::exts, or NONE
};

struct DepExt {
  std::vector<uint32_t> writers;  // >1 latest writers (after unpartition)
  std::vector<uint32_t> readers;
};

struct HItem {
  uint32_t kind;       // 1 SCAL, 2 AXPY, 3 COPY
  uint32_t k;          // tasks in this item
  uint32_t slot0, slot1;
  uint64_t x, y, n;    // device addresses / elements
  uint32_t arg;        // AXPY: scalar bits
  uint32_t fofs;       // SCAL: factor offset in the factor pool (TAG: lane pool)
  uint32_t fcap;       // SCAL: reserved factors at fofs
  uint32_t npred;
  uint32_t nsucc;      // updated atomically by lanes for shared predecessors
  uint32_t stamp : 31; // dedupe marker (sequential path; item ids < 2^31)
  // 1: some predecessor's operand on the (sub)handle it was found through has
  // another base address than this item's operand there (partition-inherited
  // state: a parent, parts, or a reused slot): its chunks need not line up
  // with this item's, so every predecessor counts as a whole (no chunk-wise
  // release)
  uint32_t item_deps : 1;
};

struct LaneEntry {
  uint32_t slot;
  uint32_t fbits;
};

// A run of consecutive tasks of one SCAL batch whose handles belong to the
// same builder group (stream positions [start, start + len) of the batch).
struct RunRec {
  uint32_t start;
  uint32_t len;
};

// A handle's run in a direct round (Builder::lane_count): its tasks' factors
// are fpool[start, start + m), split into `items` chained items.
struct RunH {
  uint32_t slot, start, m, items;
};

struct alignas(64) Lane {
  vec<LaneEntry> gather;              // the lane's entries of one round, gathered from the runs
  vec<uint32_t> gtask;                // their task indices (record_tasks only)
  vec<uint32_t> cnt;                  // lane_runs scratch: per local slot counters
  vec<uint32_t> tasks;                // lane_runs scratch: task index per sorted factor
  vec<HItem> items;
  vec<uint64_t> edges;                // (pred << 32) | succ, ids possibly TAGged
  vec<float> fpool;
  std::vector<uint32_t> touched;      // slots whose state now holds a tagged id
  std::vector<uint32_t> relocated;    // global items whose factors moved to fpool
  std::vector<uint64_t> recorded;     // (task << 32) | tagged item (record_tasks)
  uint64_t fused = 0;
  // direct rounds (lane_count / lane_write): the lane's handle runs, its
  // totals, and its bases in the epoch's arrays
  vec<RunH> hr;
  vec<uint8_t> reuse;                 // per item with > 1 factor: 1 = same list as the lane's previous one
  uint64_t d_items = 0, d_elems = 0, d_work = 0, d_fac = 0, d_tasks = 0, d_units = 0, d_ready = 0;
  uint64_t ibase = 0, fbase = 0, qbase = 0;
  char pad_[64];                      // keep neighbouring lanes off this cache line
  void clear() {
    items.clear();
    edges.clear();
    fpool.clear();
    touched.clear();
    relocated.clear();
    recorded.clear();
    fused = 0;
  }
};

class Builder {
 public:
  // Epoch-scoped outputs
  vec<HItem> items;
  vec<uint64_t> edges;              // (pred << 32) | succ
  vec<float> fpool;                 // factor lists of SCAL items
  std::vector<DepExt> exts;
  std::vector<uint32_t> task_item;  // per epoch task (only if record_tasks)
  std::vector<uint32_t> task_pos;
  uint64_t ntasks = 0;              // tasks of this epoch (local or not)
  uint64_t fused = 0;
  bool record_tasks = false;
  bool fusion = true;
  uint32_t max_fused = 256;
  uint32_t epoch = 0;

  void clear() {
    items.clear();
    edges.clear();
    fpool.clear();
    exts.clear();
    task_item.clear();
    task_pos.clear();
    ntasks = 0;
    fused = 0;
  }
  void next_epoch() {
    clear();
    ++epoch;
  }

  void record(uint32_t item, uint32_t pos) {
    if (record_tasks) {
      task_item.push_back(item);
      task_pos.push_back(pos);
    }
  }

  // A task executed on another rank (kept for the task -> item map).
  void add_remote() {
    record(NONE, 0);
    ++ntasks;
  }

  // ---- sequential path ------------------------------------------------
  // SCAL(f; x:RW) on leaf slot s (x = device address of element 0, n elems).
  void add_scal(DepState &st, uint32_t s, uint64_t x, uint64_t n, uint32_t fbits) {
    fresh(st);
    ++ntasks;
    if (fusion && st.ext == NONE && st.writer != NONE) {
      HItem &w = items[st.writer];
      if (w.kind == 1 && w.slot0 == s && w.nsucc == 0 && w.k < max_fused) {
        append_factor(w, fbits);
        record(st.writer, w.k - 1);
        ++fused;
        return;
      }
    }
    const uint32_t t = new_item(1, s, NONE, x, 0, n, 0);
    HItem &it = items[t];
    it.fofs = (uint32_t)fpool.size();
    it.fcap = 4;
    fpool.resize(fpool.size() + 4);
    memcpy(&fpool[it.fofs], &fbits, 4);
    collect(st, t, 3u, s);
    st.writer = t;
    st.ext = NONE;
  }

  // Generic task with two accesses (AXPY: x R, y RW; COPY: x R, y W).
  void add_task(uint32_t kind, DepState *st0, uint32_t s0, uint32_t m0, DepState *st1, uint32_t s1, uint32_t m1,
                uint64_t x, uint64_t y, uint64_t n, uint32_t arg) {
    fresh(*st0);
    if (st1 != st0) fresh(*st1);
    ++ntasks;
    const uint32_t t = new_item(kind, s0, s1, x, y, n, arg);
    if (st1 == st0) {  // same handle twice: modes OR-ed (reading R6)
      const uint32_t m = m0 | m1;
      collect(*st0, t, m, s0);
      update(*st0, t, m);
    } else {
      collect(*st0, t, m0, s0);
      collect(*st1, t, m1, s1);
      update(*st0, t, m0);
      update(*st1, t, m1);
    }
  }

  // Partition: every part inherits the parent's state (reading R9).
  void partition_state(DepState &parent, DepState *parts, uint32_t nparts);
  // Unpartition: the parent's writers/readers are the union over the parts.
  void unpartition_state(DepState &parent, DepState *parts, uint32_t nparts);

  // ---- parallel lanes (SCAL runs) -------------------------------------
  // Process all of a lane's entries at once: a stable counting sort by slot
  // puts each handle's factors contiguously (submission order kept), then
  // every run becomes items without further copies (factor lists point into
  // the sorted lane pool).  `chunks[c]` / `counts[c]` are the entries bucketed
  // by chunk c of the stream (chunk order = submission order); `loc` maps an
  // owned slot to a dense local index < nlocal and `slot_of` back; `geom(s)`
  // gives the slot's (device address, elements).
  // `ctasks[c]` (only read when record_tasks) holds the epoch task index of
  // each entry of chunks[c].
  template <class Loc, class SlotOf, class Geom>
  void lane_runs(Lane &L, const LaneEntry *const *chunks, const uint32_t *const *ctasks, const size_t *counts,
                 int nchunks, DepState *deps, uint32_t nlocal, Loc &&loc, SlotOf &&slot_of, Geom &&geom);
  // Renumber lane items into the global arrays; deps[] of touched slots fixed.
  // Runs lane p's share on worker p via `par` (a fork/join runner).
  template <class Par>
  void merge(std::vector<Lane> &lanes, size_t nlanes, DepState *deps, Par &&par, int nworkers);

  const float *factors(const HItem &it) const { return &fpool[it.fofs]; }

  // ---- direct rounds ---------------------------------------------------
  // A round of a pipelined SCAL run is its own epoch, flushed right after it
  // is built: every handle's tasks form one chain that starts ready (the
  // earlier epochs precede it in stream order) and no two handles interact.
  // Such a round skips the item / edge / merge / pack pipeline: lane_count
  // sorts the lane's tasks by handle (stable) and counts items, elements and
  // distinct factor lists; the runtime lays the epoch out from the lanes'
  // totals; lane_write then writes the device descriptors themselves (item
  // ids = the lane's base + position; a chain's successor is the next id,
  // stored inline).  Same items, same factor order as lane_runs would build.
  template <class Src, class Loc, class SlotOf, class Geom>
  void lane_count(Lane &L, Src &&src, uint32_t nlocal, Loc &&loc, SlotOf &&slot_of, Geom &&geom);
  template <class Geom, class Item>
  void lane_write(Lane &L, uint64_t chunk_elems, float *fac, unsigned long long *queue, Geom &&geom, Item &&item);

 private:
  void fresh(DepState &st) {
    if (st.epoch != epoch) {
      st.epoch = epoch;
      st.writer = NONE;
      st.ext = NONE;
    }
  }

  DepExt &ext_of(DepState &st) {
    if (st.ext == NONE) {
      st.ext = (uint32_t)exts.size();
      exts.emplace_back();
    }
    return exts[st.ext];
  }

  void append_factor(HItem &w, uint32_t fbits) {
    if (w.k == w.fcap) {
      const uint32_t cap = w.fcap * 2;
      const uint32_t ofs = (uint32_t)fpool.size();
      fpool.resize(fpool.size() + cap);
      memmove(&fpool[ofs], &fpool[w.fofs], 4ull * w.k);
      w.fofs = ofs;
      w.fcap = cap;
    }
    memcpy(&fpool[w.fofs + w.k], &fbits, 4);
    ++w.k;
  }

  uint32_t new_item(uint32_t kind, uint32_t s0, uint32_t s1, uint64_t x, uint64_t y, uint64_t n, uint32_t arg) {
    const uint32_t t = (uint32_t)items.size();
    items.push_back(HItem{kind, 1, s0, s1, x, y, n, arg, 0, 0, 0, 0, STAMP_NONE, 0});
    record(t, 0);
    return t;
  }

  void edge(uint32_t p, uint32_t t) {
    HItem &pi = items[p];
    if (pi.stamp == t) return;
    pi.stamp = t;
    ++pi.nsucc;
    ++items[t].npred;
    edges.push_back(((uint64_t)p << 32) | t);
  }

  // The predecessors in the state of (sub)handle `slot`, which item t accesses.
  // A predecessor with an operand at the same base address as t's operand on
  // `slot` touched, in its chunk c, exactly the elements t's chunk c touches
  // there (equal lengths are checked on the device); any other -- found
  // through partition-inherited state, or on a slot id reused within the
  // epoch by another part -- makes t wait for whole predecessors (item_deps).
  // Base addresses, not slot ids: a freed slot range is reused by the next
  // partition with as many parts, possibly of another parent.
  void collect(DepState &st, uint32_t t, uint32_t mode, uint32_t slot) {
    const uint64_t base = slot == items[t].slot0 ? items[t].x : items[t].y;
    auto add = [&](uint32_t p) {
      const HItem &pi = items[p];
      if (pi.x != base && pi.y != base) items[t].item_deps = 1;
      edge(p, t);
    };
    if (st.writer != NONE) add(st.writer);
    if (st.ext != NONE) {
      const DepExt &e = exts[st.ext];
      for (uint32_t w : e.writers) add(w);
      if (mode & 2u)
        for (uint32_t r : e.readers) add(r);
    }
  }

  void update(DepState &st, uint32_t t, uint32_t mode) {
    if (mode & 2u) {
      st.writer = t;
      st.ext = NONE;           // the DepExt entry is simply dropped
    } else {
      ext_of(st).readers.push_back(t);
    }
  }
};

// ---------------------------------------------------------------- merge --
template <class Par>
void Builder::merge(std::vector<Lane> &lanes, size_t nlanes, DepState *deps, Par &&par, int nworkers) {
  const size_t P = nlanes;
  std::vector<uint32_t> ibase(P), fbase(P);
  std::vector<size_t> ebase(P);
  size_t ni = items.size(), nf = fpool.size(), ne = edges.size();
  for (size_t p = 0; p < P; ++p) {
    ibase[p] = (uint32_t)ni;
    fbase[p] = (uint32_t)nf;
    ebase[p] = ne;
    ni += lanes[p].items.size();
    nf += lanes[p].fpool.size();
    ne += lanes[p].edges.size();
    fused += lanes[p].fused;
  }
  items.resize(ni);
  fpool.resize(nf);
  edges.resize(ne);
  par([&](int w) {
   for (size_t p = (size_t)w; p < P; p += (size_t)nworkers) {
    Lane &L = lanes[p];
    const uint32_t ib = ibase[p], fb = fbase[p];
    auto fix = [ib](uint32_t id) { return (id & TAG) && id != NONE ? ib + (id & ~TAG) : id; };
    if (!L.fpool.empty()) memcpy(&fpool[fb], L.fpool.data(), 4 * L.fpool.size());
    for (size_t j = 0; j < L.items.size(); ++j) {
      HItem it = L.items[j];
      if (it.fofs & TAG) it.fofs = fb + (it.fofs & ~TAG);
      items[ib + j] = it;
    }
    for (uint32_t w : L.relocated) items[w].fofs = fb + (items[w].fofs & ~TAG);
    uint64_t *E = edges.data() + ebase[p];
    for (size_t j = 0; j < L.edges.size(); ++j) {
      const uint64_t e = L.edges[j];
      E[j] = ((uint64_t)fix((uint32_t)(e >> 32)) << 32) | fix((uint32_t)e);
    }
    for (uint32_t s : L.touched) deps[s].writer = fix(deps[s].writer);
    if (record_tasks)
      for (uint64_t r : L.recorded) task_item[r >> 32] = fix((uint32_t)r);
   }
  });
}

// ------------------------------------------------------------ lane_runs --
template <class Loc, class SlotOf, class Geom>
void Builder::lane_runs(Lane &L, const LaneEntry *const *chunks, const uint32_t *const *ctasks, const size_t *counts,
                        int nchunks, DepState *deps, uint32_t nlocal, Loc &&loc, SlotOf &&slot_of, Geom &&geom) {
  L.clear();
  size_t n = 0;
  for (int c = 0; c < nchunks; ++c) n += counts[c];
  if (n == 0) return;
  L.cnt.assign(nlocal + 1, 0);
  uint32_t *cnt = L.cnt.data();
  for (int c = 0; c < nchunks; ++c)
    for (size_t j = 0; j < counts[c]; ++j) ++cnt[loc(chunks[c][j].slot) + 1];
  for (uint32_t l = 1; l <= nlocal; ++l) cnt[l] += cnt[l - 1];
  L.fpool.resize(n);
  if (record_tasks) L.tasks.resize(n);
  float *fs = L.fpool.data();
  for (int c = 0; c < nchunks; ++c)
    for (size_t j = 0; j < counts[c]; ++j) {
      const LaneEntry &e = chunks[c][j];
      const uint32_t pos = cnt[loc(e.slot)]++;
      memcpy(fs + pos, &e.fbits, 4);
      if (record_tasks) L.tasks[pos] = ctasks[c][j];
    }
  // now cnt[l] = end of run l; start of run l = cnt[l-1] (0 for l = 0)
  uint32_t b = 0;
  for (uint32_t l = 0; l < nlocal; ++l) {
    const uint32_t e_ = cnt[l];
    if (e_ == b) continue;
    const uint32_t s = slot_of(l);
    DepState &st = deps[s];
    fresh(st);
    const uint32_t m = e_ - b;
    uint32_t i = 0;
    uint32_t prev = NONE;
    if (fusion && st.ext == NONE && st.writer != NONE) {
      const uint32_t w = st.writer;   // global: this run is the slot's only one in the batch
      HItem &it = items[w];
      if (it.kind == 1 && it.slot0 == s && __atomic_load_n(&it.nsucc, __ATOMIC_RELAXED) == 0 && it.k < max_fused) {
        const uint32_t take = std::min(m, max_fused - it.k);
        if (!(it.fofs & TAG) && it.k + take <= it.fcap) {
          memcpy(&fpool[it.fofs + it.k], fs + b, 4ull * take);
        } else {
          const uint32_t cap = std::max<uint32_t>(8, 2 * (it.k + take));
          const uint32_t ofs = (uint32_t)L.fpool.size();
          L.fpool.resize(ofs + cap);
          fs = L.fpool.data();
          memcpy(fs + ofs, &fpool[it.fofs], 4ull * it.k);
          memcpy(fs + ofs + it.k, fs + b, 4ull * take);
          it.fofs = TAG | ofs;
          it.fcap = cap;
          L.relocated.push_back(w);
        }
        if (record_tasks)
          for (uint32_t q = 0; q < take; ++q) {
            task_item[L.tasks[b + q]] = w;
            task_pos[L.tasks[b + q]] = it.k + q;
          }
        it.k += take;
        i = take;
        L.fused += take;
        prev = w;
      }
    }
    const auto g = geom(s);
    auto chain_rest = [&]() {
      if (!(i < m && prev != NONE)) return;
      // the rest of the run: a chain of items, each the single successor of
      // the previous one (the common case: unfused sweeps, long fused runs);
      // written in place, no per-item vector growth
      const uint32_t step = fusion ? max_fused : 1u;
      const uint32_t cnt_items = (m - i + step - 1) / step;
      size_t li = L.items.size(), le = L.edges.size();
      L.items.resize(li + cnt_items);
      L.edges.resize(le + cnt_items);
      HItem *IT = L.items.data();
      uint64_t *ED = L.edges.data();
      if (prev & TAG) ++IT[prev & ~TAG].nsucc;
      else __atomic_fetch_add(&items[prev].nsucc, 1u, __ATOMIC_RELAXED);
      for (uint32_t q = 0; q < cnt_items; ++q, ++li, ++le) {
        const uint32_t take = std::min(m - i, step);
        const uint32_t t = TAG | (uint32_t)li;
        IT[li] = HItem{1, take, s, NONE, g.first, 0, g.second, 0, TAG | (b + i), take, 1, q + 1 < cnt_items ? 1u : 0u,
                       STAMP_NONE, 0};
        ED[le] = ((uint64_t)prev << 32) | t;
        if (record_tasks)
          for (uint32_t r = 0; r < take; ++r) {
            L.recorded.push_back(((uint64_t)L.tasks[b + i + r] << 32) | t);
            task_pos[L.tasks[b + i + r]] = r;
          }
        L.fused += take - 1;
        prev = t;
        i += take;
      }
    };
    chain_rest();
    while (i < m) {
      const uint32_t take = fusion ? std::min(m - i, max_fused) : 1u;
      const uint32_t local = (uint32_t)L.items.size();
      const uint32_t t = TAG | local;
      L.items.push_back(HItem{1, take, s, NONE, g.first, 0, g.second, 0, TAG | (b + i), take, 0, 0, STAMP_NONE, 0});
      uint32_t np = 0;
      auto link = [&](uint32_t p) {
        if (p & TAG) ++L.items[p & ~TAG].nsucc;
        else __atomic_fetch_add(&items[p].nsucc, 1u, __ATOMIC_RELAXED);
        // (a global predecessor whose operand has another base: as collect())
        if (!(p & TAG) && items[p].x != g.first && items[p].y != g.first) L.items[local].item_deps = 1;
        L.edges.push_back(((uint64_t)p << 32) | t);
        ++np;
      };
      if (prev != NONE) {
        link(prev);
      } else {
        // first item of the run: writer(s) and readers of the handle (W access)
        if (st.writer != NONE) link(st.writer);
        if (st.ext != NONE) {
          const DepExt &x = exts[st.ext];
          uint32_t seen_w = st.writer;
          for (uint32_t q : x.writers)
            if (q != seen_w) link(q);
          for (uint32_t q : x.readers) {
            bool dup = q == st.writer;
            for (uint32_t r : x.writers) dup |= (r == q);
            if (!dup) link(q);
          }
        }
      }
      L.items[local].npred = np;
      if (record_tasks)
        for (uint32_t q = 0; q < take; ++q) {
          L.recorded.push_back(((uint64_t)L.tasks[b + i + q] << 32) | t);
          task_pos[L.tasks[b + i + q]] = q;
        }
      L.fused += take - 1;
      prev = t;
      i += take;
      chain_rest();
    }
    st.writer = prev;
    st.ext = NONE;
    if (prev & TAG) L.touched.push_back(s);
    b = e_;
  }
}

// ------------------------------------------------------- direct rounds --
template <class Src, class Loc, class SlotOf, class Geom>
void Builder::lane_count(Lane &L, Src &&src, uint32_t nlocal, Loc &&loc, SlotOf &&slot_of, Geom &&geom) {
  L.hr.clear();
  L.reuse.clear();
  L.d_items = L.d_elems = L.d_work = L.d_fac = 0;
  L.d_tasks = 0;
  // src(visit): visit(slot, fbits) for each of the lane's tasks in stream
  // order (twice: a counting pass, then the scatter of the factors)
  L.cnt.assign(nlocal + 1, 0);
  uint32_t *cnt = L.cnt.data();
  src([&](uint32_t s, uint32_t) { ++cnt[loc(s) + 1]; });
  for (uint32_t l = 1; l <= nlocal; ++l) cnt[l] += cnt[l - 1];
  const size_t n = cnt[nlocal];
  L.d_tasks = n;
  if (n == 0) return;
  L.fpool.resize(n);
  float *fs = L.fpool.data();
  src([&](uint32_t s, uint32_t fb) { memcpy(fs + cnt[loc(s)]++, &fb, 4); });
  const uint32_t step = fusion ? max_fused : 1u;
  const float *pf = nullptr;   // the lane's previous list of > 1 factors
  uint32_t pk = 0;
  uint32_t b = 0;
  for (uint32_t l = 0; l < nlocal; ++l) {
    const uint32_t e = cnt[l];
    if (e == b) continue;
    const uint32_t m = e - b, s = slot_of(l);
    const uint32_t items = (m + step - 1) / step;
    L.hr.push_back(RunH{s, b, m, items});
    const uint64_t nx = geom(s).second;
    L.d_items += items;
    L.d_elems += (uint64_t)items * nx;
    L.d_work += (uint64_t)m * nx;
    for (uint32_t q = 0; q < items && step > 1; ++q) {
      const uint32_t take = std::min(step, m - q * step);
      if (take == 1) continue;
      const float *f = fs + b + q * step;
      const bool same = pf && pk == take && memcmp(pf, f, 4ull * take) == 0;
      L.reuse.push_back(same ? 1 : 0);
      if (!same) {
        L.d_fac += take;
        pf = f;
        pk = take;
      }
    }
    b = e;
  }
}

// item(id) -> DItem& of the epoch; ids are L.ibase + position; factor lists
// go to fac[L.fbase ...], the initially ready units to queue[L.qbase ...].
template <class Geom, class Item>
void Builder::lane_write(Lane &L, uint64_t chunk_elems, float *fac, unsigned long long *queue, Geom &&geom,
                         Item &&item) {
  const uint32_t step = fusion ? max_fused : 1u;
  const float *fs = L.fpool.data();
  uint32_t id = (uint32_t)L.ibase;
  uint32_t fo = (uint32_t)L.fbase, pfo = 0;
  uint64_t qi = L.qbase;
  size_t ri = 0;
  for (const RunH &h : L.hr) {
    const auto g = geom(h.slot);
    // the chain's first item starts ready: its units join the initial queue
    const uint32_t nc = units_of((uint32_t)g.second, chunk_elems);
    for (uint32_t c = 0; c < nc; ++c) queue[qi++] = ((unsigned long long)id << 32) | c;
    for (uint32_t q = 0; q < h.items; ++q, ++id) {
      const uint32_t take = std::min(step, h.m - q * step);
      const float *f = fs + h.start + q * step;
      const bool more = q + 1 < h.items;
      auto &d = item(id);
      d.x = g.first;
      d.y = 0;
      d.n = (uint32_t)g.second;
      d.meta = make_meta(K_SCAL, q > 0, take, more ? 1 : 0, false, g.second <= chunk_elems);
      if (take == 1) {
        memcpy(&d.arg, f, 4);
      } else {
        if (!L.reuse[ri++]) {
          memcpy(fac + fo, f, 4ull * take);
          pfo = fo;
          fo += take;
        }
        d.arg = pfo;
      }
      d.succ = more ? id + 1 : 0u;   // single successor inline
      // (pend[id] is not written: a chain item has one predecessor
      // (K_SINGLE_PRED), released without its counter)
    }
  }
}

}  // namespace bt
