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
// parent's state to the union of its parts' states (reading R9) -- so no
// barrier task is needed and tiles stay independent.
//
// Vertical fusion (BASELINE north_star: "a fused pass over consecutive inout
// scalings of the same tile"): a SCAL(RW) whose only predecessor is the
// current single writer W of its handle, where W is a SCAL item of this epoch
// on the same handle with no successor yet, is appended to W's factor list
// instead of becoming a new item.  Factor lists are stored as a trie of
// (parent, factor) nodes so that the tiles of a sweep-major stream share one
// list (C5: 16,384 items, one 64-factor list).
#pragma once
#include <stdint.h>

#include <vector>

namespace bt {

constexpr uint32_t NONE = 0xFFFFFFFFu;

struct DepState {
  uint32_t epoch = NONE;           // states of older epochs are empty
  uint32_t writer = NONE;          // single latest writer (common case)
  std::vector<uint32_t> writers;   // >1 latest writers (after unpartition)
  std::vector<uint32_t> readers;
  void reset(uint32_t e) {
    epoch = e;
    writer = NONE;
    writers.clear();
    readers.clear();
  }
};

struct HItem {
  uint32_t kind;
  uint32_t k;          // tasks in this item
  uint32_t slot0, slot1;
  uint64_t x, y, n;    // device addresses / elements
  uint32_t arg;        // AXPY scalar bits; SCAL: trie node of the factor list
  uint32_t npred;
  uint32_t nsucc;
  uint32_t stamp;      // dedupe marker (id of the item being built)
};

struct TrieNode {
  uint32_t parent;
  uint32_t fbits;
  uint32_t child;      // first child created (memo), NONE if none
  uint32_t child_fbits;
};

struct Access {
  uint32_t slot;
  uint32_t mode;       // BT_R | BT_W bits
};

class Builder {
 public:
  // Epoch-scoped outputs
  std::vector<HItem> items;
  std::vector<uint64_t> edges;      // (pred << 32) | succ, in creation order
  std::vector<TrieNode> nodes;      // factor trie; node 0 is the root
  std::vector<uint32_t> task_item;  // per epoch task (only if record_tasks)
  std::vector<uint32_t> task_pos;
  uint64_t ntasks = 0;              // tasks of this epoch (local or not)
  uint64_t fused = 0;
  bool record_tasks = false;
  bool fusion = true;
  uint32_t max_fused = 256;
  uint32_t epoch = 0;

  Builder() { clear(); }

  void clear() {
    items.clear();
    edges.clear();
    nodes.clear();
    nodes.push_back(TrieNode{NONE, 0, NONE, 0});
    task_item.clear();
    task_pos.clear();
    ntasks = 0;
    fused = 0;
  }

  void next_epoch() {
    clear();
    ++epoch;
  }

  // Record a task executed on another rank (kept for the task->item map).
  void add_remote() {
    if (record_tasks) {
      task_item.push_back(NONE);
      task_pos.push_back(0);
    }
    ++ntasks;
  }

  // SCAL(f; x:RW) on leaf slot s (x = device address of element 0, n elems).
  void add_scal(DepState &st, uint32_t s, uint64_t x, uint64_t n, uint32_t fbits) {
    fresh(st);
    if (fusion && st.readers.empty() && st.writers.empty() && st.writer != NONE) {
      HItem &w = items[st.writer];
      if (w.kind == 1 && w.slot0 == s && w.nsucc == 0 && w.k < max_fused) {
        w.arg = child(w.arg, fbits);
        if (record_tasks) {
          task_item.push_back(st.writer);
          task_pos.push_back(w.k);
        }
        ++w.k;
        ++fused;
        ++ntasks;
        return;
      }
    }
    const uint32_t t = new_item(1, s, NONE, x, 0, n, child(0, fbits));
    depend_write(st, t);
    st.writer = t;
  }

  // Generic task with up to two accesses (AXPY: x R, y RW; COPY: x R, y W).
  void add_task(uint32_t kind, DepState *st0, const Access &a0, DepState *st1, const Access &a1, uint64_t x,
                uint64_t y, uint64_t n, uint32_t arg) {
    fresh(*st0);
    if (st1 != st0) fresh(*st1);
    const uint32_t t = new_item(kind, a0.slot, a1.slot, x, y, n, arg);
    if (st1 == st0) {  // same handle twice: modes OR-ed (reading R6)
      const uint32_t m = a0.mode | a1.mode;
      apply(*st0, t, m);
    } else {
      // collect all predecessors first, then update the states
      collect(*st0, t, a0.mode);
      collect(*st1, t, a1.mode);
      update(*st0, t, a0.mode);
      update(*st1, t, a1.mode);
    }
  }

  // Partition: every part inherits the parent's state (reading R9).
  void partition_state(DepState &parent, DepState *parts, uint32_t nparts) {
    fresh(parent);
    for (uint32_t i = 0; i < nparts; ++i) {
      DepState &c = parts[i];
      c.reset(epoch);
      c.writer = parent.writer;
      c.writers = parent.writers;
      c.readers = parent.readers;
    }
  }

  // Unpartition: the parent's writers/readers are the union over the parts.
  void unpartition_state(DepState &parent, DepState *parts, uint32_t nparts) {
    parent.reset(epoch);
    std::vector<uint32_t> w, r;
    for (uint32_t i = 0; i < nparts; ++i) {
      DepState &c = parts[i];
      if (c.epoch != epoch) continue;
      if (c.writer != NONE) w.push_back(c.writer);
      w.insert(w.end(), c.writers.begin(), c.writers.end());
      r.insert(r.end(), c.readers.begin(), c.readers.end());
    }
    dedupe(w);
    dedupe(r);
    if (w.size() == 1) parent.writer = w[0];
    else parent.writers = std::move(w);
    parent.readers = std::move(r);
  }

 private:
  void fresh(DepState &st) {
    if (st.epoch != epoch) st.reset(epoch);
  }

  static void dedupe(std::vector<uint32_t> &v);

  uint32_t child(uint32_t parent, uint32_t fbits) {
    TrieNode &p = nodes[parent];
    if (p.child != NONE && p.child_fbits == fbits) return p.child;
    const uint32_t id = (uint32_t)nodes.size();
    if (p.child == NONE) {
      p.child = id;
      p.child_fbits = fbits;
    }
    nodes.push_back(TrieNode{parent, fbits, NONE, 0});
    return id;
  }

  uint32_t new_item(uint32_t kind, uint32_t s0, uint32_t s1, uint64_t x, uint64_t y, uint64_t n, uint32_t arg) {
    const uint32_t t = (uint32_t)items.size();
    items.push_back(HItem{kind, 1, s0, s1, x, y, n, arg, 0, 0, NONE});
    if (record_tasks) {
      task_item.push_back(t);
      task_pos.push_back(0);
    }
    ++ntasks;
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

  void collect(DepState &st, uint32_t t, uint32_t mode) {
    if (st.writer != NONE) edge(st.writer, t);
    for (uint32_t w : st.writers) edge(w, t);
    if (mode & 2u)
      for (uint32_t r : st.readers) edge(r, t);
  }

  void update(DepState &st, uint32_t t, uint32_t mode) {
    if (mode & 2u) {
      st.writer = t;
      st.writers.clear();
      st.readers.clear();
    } else {
      st.readers.push_back(t);
    }
  }

  void apply(DepState &st, uint32_t t, uint32_t mode) {
    collect(st, t, mode);
    update(st, t, mode);
  }

  void depend_write(DepState &st, uint32_t t) {
    collect(st, t, 3u);
    st.writers.clear();
    st.readers.clear();
  }
};

}  // namespace bt
