// builder.cpp -- out-of-line parts of the dependency builder (builder.hpp).
#include "builder.hpp"

#include <algorithm>

namespace bt {

namespace {
void dedupe(std::vector<uint32_t> &v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
}
}  // namespace

void Builder::partition_state(DepState &parent, DepState *parts, uint32_t nparts) {
  fresh(parent);
  for (uint32_t i = 0; i < nparts; ++i) {
    DepState &c = parts[i];
    c.epoch = epoch;
    c.writer = parent.writer;
    c.ext = NONE;
    if (parent.ext != NONE) {   // private copy: parts gain readers independently
      const uint32_t id = (uint32_t)exts.size();
      exts.push_back(exts[parent.ext]);
      c.ext = id;
    }
  }
}

void Builder::unpartition_state(DepState &parent, DepState *parts, uint32_t nparts) {
  std::vector<uint32_t> w, r;
  for (uint32_t i = 0; i < nparts; ++i) {
    const DepState &c = parts[i];
    if (c.epoch != epoch) continue;
    if (c.writer != NONE) w.push_back(c.writer);
    if (c.ext != NONE) {
      const DepExt &e = exts[c.ext];
      w.insert(w.end(), e.writers.begin(), e.writers.end());
      r.insert(r.end(), e.readers.begin(), e.readers.end());
    }
  }
  dedupe(w);
  dedupe(r);
  parent.epoch = epoch;
  parent.writer = NONE;
  parent.ext = NONE;
  if (w.size() == 1) {
    parent.writer = w[0];
    w.clear();
  }
  if (!w.empty() || !r.empty()) {
    DepExt &e = ext_of(parent);
    e.writers = std::move(w);
    e.readers = std::move(r);
  }
}

namespace {
inline void lane_append(vec<float> &gpool, Lane &L, HItem &it, uint32_t fbits, uint32_t w, bool global) {
  if (it.fofs & TAG) {
    uint32_t ofs = it.fofs & ~TAG;
    if (it.k == it.fcap) {
      const uint32_t cap = it.fcap * 2;
      const uint32_t n = (uint32_t)L.fpool.size();
      L.fpool.resize(n + cap);
      memmove(&L.fpool[n], &L.fpool[ofs], 4ull * it.k);
      ofs = n;
      it.fofs = TAG | n;
      it.fcap = cap;
    }
    memcpy(&L.fpool[ofs + it.k], &fbits, 4);
  } else if (it.k < it.fcap) {          // global item, room in its global region
    memcpy(&gpool[it.fofs + it.k], &fbits, 4);
  } else {                              // global item, full: move it to the lane pool
    const uint32_t cap = std::max<uint32_t>(8, it.fcap * 2);
    const uint32_t n = (uint32_t)L.fpool.size();
    L.fpool.resize(n + cap);
    memcpy(&L.fpool[n], &gpool[it.fofs], 4ull * it.k);
    memcpy(&L.fpool[n + it.k], &fbits, 4);
    it.fofs = TAG | n;
    it.fcap = cap;
    if (global) L.relocated.push_back(w);
  }
  ++it.k;
}
}  // namespace

void Builder::lane_scal(Lane &L, DepState &st, const LaneEntry &e, uint64_t x, uint64_t n) {
  fresh(st);
  const uint32_t s = e.slot;
  if (fusion && st.ext == NONE && st.writer != NONE) {
    const uint32_t w = st.writer;
    if (w & TAG) {
      HItem &it = L.items[w & ~TAG];   // lane items are SCALs on this slot
      if (it.nsucc == 0 && it.k < max_fused) {
        lane_append(fpool, L, it, e.fbits, w, false);
        if (record_tasks) {
          L.recorded.push_back(((uint64_t)e.task << 32) | w);
          task_pos[e.task] = it.k - 1;
        }
        ++L.fused;
        return;
      }
    } else {
      HItem &it = items[w];
      if (it.kind == 1 && it.slot0 == s && __atomic_load_n(&it.nsucc, __ATOMIC_RELAXED) == 0 &&
          it.k < max_fused) {
        lane_append(fpool, L, it, e.fbits, w, true);
        if (record_tasks) {
          task_item[e.task] = w;
          task_pos[e.task] = it.k - 1;
        }
        ++L.fused;
        return;
      }
    }
  }
  const uint32_t local = (uint32_t)L.items.size();
  const uint32_t t = TAG | local;
  const uint32_t fo = (uint32_t)L.fpool.size();
  L.fpool.resize(fo + 8);
  memcpy(&L.fpool[fo], &e.fbits, 4);
  L.items.push_back(HItem{1, 1, s, NONE, x, 0, n, 0, TAG | fo, 8, 0, 0, NONE});
  // predecessors: writer(s) and readers (W access), deduplicated
  uint32_t pbuf[8];
  std::vector<uint32_t> pv;
  uint32_t np = 0;
  auto add = [&](uint32_t p) {
    for (uint32_t i = 0; i < np && i < 8; ++i)
      if (pbuf[i] == p) return;
    if (np >= 8)
      for (uint32_t q : pv)
        if (q == p) return;
    if (np < 8) pbuf[np] = p;
    else pv.push_back(p);
    ++np;
  };
  if (st.writer != NONE) add(st.writer);
  if (st.ext != NONE) {
    const DepExt &x2 = exts[st.ext];
    for (uint32_t q : x2.writers) add(q);
    for (uint32_t q : x2.readers) add(q);
  }
  for (uint32_t i = 0; i < np; ++i) {
    const uint32_t p = i < 8 ? pbuf[i] : pv[i - 8];
    if (p & TAG) ++L.items[p & ~TAG].nsucc;
    else __atomic_fetch_add(&items[p].nsucc, 1u, __ATOMIC_RELAXED);
    L.edges.push_back(((uint64_t)p << 32) | t);
  }
  L.items[local].npred = np;
  st.writer = t;
  st.ext = NONE;
  L.touched.push_back(s);
  if (record_tasks) {
    L.recorded.push_back(((uint64_t)e.task << 32) | t);
    task_pos[e.task] = 0;
  }
}

}  // namespace bt
