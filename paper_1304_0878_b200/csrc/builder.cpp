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

}  // namespace bt
