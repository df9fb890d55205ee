// builder.cpp -- out-of-line parts of the dependency builder (builder.hpp).
#include "builder.hpp"

#include <algorithm>

namespace bt {

void Builder::dedupe(std::vector<uint32_t> &v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
}

}  // namespace bt
