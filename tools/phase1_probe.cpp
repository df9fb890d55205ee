// Host probe: cost of the builder's phase 1 (validate + bucket a 1 M-task
// SCAL run by (round, lane)) on this machine's cores, against a plain
// streaming read of the same task arrays.  Mirrors scal_run_parallel's loop
// shape without the runtime (no GPU needed).
//
//   g++ -O2 -std=c++17 -pthread tools/phase1_probe.cpp -o /tmp/phase1_probe && /tmp/phase1_probe
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <functional>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

struct SlotHot {
  uint32_t gen, flags;
  int32_t rank;
  uint32_t grp;
  float *dptr;
  uint64_t nx;
};
struct Entry {
  uint32_t slot, fbits;
};

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Team {
  int n;
  std::vector<std::thread> th;
  std::atomic<uint64_t> gen{0};
  std::atomic<int> left{0};
  std::function<void(int)> job;
  bool stop = false;
  explicit Team(int n_) : n(n_) {
    for (int i = 1; i < n; ++i)
      th.emplace_back([this, i] {
        uint64_t seen = 0;
        for (;;) {
          uint64_t g;
          while ((g = gen.load(std::memory_order_acquire)) == seen) {
          }
          seen = g;
          if (stop) return;
          job(i);
          left.fetch_sub(1, std::memory_order_acq_rel);
        }
      });
  }
  template <class F>
  void run(F &&f) {
    job = f;
    left.store(n - 1);
    gen.fetch_add(1, std::memory_order_release);
    job(0);
    while (left.load(std::memory_order_acquire)) {
    }
  }
  ~Team() {
    stop = true;
    gen.fetch_add(1);
    for (auto &t : th) t.join();
  }
};

int main(int argc, char **argv) {
  const bool flush = argc > 1;   // evict the caches before each timed pass (as between builder steps)
  std::vector<uint64_t> junk(flush ? (256u << 20) / 8 : 0, 1);
  const size_t N = 1 << 20, S = 16384;
  const int R = 8;
  std::vector<uint64_t> h(N);
  std::vector<float> sc(N);
  std::vector<int32_t> cl(N, 1);
  std::vector<SlotHot> hot(S + 1);
  for (size_t s = 0; s <= S; ++s) hot[s] = {1, 1, 0, 0, nullptr, 64};
  for (size_t j = 0; j < N; ++j) {
    h[j] = (1ull << 32) | (1 + j % S + 1);
    sc[j] = 1.0f + j % 7;
  }
  for (int T : {1, 2, 4, 8, 12, 14, 16}) {
    const uint32_t G = (uint32_t)(T * R);
    for (size_t s = 1; s <= S; ++s) hot[s].grp = (uint32_t)(((s - 1) * R / S) * T + ((s - 1) >> 6) % T);
    std::vector<std::vector<std::vector<Entry>>> buckets(T, std::vector<std::vector<Entry>>(G));
    for (auto &b : buckets)
      for (auto &v : b) v.reserve(2 * N / (T * G) + 64);
    Team team(T);
    std::vector<uint64_t> sink(T * 8);
    double best_h = 1e9, best_b = 1e9, best_r = 1e9, best_l = 1e9, best_v = 1e9;
    std::vector<uint64_t> key(S + 1);
    for (size_t s = 0; s <= S; ++s) key[s] = (1ull << 32) | (uint64_t)hot[s].grp << 1 | 1u;
    std::vector<std::vector<Entry *>> curs(T, std::vector<Entry *>(G)), ends(T, std::vector<Entry *>(G));
    for (int rep = 0; rep < 30; ++rep) {
      if (flush) {
        team.run([&](int c) {
          const size_t lo = junk.size() * c / T, hi = junk.size() * (c + 1) / T;
          for (size_t i = lo; i < hi; i += 8) junk[i] += 1;
        });
      }
      double t0 = now_ms();
      team.run([&](int c) {
        size_t lo = N * c / T, hi = N * (c + 1) / T;
        auto &mine = buckets[c];
        for (auto &v : mine) v.clear();
        for (size_t j = lo; j < hi; ++j) {
          const uint32_t s = (uint32_t)h[j] - 1u;
          if (cl[j] != 1 || s >= hot.size()) std::abort();
          const SlotHot &sh = hot[s];
          if (sh.gen != (uint32_t)(h[j] >> 32) || sh.flags != 1 || sh.rank != 0) std::abort();
          Entry e;
          e.slot = s;
          memcpy(&e.fbits, &sc[j], 4);
          mine[sh.grp].push_back(e);
        }
      });
      const double e0 = now_ms();
      if (flush) team.run([&](int c) {
          const size_t lo = junk.size() * c / T, hi = junk.size() * (c + 1) / T;
          for (size_t i = lo; i < hi; i += 8) junk[i] += 1;
        });
      double t1 = now_ms();
      // lean variant: one packed 8-byte key per slot (gen | grp | ok bit),
      // raw bucket cursors
      team.run([&](int c) {
        size_t lo = N * c / T, hi = N * (c + 1) / T;
        Entry **cur = curs[c].data();
        Entry **end = ends[c].data();
        const uint64_t *kt = key.data();
        const size_t nk = key.size();
        for (uint32_t g = 0; g < G; ++g) cur[g] = buckets[c][g].data(), end[g] = cur[g] + buckets[c][g].capacity();
        uint32_t badc = 0;
        for (size_t j = lo; j < hi; ++j) {
          const uint64_t hj = h[j];
          const uint32_t s = (uint32_t)hj - 1u;
          const uint64_t k = s < nk ? kt[s] : 0;
          badc |= (uint32_t)(cl[j] != 1) | (uint32_t)((k >> 32) != (hj >> 32)) | (uint32_t)(k & 1) ^ 1u;
          const uint32_t g = (uint32_t)k >> 1;
          Entry *p = cur[g];
          p->slot = s;
          memcpy(&p->fbits, &sc[j], 4);
          cur[g] = p + 1;
          if (__builtin_expect(p + 1 == end[g], 0)) std::abort();
        }
        if (badc) std::abort();
      });
      const double e1 = now_ms();
      if (flush) team.run([&](int c) {
          const size_t lo = junk.size() * c / T, hi = junk.size() * (c + 1) / T;
          for (size_t i = lo; i < hi; i += 8) junk[i] += 1;
        });
      double t1b = now_ms();
      // validate + group only (no bucket stores)
      team.run([&](int c) {
        size_t lo = N * c / T, hi = N * (c + 1) / T;
        const uint64_t *kt = key.data();
        const size_t nk = key.size();
        uint32_t badc = 0, gs = 0;
        for (size_t j = lo; j < hi; ++j) {
          const uint64_t hj = h[j];
          const uint32_t s = (uint32_t)hj - 1u;
          const uint64_t k = s < nk ? kt[s] : 0;
          badc |= (uint32_t)(cl[j] != 1) | (uint32_t)((k >> 32) != (hj >> 32)) | (uint32_t)(k & 1) ^ 1u;
          gs += (uint32_t)k >> 1;
        }
        if (badc) std::abort();
        sink[c * 8 + 1] = gs;
      });
      const double e2 = now_ms();
      // validate + run records with the full SlotHot table (the runtime's phase 1)
      double t3 = now_ms();
      team.run([&](int c) {
        size_t lo = N * c / T, hi = N * (c + 1) / T;
        uint32_t badc = 0, cur = ~0u, nr = 0;
        for (size_t j = lo; j < hi; ++j) {
          const uint32_t s = (uint32_t)h[j] - 1u;
          if (cl[j] != 1 || s >= hot.size()) std::abort();
          const SlotHot &sh = hot[s];
          badc |= (sh.gen != (uint32_t)(h[j] >> 32)) | (sh.flags != 1) | (sh.rank != 0);
          if (sh.grp != cur) { cur = sh.grp; ++nr; }
        }
        if (badc) std::abort();
        sink[c * 8 + 2] = nr;
      });
      const double e3 = now_ms();
      if (rep > 3) best_h = std::min(best_h, e3 - t3);
      if (flush) team.run([&](int c) {
          const size_t lo = junk.size() * c / T, hi = junk.size() * (c + 1) / T;
          for (size_t i = lo; i < hi; i += 8) junk[i] += 1;
        });
      double t1c = now_ms();
      team.run([&](int c) {
        size_t lo = N * c / T, hi = N * (c + 1) / T;
        uint64_t acc = 0;
        for (size_t j = lo; j < hi; ++j) acc += h[j] + (uint32_t)cl[j] + (uint64_t)sc[j];
        sink[c * 8] = acc;
      });
      double t2 = now_ms();
      if (rep > 3) {
        best_b = std::min(best_b, e0 - t0);
        best_l = std::min(best_l, e1 - t1);
        best_v = std::min(best_v, e2 - t1b);
        best_r = std::min(best_r, t2 - t1c);
      }
    }
    printf("{\"threads\": %d, \"bucket_ms\": %.3f, \"lean_bucket_ms\": %.3f, \"validate_ms\": %.3f, \"stream_read_ms\": %.3f, \"slothot_runs_ms\": %.3f}\n",
           T, best_b, best_l, best_v, best_r, best_h);
  }
  return 0;
}
