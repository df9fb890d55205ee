// scheduler.cu -- the persistent sm_100a scheduler kernel and its task bodies.
//
// One launch executes one epoch: a DAG of work items built on the host from
// the submission order (runtime.cpp).  Each resident CTA is warp-specialised:
//
//   warp 0 (scheduler)   pop     t = atomicAdd(head, 1); spin on ld.acquire
//                                (queue[t]) until the unit (item, chunk) is
//                                published; t >= total_units ends the CTA.
//                        stage   copy the item's factor list to shared memory
//                        release when an item's last chunk is done, decrement
//                                each successor's pending counter; a successor
//                                reaching 0 is ready: its chunks are appended
//                                to the queue (atomicAdd(tail), fence.acq_rel,
//                                relaxed stores).
//   warps 1..8 (compute) run the task body on the unit's elements:
//            SCAL   x[i] = x[i]*f_1*...*f_k   (k sequential RN multiplies in
//                   submission order: PAPER.md:157-158; a fused chain of k
//                   vector_scal tasks is exactly k roundings per element)
//            AXPY   y[i] = fl(fl(a*x[i]) + y[i])
//            COPY   y[i] = x[i]
//
// The two roles exchange units through two shared-memory slots: FULL[b] is a
// named barrier (scheduler -> compute), EMPTY[b] an mbarrier the scheduler
// polls without blocking (compute -> scheduler).  Popping unit u+1 and
// releasing unit u-1 overlap the body of unit u, so the scheduling cost
// leaves the critical path of a busy CTA; while spinning for a not yet
// published unit the scheduler keeps releasing the units its CTA finishes.
//
// This is StarPU's "scheduler's queue" moved on-device:
// dependencies inferred at submission become per-item
// counters, and a completed task releases its successors without a host
// round trip.  Ready order is FIFO by publication.
//
// Data accesses are 256-bit (ld/st.global.cg.v8.f32 -> LDG/STG.E.ENL2.256),
// L2-only (data is produced by other CTAs of the same launch, so L1 must not
// hold it), coalesced: consecutive threads touch consecutive 32-byte sectors.
// All arithmetic is IEEE binary32 round-to-nearest (__fmul_rn/__fmul2_rn/
// __fadd_rn; the library is also built with -fmad=false), no FTZ.
#include <cuda_runtime.h>
#include <stdint.h>

#include "device_abi.h"

namespace bt {

// Two kernel variants share one block size (288 threads, 3 CTAs per SM):
//  "sw" (single scheduler warp + 8 compute warps, 2 slots): best for large
//       work units (FP32- or HBM-bound bodies; C3, C5);
//  "rw" (pop warp + release warp + 7 compute warps, 4 slots): best for small
//       units where scheduling dominates (C2, C4).
constexpr int kBlock = 288;
constexpr int kComputeSW = 256, kSlotsSW = 2;
constexpr int kComputeRW = 224, kSlotsRW = 4;
constexpr int kMaxFactors = 1024;              // upper bound of bt_config.max_fused
constexpr unsigned long long kStop = ~0ull - 1;
// named barrier ids (0 is __syncthreads): FULL[slot] = 1 + slot
constexpr int kBarFull = 1;
constexpr int kBarCompute = 5;   // the rw kernel's compute warps only (in-slot continuation)

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Named barriers with immediate ids (a register id makes ptxas reserve all 16
// hardware barriers and caps the CTAs per SM).
template <int ID>
__device__ __forceinline__ void bar_sync_n(int n) {
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "r"(n) : "memory");
}
template <int ID>
__device__ __forceinline__ void bar_arrive_n(int n) {
  asm volatile("bar.arrive %0, %1;" ::"n"(ID), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_sync(int id, int n) {
  switch (id) {
    case 1: bar_sync_n<1>(n); break;
    case 2: bar_sync_n<2>(n); break;
    case 3: bar_sync_n<3>(n); break;
    default: bar_sync_n<4>(n); break;
  }
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  switch (id) {
    case 1: bar_arrive_n<1>(n); break;
    case 2: bar_arrive_n<2>(n); break;
    case 3: bar_arrive_n<3>(n); break;
    default: bar_arrive_n<4>(n); break;
  }
}

// ---- 256-bit global accesses, cached in L2 only --------------------------
__device__ __forceinline__ void ld8(const float *p, float (&r)[8]) {
  asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]),
                 "=f"(r[7])
               : "l"(p)
               : "memory");
}
__device__ __forceinline__ void st8(float *p, const float (&r)[8]) {
  asm volatile("st.global.cg.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r[0]), "f"(r[1]),
               "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
               : "memory");
}

// ---- SCAL chain: v <- v * f_0 * f_1 * ... * f_{k-1}, one rounding each ----
// Packed FMUL2 (per-lane identical to __fmul_rn) halves the instruction count;
// the factor order is the submission order, never reassociated.
template <int NV>
__device__ __forceinline__ void chain_apply(float (&v)[NV][8], const float *sf, uint32_t k) {
  uint32_t j = 0;
#ifndef BT_TRACE_DETAIL
#define BT_TRACE_DETAIL 0
#endif
#ifndef BT_FACTOR_UNROLL16
#define BT_FACTOR_UNROLL16 1
#endif
#if BT_FACTOR_UNROLL16
  for (; j + 16 <= k; j += 16) {
    const float4 f4a = *reinterpret_cast<const float4 *>(sf + j);
    const float4 f4b = *reinterpret_cast<const float4 *>(sf + j + 4);
    const float4 f4c = *reinterpret_cast<const float4 *>(sf + j + 8);
    const float4 f4d = *reinterpret_cast<const float4 *>(sf + j + 12);
    const float fs[16] = {f4a.x, f4a.y, f4a.z, f4a.w, f4b.x, f4b.y, f4b.z, f4b.w,
                          f4c.x, f4c.y, f4c.z, f4c.w, f4d.x, f4d.y, f4d.z, f4d.w};
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const float2 ff = make_float2(fs[jj], fs[jj]);
#pragma unroll
      for (int a = 0; a < NV; ++a)
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          const float2 t = __fmul2_rn(make_float2(v[a][q], v[a][q + 1]), ff);
          v[a][q] = t.x;
          v[a][q + 1] = t.y;
        }
    }
  }
#endif
  for (; j + 8 <= k; j += 8) {
    const float4 f4a = *reinterpret_cast<const float4 *>(sf + j);
    const float4 f4b = *reinterpret_cast<const float4 *>(sf + j + 4);
    const float fs[8] = {f4a.x, f4a.y, f4a.z, f4a.w, f4b.x, f4b.y, f4b.z, f4b.w};
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const float2 ff = make_float2(fs[jj], fs[jj]);
#pragma unroll
      for (int a = 0; a < NV; ++a)
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          const float2 t = __fmul2_rn(make_float2(v[a][q], v[a][q + 1]), ff);
          v[a][q] = t.x;
          v[a][q + 1] = t.y;
        }
    }
  }
  for (; j + 4 <= k; j += 4) {
    const float4 f4 = *reinterpret_cast<const float4 *>(sf + j);
    const float fs[4] = {f4.x, f4.y, f4.z, f4.w};
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const float2 ff = make_float2(fs[jj], fs[jj]);
#pragma unroll
      for (int a = 0; a < NV; ++a)
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          const float2 t = __fmul2_rn(make_float2(v[a][q], v[a][q + 1]), ff);
          v[a][q] = t.x;
          v[a][q + 1] = t.y;
        }
    }
  }
  for (; j < k; ++j) {
    const float2 ff = make_float2(sf[j], sf[j]);
#pragma unroll
    for (int a = 0; a < NV; ++a)
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        const float2 t = __fmul2_rn(make_float2(v[a][q], v[a][q + 1]), ff);
        v[a][q] = t.x;
        v[a][q + 1] = t.y;
      }
  }
}

__device__ __forceinline__ float chain_scalar(float v, const float *sf, uint32_t k) {
  for (uint32_t j = 0; j < k; ++j) v = __fmul_rn(v, sf[j]);
  return v;
}

// Elements before the first 32-byte boundary of p (p is 4-byte aligned).
__device__ __forceinline__ uint64_t head_elems(const float *p, uint64_t n) {
  const uint64_t h = ((32u - (reinterpret_cast<uintptr_t>(p) & 31u)) & 31u) >> 2;
  return h < n ? h : n;
}

template <int U, int C>
__device__ void scal_range(float *x, uint64_t n, const float *sf, uint32_t k, int tid) {
  const uint64_t head = head_elems(x, n);
  for (uint64_t i = tid; i < head; i += C) __stcg(x + i, chain_scalar(__ldcg(x + i), sf, k));
  float *xv = x + head;
  const uint64_t nv = (n - head) >> 3;
  uint64_t i = tid;
  for (; i + (U - 1) * C < nv; i += U * C) {
    float v[U][8];
#pragma unroll
    for (int a = 0; a < U; ++a) ld8(xv + 8 * (i + a * C), v[a]);
    chain_apply<U>(v, sf, k);
#pragma unroll
    for (int a = 0; a < U; ++a) st8(xv + 8 * (i + a * C), v[a]);
  }
  for (; i < nv; i += C) {
    float v[1][8];
    ld8(xv + 8 * i, v[0]);
    chain_apply<1>(v, sf, k);
    st8(xv + 8 * i, v[0]);
  }
  for (uint64_t t = head + 8 * nv + tid; t < n; t += C) __stcg(x + t, chain_scalar(__ldcg(x + t), sf, k));
}

// Software-pipelined variant: the next step's U vectors are loaded before the
// current step's multiplies, so a warp never waits for a load at a step start
// (two register sets, A and B, alternate; U = 2 keeps them within the budget).
template <int U, int C>
__device__ void scal_range_pf(float *x, uint64_t n, const float *sf, uint32_t k, int tid) {
  const uint64_t head = head_elems(x, n);
  for (uint64_t i = tid; i < head; i += C) __stcg(x + i, chain_scalar(__ldcg(x + i), sf, k));
  float *xv = x + head;
  const uint64_t nv = (n - head) >> 3;
  uint64_t i = tid;
  if (i + (U - 1) * C < nv) {
    float a[U][8], b[U][8];
#pragma unroll
    for (int q = 0; q < U; ++q) ld8(xv + 8 * (i + q * C), a[q]);
    for (;;) {
      // A holds step i; prefetch step i + U*C into B
      uint64_t j = i + U * C;
      bool more = j + (U - 1) * C < nv;
      if (more) {
#pragma unroll
        for (int q = 0; q < U; ++q) ld8(xv + 8 * (j + q * C), b[q]);
      }
      chain_apply<U>(a, sf, k);
#pragma unroll
      for (int q = 0; q < U; ++q) st8(xv + 8 * (i + q * C), a[q]);
      i = j;
      if (!more) break;
      // B holds step i; prefetch into A
      j = i + U * C;
      more = j + (U - 1) * C < nv;
      if (more) {
#pragma unroll
        for (int q = 0; q < U; ++q) ld8(xv + 8 * (j + q * C), a[q]);
      }
      chain_apply<U>(b, sf, k);
#pragma unroll
      for (int q = 0; q < U; ++q) st8(xv + 8 * (i + q * C), b[q]);
      i = j;
      if (!more) break;
    }
  }
  for (; i < nv; i += C) {
    float v[1][8];
    ld8(xv + 8 * i, v[0]);
    chain_apply<1>(v, sf, k);
    st8(xv + 8 * i, v[0]);
  }
  for (uint64_t t = head + 8 * nv + tid; t < n; t += C) __stcg(x + t, chain_scalar(__ldcg(x + t), sf, k));
}

// AXPY: y[i] = fl(fl(a*x[i]) + y[i]) (two roundings, no FFMA).
__device__ __forceinline__ float axpy1(float a, float x, float y) { return __fadd_rn(__fmul_rn(a, x), y); }

template <int C>
__device__ void axpy_range(const float *x, float *y, uint64_t n, float a, int tid) {
  if (((reinterpret_cast<uintptr_t>(x) ^ reinterpret_cast<uintptr_t>(y)) & 31u) != 0) {
    for (uint64_t i = tid; i < n; i += C) __stcg(y + i, axpy1(a, __ldcg(x + i), __ldcg(y + i)));
    return;
  }
  const uint64_t head = head_elems(y, n);
  for (uint64_t i = tid; i < head; i += C) __stcg(y + i, axpy1(a, __ldcg(x + i), __ldcg(y + i)));
  const float *xv = x + head;
  float *yv = y + head;
  const uint64_t nv = (n - head) >> 3;
  uint64_t i = tid;
  // two vectors of x and y per step: 128 bytes of loads in flight per thread
  // (the accesses are asm volatile: the compiler does not overlap iterations);
  // CTA-wide bodies only (the warp-wide "wq" bodies stay within 64 registers)
  if constexpr (C >= 128)
  for (; i + C < nv; i += 2 * C) {
    float xr[2][8], yr[2][8];
    ld8(xv + 8 * i, xr[0]);
    ld8(xv + 8 * (i + C), xr[1]);
    ld8(yv + 8 * i, yr[0]);
    ld8(yv + 8 * (i + C), yr[1]);
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
      for (int q = 0; q < 8; ++q) yr[v][q] = axpy1(a, xr[v][q], yr[v][q]);
    st8(yv + 8 * i, yr[0]);
    st8(yv + 8 * (i + C), yr[1]);
  }
  for (; i < nv; i += C) {
    float xr[8], yr[8];
    ld8(xv + 8 * i, xr);
    ld8(yv + 8 * i, yr);
#pragma unroll
    for (int q = 0; q < 8; ++q) yr[q] = axpy1(a, xr[q], yr[q]);
    st8(yv + 8 * i, yr);
  }
  for (uint64_t t = head + 8 * nv + tid; t < n; t += C) __stcg(y + t, axpy1(a, __ldcg(x + t), __ldcg(y + t)));
}

template <int C>
__device__ void copy_range(const float *x, float *y, uint64_t n, int tid) {
  if (x == y) return;
  if (((reinterpret_cast<uintptr_t>(x) ^ reinterpret_cast<uintptr_t>(y)) & 31u) != 0) {
    for (uint64_t i = tid; i < n; i += C) __stcg(y + i, __ldcg(x + i));
    return;
  }
  const uint64_t head = head_elems(y, n);
  for (uint64_t i = tid; i < head; i += C) __stcg(y + i, __ldcg(x + i));
  const float *xv = x + head;
  float *yv = y + head;
  const uint64_t nv = (n - head) >> 3;
  uint64_t i = tid;
  // four vectors per step: 128 bytes of loads in flight per thread (CTA-wide bodies)
  if constexpr (C >= 128)
  for (; i + 3 * C < nv; i += 4 * C) {
    float a[8], b[8], c[8], d[8];
    ld8(xv + 8 * i, a);
    ld8(xv + 8 * (i + C), b);
    ld8(xv + 8 * (i + 2 * C), c);
    ld8(xv + 8 * (i + 3 * C), d);
    st8(yv + 8 * i, a);
    st8(yv + 8 * (i + C), b);
    st8(yv + 8 * (i + 2 * C), c);
    st8(yv + 8 * (i + 3 * C), d);
  }
  for (; i + C < nv; i += 2 * C) {
    float a[8], b[8];
    ld8(xv + 8 * i, a);
    ld8(xv + 8 * (i + C), b);
    st8(yv + 8 * i, a);
    st8(yv + 8 * (i + C), b);
  }
  for (; i < nv; i += C) {
    float a[8];
    ld8(xv + 8 * i, a);
    st8(yv + 8 * i, a);
  }
  for (uint64_t t = head + 8 * nv + tid; t < n; t += C) __stcg(y + t, __ldcg(x + t));
}

// Loads of an epoch's read-only descriptors (items, successors, factors): the
// non-coherent path (ld.global.nc) for ordinary launches; L2-only loads
// (ld.global.cg) in stream launches, whose sub-epoch blobs are copied in while
// the kernel runs (ld.global.nc is defined only for data read-only for the
// whole kernel).
template <bool NC, class T>
__device__ __forceinline__ T ldro(const T *p) {
  if constexpr (NC) return __ldg(p);
  else return __ldcg(p);
}

// ---- scheduler-warp helpers (lane 0 only) ---------------------------------
__device__ __forceinline__ void raise_error(const EpochArgs &a, unsigned code) {
  atomicCAS(&a.ctr->error, 0u, code);
  atomicExch(&a.ctr->abort, 1u);
  if (a.stream_abort) atomicExch(a.stream_abort, 1u);
}

// Pop the unit at ticket t (spinning until published), or kStop.
__device__ __forceinline__ unsigned long long pop_unit(const EpochArgs &a, unsigned long long &t) {
  t = atomicAdd(&a.ctr->head, 1ull);
  if (t >= a.total_units) return kStop;
  unsigned long long u = ld_acquire_u64(&a.queue[t]);
  if (u == Q_EMPTY) {
    const uint64_t start = globaltimer();
    for (unsigned spin = 0;; ++spin) {
      __nanosleep(spin < 64 ? 32 : 256);
      u = ld_acquire_u64(&a.queue[t]);
      if (u != Q_EMPTY) break;
      if ((spin & 63) == 63) {
        if (ld_relaxed_u32(&a.ctr->abort)) return kStop;
        if (globaltimer() - start > a.watchdog_ns) {
          raise_error(a, ERR_WATCHDOG);
          return kStop;
        }
      }
    }
  }
  if ((u >> 32) >= a.nitems) {
    raise_error(a, ERR_BAD_UNIT);
    return kStop;
  }
  return u;
}

// Completion of one unit (scheduler lane 0).  Memory-model pattern: the
// compute warps' stores are ordered before this thread by the CTA-scope
// mbarrier (release/acquire), then every counter update is an acq_rel RMW at
// gpu scope: it releases everything this thread has observed (cumulativity)
// and acquires what the other predecessors / chunks released with theirs; a
// ready successor's units are published by relaxed stores after one
// fence.acq_rel (no sequentially-consistent fence anywhere).
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned *p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// CTA-local continuation mailbox ("rw" kernel): one ready successor may be
// handed to this CTA's own pop warp instead of the global queue, so a chain
// of dependent tasks stays on one SM (its tile stays in L2) and skips the
// queue round trip.  state: 0 empty, 2 being written, 1 full.
// The first successor's descriptor can travel with it (staged: the release
// warp loaded it while the predecessor was computing), so the pop warp starts
// the continuation without a global load.
struct Mailbox {
  unsigned long long *unit;
  unsigned *state;
  uint4 *item;        // 2 x 16 bytes: the staged DItem
  unsigned *staged;   // 1: *item holds the unit's descriptor
  uint64_t *bar;      // mbarrier (count 1): one phase per put, wakes a pop warp in try_wait
};

__device__ __forceinline__ bool mailbox_put(const Mailbox &mb, unsigned long long unit, bool stage = false,
                                            uint4 i0 = uint4{}, uint4 i1 = uint4{}) {
  if (!mb.unit || atomicCAS(mb.state, 0u, 2u) != 0u) return false;
  *reinterpret_cast<volatile unsigned long long *>(mb.unit) = unit;
  if (stage) {
    mb.item[0] = i0;
    mb.item[1] = i1;
  }
  *reinterpret_cast<volatile unsigned *>(mb.staged) = stage ? 1u : 0u;
  __threadfence_block();
  *reinterpret_cast<volatile unsigned *>(mb.state) = 1u;
  if (mb.bar)
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                     (unsigned)__cvta_generic_to_shared(mb.bar))
                 : "memory");
  return true;
}

// Release metadata of a unit: read-only descriptors, so the release warp
// loads them while the unit is still being computed (off the critical path).
struct RelMeta {
  uint32_t n, nchunks, nsucc, off;   // off: the successor list (or the single successor's id)
  uint32_t s0, s0kind, s0nc, s0n;    // first successor (valid if nsucc > 0); s0kind = its meta
  uint4 i0, i1;                   // its descriptor (DItem as 2 x 16 bytes)
  bool s0stage;                   // a continuation candidate that needs no factor list
};

// Successors of an item: count and where the list starts (device_abi.h
// DItem::succ; an escaped count is stored in front of the list).
template <bool NC>
__device__ __forceinline__ void succ_list(const EpochArgs &a, uint32_t field, uint32_t succ, uint32_t &n,
                                          uint32_t &off) {
  if (field == K_NSUCC_ESC) {
    n = ldro<NC>(&a.succ[succ]);
    off = succ + 1;
  } else {
    n = field;
    off = succ;
  }
}
// self: the item's descriptor already staged in shared memory, or null.
template <bool NC = true>
__device__ __forceinline__ RelMeta release_meta(const EpochArgs &a, uint32_t item, const DItem *self = nullptr) {
  RelMeta m;
  uint32_t n, meta, succ;
  if (self) {
    n = self->n;
    meta = self->meta;
    succ = self->succ;
  } else {
    const DItem &it = a.items[item];
    n = ldro<NC>(&it.n);
    meta = ldro<NC>(&it.meta);
    succ = ldro<NC>(&it.succ);
  }
  m.n = n;
  m.nchunks = units_of(n, a.chunk_elems);
  succ_list<NC>(a, meta >> K_NSUCC_SHIFT, succ, m.nsucc, m.off);
  m.s0 = m.s0kind = m.s0nc = m.s0n = 0;
  m.s0stage = false;
  m.i0 = m.i1 = uint4{};
  if (m.nsucc) {
    m.s0 = m.nsucc == 1 ? m.off : ldro<NC>(&a.succ[m.off]);   // a single successor is stored inline
    const uint4 *src = reinterpret_cast<const uint4 *>(a.items + m.s0);
    m.i0 = ldro<NC>(src);       // x, y
    m.i1 = ldro<NC>(src + 1);   // n (x), meta (y), arg (z), succ (w)
    static_assert(offsetof(DItem, n) == 16 && offsetof(DItem, meta) == 20 && offsetof(DItem, arg) == 24,
                  "DItem layout");
    m.s0kind = m.i1.y;
    m.s0n = m.i1.x;
    m.s0nc = units_of(m.i1.x, a.chunk_elems);
    m.s0stage = (m.s0kind & K_SINGLE_PRED) && m.s0nc == 1 &&
                ((m.s0kind & K_MASK) != K_SCAL || ((m.s0kind >> K_K_SHIFT) & K_K_MASK) == 1);
  }
  return m;
}

// Publish units [c0, c1) of successor s (ready): the queue (or its priority
// level) gets them after one release fence.
__device__ __forceinline__ void publish_units(const EpochArgs &a, uint32_t s, uint32_t skind, uint32_t c0, uint32_t c1) {
  const uint32_t nc = c1 - c0;
  unsigned long long *qd;
  if (a.bk) {   // priority level of the successor (device_abi.h Bucket)
    Bucket *bk = a.bk + ((skind >> K_LEVEL_SHIFT) & K_LEVEL_MASK);
    const unsigned long long pos = atomicAdd(&bk->tail, (unsigned long long)nc);
    qd = a.queue + a.nready + __ldcg(&bk->pbase) + (pos - __ldcg(&bk->ready));
  } else {
    qd = a.queue + atomicAdd(&a.ctr->tail, (unsigned long long)nc);
  }
  fence_acq_rel_gpu();   // one release fence covers the nc relaxed publications
#pragma unroll 1
  for (uint32_t c = 0; c < nc; ++c) st_relaxed_u64(qd + c, ((unsigned long long)s << 32) | (c0 + c));
}

// Completion of unit (item, ch).  Per successor s:
//  * chunk-wise (device_abi.h K_ITEM_DEPS; same length, the item has several
//    chunks): chunk ch of s loses one predecessor now;
//  * otherwise, once the item's last chunk is done, every chunk of s does.
// A single-predecessor successor's chunks are ready at once (no counter); with
// more predecessors the counter's acq_rel RMW both releases ours and acquires
// theirs (the publication is a release either way: fence.acq_rel, then the
// relaxed slot stores the consumer reads with ld.acquire).  One loop serves
// every case -- small units are its one-iteration instance -- so that the
// kernels, which inline this at several sites, stay small (a separate general
// path grew the stream kernel by 70 % and cost the 1-wide chain 6 %).
template <bool NC = true>
__device__ __forceinline__ void release_unit(const EpochArgs &a, unsigned long long unit, const Mailbox &mb = Mailbox{},
                                             const RelMeta *pre = nullptr) {
  const uint32_t item = (uint32_t)(unit >> 32), ch = (uint32_t)unit;
  const RelMeta m = pre ? *pre : release_meta<NC>(a, item);
  const uint32_t nchunks = m.nchunks, nsucc = m.nsucc, off = m.off;
  bool item_done = true;
  if (nchunks > 1) item_done = atom_add_acq_rel(&a.chunk_done[item], 1u) + 1 == nchunks;
  for (uint32_t i = 0; i < nsucc; ++i) {
    const uint32_t s = i == 0 ? m.s0 : ldro<NC>(&a.succ[off + i]);
    const uint32_t skind = i == 0 ? m.s0kind : ldro<NC>(&a.items[s].meta);
    // units [c0, c1) of s lose this predecessor; cnt + c: their counters
    uint32_t c0 = 0, c1 = 1;
    int32_t *cnt = a.pending + s;
    if (nchunks > 1 || !(skind & K_ONE_UNIT)) {
      const uint32_t sn = i == 0 ? m.s0n : ldro<NC>(&a.items[s].n);
      const bool chunkwise = nchunks > 1 && !(skind & (K_ONE_UNIT | K_ITEM_DEPS)) && sn == m.n;
      if (chunkwise) {
        c0 = ch;
        c1 = ch + 1;
      } else if (!item_done) {
        continue;
      } else if (!(skind & K_ONE_UNIT)) {
        c1 = units_of(sn, a.chunk_elems);
      }
      if (!(skind & (K_ONE_UNIT | K_SINGLE_PRED))) cnt = a.cpending + ldro<NC>(&a.unit_base[s]);
    }
    // a single ready unit may run on this CTA next (the mailbox: its tile is
    // in L2); a whole single-unit successor travels with its descriptor
    const bool one = c1 - c0 == 1;
    for (uint32_t c = c0; c < c1; ++c) {
      if (!(skind & K_SINGLE_PRED) && atom_add_acq_rel(reinterpret_cast<unsigned *>(cnt + c), 0xFFFFFFFFu) != 1u)
        continue;
      if (one && mailbox_put(mb, ((unsigned long long)s << 32) | c, i == 0 && m.s0stage, m.i0, m.i1)) continue;
      const uint32_t e = (skind & K_SINGLE_PRED) ? c1 : c + 1;   // no counters: all at once
      publish_units(a, s, skind, c, e);
      c = e - 1;
    }
  }
  atomicAdd(&a.ctr->done, 1ull);
}

// ---- mbarrier (compute warps -> scheduler warp: "unit done") -------------
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
// Non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t *bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Blocking: suspend (mbarrier.try_wait) until the phase with this parity completes;
// a busy test_wait loop would steal issue slots from the compute warps.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  const unsigned addr = (unsigned)__cvta_generic_to_shared(bar);
  unsigned ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  }
}

// Suspend until the phase with this parity completes or about hint_ns pass.
__device__ __forceinline__ bool mbar_try_wait_hint(uint64_t *bar, unsigned parity, unsigned hint_ns) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(parity), "r"(hint_ns)
      : "memory");
  return ok != 0;
}

// Scheduler-warp state (lane 0): the unit held in each slot and whether it
// still awaits release; trace stamps of that unit.
struct SlotState {
  unsigned long long unit;
  unsigned parity;      // parity of the slot's next EMPTY phase
  bool unreleased;
  uint64_t g0;          // trace: globaltimer at pop start
  long long pop_cyc, body_c0;
  unsigned long long ticket;
};

template <bool NC = true>
__device__ __forceinline__ void finish_slot(const EpochArgs &a, SlotState &s) {
  const long long c1 = a.trace ? clock64() : 0;
  release_unit<NC>(a, s.unit);
  s.unreleased = false;
  if (a.trace) {
    const long long c2 = clock64();
    a.trace[4 * s.ticket + 0] = s.g0;
    a.trace[4 * s.ticket + 1] = (unsigned long long)s.pop_cyc;
    a.trace[4 * s.ticket + 2] = (unsigned long long)(c1 - s.body_c0);
    a.trace[4 * s.ticket + 3] = (unsigned long long)(c2 - c1);
    a.trace_item[s.ticket] = (uint32_t)(s.unit >> 32);
  }
}

// Block until the unit in slot s is done by the compute warps, then release it.
template <bool NC = true>
__device__ __forceinline__ void drain_slot(const EpochArgs &a, SlotState &s, uint64_t *empty) {
  if (!s.unreleased) return;
  mbar_wait(empty, s.parity);
  s.parity ^= 1;
  finish_slot<NC>(a, s);
}

// If the unit in slot s is already done, release it now (non-blocking).
template <bool NC = true>
__device__ __forceinline__ void poll_slot(const EpochArgs &a, SlotState &s, uint64_t *empty) {
  if (s.unreleased && mbar_test(empty, s.parity)) {
    s.parity ^= 1;
    finish_slot<NC>(a, s);
  }
}

#ifndef BT_MIN_CTAS
#define BT_MIN_CTAS 3   // 3 x 288 threads per SM: caps registers at 75 (measured best, profiles/r01_summary.md)
#endif

__device__ __forceinline__ unsigned ld_acquire_cta_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_u32(unsigned *p, unsigned v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v)
               : "memory");
}

// Compute warps: run units slot after slot until the STOP unit.
#ifndef BT_BULK
#define BT_BULK 0
#endif
#if BT_BULK
// ---- SCAL chain through shared memory with 1-D bulk copies (TMA engine) ----
// Each compute warp streams its sub-blocks of the unit through two 2 KiB
// shared-memory stages: lane 0 issues cp.async.bulk global->shared for the
// next sub-block (completion on an mbarrier with expect_tx) and
// cp.async.bulk shared->global for the finished one, so the warps' FMUL2
// stream never waits on a global load.
#ifndef BT_BULK_SB
#define BT_BULK_SB 512
#endif
constexpr int kSB = BT_BULK_SB;               // floats per sub-block (2 KiB)
constexpr int kSBQ = kSB / 128;               // float4s per lane per sub-block

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_load(float *smem, const float *gmem, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(float *gmem, const float *smem, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem),
               "r"((unsigned)__cvta_generic_to_shared(smem)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

// x: 32-byte aligned start of the vector part, nv: 8-float vectors.
// buf: this warp's 2 x kSB floats; bar: its 2 mbarriers; ph: their phase bits.
template <int W>
__device__ void scal_bulk(float *x, uint64_t nv, const float *sf, uint32_t k, int w, int lane, float *buf,
                          uint64_t *bar, unsigned &ph) {
  const uint64_t nflt = 8 * nv;
  const uint64_t nsb = (nflt + kSB - 1) / kSB;
  if ((uint64_t)w >= nsb) return;
  auto sb_bytes = [&](uint64_t j) -> unsigned {
    const uint64_t lo = j * kSB;
    return (unsigned)(4 * (nflt - lo < (uint64_t)kSB ? nflt - lo : (uint64_t)kSB));
  };
  fence_proxy_async();   // generic-proxy writes acquired earlier -> visible to the bulk loads
  if (lane == 0) {
    mbar_expect_tx(&bar[0], sb_bytes(w));
    bulk_load(buf, x + (uint64_t)w * kSB, sb_bytes(w), &bar[0]);
  }
  int st = 0;
  for (uint64_t j = w; j < nsb; j += W, st ^= 1) {
    const uint64_t jn = j + W;
    if (jn < nsb && lane == 0) {
      bulk_wait_read();   // the stage we refill has been read by its bulk store
      mbar_expect_tx(&bar[st ^ 1], sb_bytes(jn));
      bulk_load(buf + (st ^ 1) * kSB, x + jn * kSB, sb_bytes(jn), &bar[st ^ 1]);
    }
    mbar_wait(&bar[st], (ph >> st) & 1u);
    ph ^= 1u << st;
    float *sb = buf + st * kSB;
    const unsigned bytes = sb_bytes(j);
    const int nq = (int)(bytes / 16);          // float4s in this sub-block (multiple of 2)
    float v[kSBQ / 2][8];
#pragma unroll
    for (int q = 0; q < kSBQ; ++q) {
      const int idx = q * 32 + lane;
      float4 f = idx < nq ? reinterpret_cast<const float4 *>(sb)[idx] : make_float4(1.f, 1.f, 1.f, 1.f);
      v[q >> 1][(q & 1) * 4 + 0] = f.x;
      v[q >> 1][(q & 1) * 4 + 1] = f.y;
      v[q >> 1][(q & 1) * 4 + 2] = f.z;
      v[q >> 1][(q & 1) * 4 + 3] = f.w;
    }
    chain_apply<kSBQ / 2>(v, sf, k);
#pragma unroll
    for (int q = 0; q < kSBQ; ++q) {
      const int idx = q * 32 + lane;
      if (idx < nq)
        reinterpret_cast<float4 *>(sb)[idx] =
            make_float4(v[q >> 1][(q & 1) * 4 + 0], v[q >> 1][(q & 1) * 4 + 1], v[q >> 1][(q & 1) * 4 + 2],
                        v[q >> 1][(q & 1) * 4 + 3]);
    }
    fence_proxy_async();   // this lane's shared-memory writes -> visible to the bulk store
    __syncwarp();
    if (lane == 0) bulk_store(x + j * kSB, sb, bytes);
  }
  if (lane == 0) {
    bulk_wait_all();       // the unit's results are in global memory
    fence_proxy_async();   // ... and ordered before the generic-proxy release that follows
  }
  __syncwarp();
}
#endif

// STREAM: a stream launch; slot b's unit belongs to the sub-epoch whose
// arguments the scheduler warp staged in s_args[b] (else every unit uses a0).
template <int C, int S, bool PF = false, bool STREAM = false>
__device__ __forceinline__ void compute_loop(const EpochArgs &a0, const EpochArgs *s_args,
                                             const unsigned long long *s_unit,
                                             const DItem *s_item, float (*s_fac)[kMaxFactors], uint64_t *s_empty,
                                             int lane,
                                             float *s_bulk = nullptr, uint64_t *s_bulk_bar = nullptr,
                                             long long *s_cst = nullptr, long long *s_cen = nullptr) {
  const int tid = threadIdx.x - (kBlock - C);
#if BT_BULK
  const int cw = tid >> 5;
  unsigned bulk_ph = 0;
#endif
  for (unsigned u = 0;; ++u) {
    const int b = (int)(u % S);
    bar_sync(kBarFull + b, 32 + C);   // FULL[b]: the pop warp + the compute warps
    const unsigned long long unit = s_unit[b];
    if (unit == kStop) break;
    const EpochArgs &a = STREAM ? s_args[b] : a0;
#if BT_TRACE_DETAIL
    if (s_cst && tid == 0 && a.trace) s_cst[b] = clock64();
#endif
    const uint32_t chunk = (uint32_t)unit;
    const DItem it = s_item[b];                  // staged by the pop warp
    const uint64_t lo = (uint64_t)chunk * a.chunk_elems;
    const uint64_t hi = min((uint64_t)it.n, lo + a.chunk_elems);
    const uint32_t kk = it.k();
    switch (it.kind()) {
      case K_SCAL:
#if BT_BULK
        if (s_bulk) {
          float *xs = reinterpret_cast<float *>(it.x) + lo;
          const uint64_t n = hi - lo;
          const uint64_t head = head_elems(xs, n);
          for (uint64_t i = tid; i < head; i += C) __stcg(xs + i, chain_scalar(__ldcg(xs + i), s_fac[b], kk));
          const uint64_t nv = (n - head) >> 3;
          scal_bulk<C / 32>(xs + head, nv, s_fac[b], kk, cw, lane, s_bulk + cw * 2 * kSB, s_bulk_bar + 2 * cw,
                            bulk_ph);
          for (uint64_t t = head + 8 * nv + tid; t < n; t += C)
            __stcg(xs + t, chain_scalar(__ldcg(xs + t), s_fac[b], kk));
          break;
        }
#endif
        // short chains are HBM-bound: keep the next step's loads in flight
        // (C5-16 kernel 6.41 vs 6.33 TB/s); long ones are FP32-bound: the
        // wider step without prefetch is faster (C5 2.07 vs 2.08 ms).  One
        // body per kernel instance (both inlined would spill).
        if (PF)
          scal_range_pf<2, C>(reinterpret_cast<float *>(it.x) + lo, hi - lo, s_fac[b], kk, tid);
        else
          scal_range<4, C>(reinterpret_cast<float *>(it.x) + lo, hi - lo, s_fac[b], kk, tid);
        break;
      case K_AXPY:
        axpy_range<C>(reinterpret_cast<const float *>(it.x) + lo, reinterpret_cast<float *>(it.y) + lo, hi - lo,
                      __uint_as_float(it.arg), tid);
        break;
      case K_COPY:
        copy_range<C>(reinterpret_cast<const float *>(it.x) + lo, reinterpret_cast<float *>(it.y) + lo, hi - lo,
                      tid);
        break;
      default:
        if (tid == 0) raise_error(a, ERR_BAD_KIND);
        break;
    }
    // this warp's stores precede the arrive (mbarrier.arrive releases at CTA
    // scope; __syncwarp orders the other lanes' stores before lane 0's arrive)
    __syncwarp();
#if BT_TRACE_DETAIL
    if (s_cen && tid == 0 && a.trace) s_cen[b] = clock64();
#endif
    if (lane == 0) mbar_arrive(&s_empty[b]);
  }
}

#ifndef BT_INSLOT
#define BT_INSLOT 1
#endif

// Compute warps of the "rw" kernel.  As the generic loop, plus in-slot
// continuation: when a finished unit's only successor has it as its only
// predecessor and is a single unit needing no factor list, the compute warps
// run that successor next in the same slot, without a release, a queue or a
// mailbox round trip (its readiness follows from this unit's completion, and
// a barrier of the compute warps orders this unit's stores before the
// successor's loads).  Such chains -- C4's per-tile task chains, 1-wide
// dependency chains -- then cost one compute-warp barrier per link; the slot
// is released once, at the chain's last unit (s_final), and the skipped
// releases are counted into ctr->done.  Off when tracing (one record per unit).
template <int C, int S>
__device__ __forceinline__ void compute_loop_rw(const EpochArgs &a, const unsigned long long *s_unit,
                                                const DItem *s_item, float (*s_fac)[kMaxFactors], uint64_t *s_empty,
                                                DItem (*s_nitem)[2], float (*s_nfac)[2], unsigned (*s_go)[2],
                                                unsigned long long *s_final, int lane, long long *s_cst = nullptr,
                                                long long *s_cen = nullptr) {
  const int tid = threadIdx.x - (kBlock - C);
  for (unsigned u = 0;; ++u) {
    const int b = (int)(u % S);
    bar_sync(kBarFull + b, 32 + C);   // FULL[b]: the pop warp + the compute warps
    unsigned long long unit = s_unit[b];
    if (unit == kStop) break;
#if BT_TRACE_DETAIL
    if (s_cst && tid == 0 && a.trace) s_cst[b] = clock64();
#endif
    DItem it = s_item[b];                        // staged by the pop warp
    const float *fac = s_fac[b];
    unsigned par = 0, extra = 0;
    for (;;) {
      // may this unit continue in the slot?  (uniform: every thread sees it)
      const bool maybe = BT_INSLOT && !a.trace && (uint64_t)it.n <= a.chunk_elems && it.nsucc_field() == 1;
      if (maybe && tid == 0) {   // the successor's descriptor, copied to shared memory under the body
        const unsigned dst = (unsigned)__cvta_generic_to_shared(&s_nitem[b][par]);
        const DItem *src = a.items + it.succ;
#pragma unroll
        for (int q = 0; q < 2; ++q)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * q), "l"(reinterpret_cast<const char *>(src) + 16 * q)
                       : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
      const uint32_t chunk = (uint32_t)unit;
      const uint64_t lo = (uint64_t)chunk * a.chunk_elems;
      const uint64_t hi = min((uint64_t)it.n, lo + a.chunk_elems);
      switch (it.kind()) {
        case K_SCAL:   // small units (the rw kernel's domain): 2 x 8 elements per thread and step
          scal_range<2, C>(reinterpret_cast<float *>(it.x) + lo, hi - lo, fac, it.k(), tid);
          break;
        case K_AXPY:
          axpy_range<C>(reinterpret_cast<const float *>(it.x) + lo, reinterpret_cast<float *>(it.y) + lo, hi - lo,
                        __uint_as_float(it.arg), tid);
          break;
        case K_COPY:
          copy_range<C>(reinterpret_cast<const float *>(it.x) + lo, reinterpret_cast<float *>(it.y) + lo, hi - lo,
                        tid);
          break;
        default:
          if (tid == 0) raise_error(a, ERR_BAD_KIND);
          break;
      }
      if (!maybe) break;
      if (tid == 0) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        const DItem &n = s_nitem[b][par];
        const unsigned go = n.single_pred() && (uint64_t)n.n <= a.chunk_elems && (n.kind() != K_SCAL || n.k() == 1)
                                ? 1u : 0u;
        if (go) s_nfac[b][par] = __uint_as_float(n.arg);   // a single factor travels in arg
        s_go[b][par] = go;
      }
      // all compute warps: this unit's stores are done (and visible in the CTA)
      // and the decision is published; buffers alternate so a slow warp can
      // still read this step's while thread 0 fills the next
      bar_sync_n<kBarCompute>(C);
      if (!s_go[b][par]) break;
      unit = (unsigned long long)it.succ << 32;   // one successor: succ is its id
      it = s_nitem[b][par];
      fac = &s_nfac[b][par];
      par ^= 1u;
      ++extra;
    }
    if (tid == 0) {
      s_final[b] = unit;                                   // the unit the release warp releases
      if (extra) atomicAdd(&a.ctr->done, (unsigned long long)extra);   // the chain's skipped releases
    }
    __syncwarp();
#if BT_TRACE_DETAIL
    if (s_cen && tid == 0 && a.trace) s_cen[b] = clock64();
#endif
    if (lane == 0) mbar_arrive(&s_empty[b]);
  }
}

// Pop the unit at a fresh ticket (lane 0), spinning until it is published.
__device__ __forceinline__ unsigned long long pop_ticket(const EpochArgs &a, unsigned long long &t) {
  t = atomicAdd(&a.ctr->head, 1ull);
  if (t >= a.total_units) return kStop;
  unsigned long long unit = ld_acquire_u64(&a.queue[t]);
  if (unit == Q_EMPTY) {
    const uint64_t start = globaltimer();
    for (unsigned spin = 0;; ++spin) {
      __nanosleep(spin < 64 ? 32 : 256);
      unit = ld_acquire_u64(&a.queue[t]);
      if (unit != Q_EMPTY) break;
      if ((spin & 63) == 63) {
        if (ld_relaxed_u32(&a.ctr->abort)) return kStop;
        if (globaltimer() - start > a.watchdog_ns) {
          raise_error(a, ERR_WATCHDOG);
          return kStop;
        }
      }
    }
  }
  if ((unit >> 32) >= a.nitems) {
    raise_error(a, ERR_BAD_UNIT);
    return kStop;
  }
  return unit;
}

// Stage a unit for the compute warps: its item descriptor (48 bytes, lanes
// 0-2) and, for SCAL, its factor list into shared memory.
template <bool NC = true>
__device__ __forceinline__ void stage_unit(const EpochArgs &a, unsigned long long unit, DItem *item_dst,
                                           float *fac_dst, int lane) {
  if (unit == kStop) return;
  const DItem *it = a.items + (uint32_t)(unit >> 32);
  if (lane < 2) reinterpret_cast<uint4 *>(item_dst)[lane] = ldro<NC>(reinterpret_cast<const uint4 *>(it) + lane);
  const uint32_t meta = ldro<NC>(&it->meta);
  if ((meta & K_MASK) == K_SCAL) {
    const uint32_t k = (meta >> K_K_SHIFT) & K_K_MASK, arg = ldro<NC>(&it->arg);
    if (k == 1) {   // a single factor travels inline in arg: no dependent load
      if (lane == 0) fac_dst[0] = __uint_as_float(arg);
    } else {
      for (uint32_t j = lane; j < k; j += 32) fac_dst[j] = ldro<NC>(a.factors + arg + j);
    }
  }
}

// The last CTA to leave copies the epoch counters to mapped host memory, so
// the host checks completion without a device-to-host copy (which would queue
// behind the write-back copies on the copy engine).
__device__ __forceinline__ void report_exit(const EpochArgs &a) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&a.ctr->exited, 1u) == gridDim.x - 1) {
      __threadfence();
      volatile Counters *h = a.host_ctr;
      h->head = atomicAdd(&a.ctr->head, 0ull);
      h->tail = atomicAdd(&a.ctr->tail, 0ull);
      h->done = atomicAdd(&a.ctr->done, 0ull);
      h->error = atomicAdd(&a.ctr->error, 0u);
      h->exited = gridDim.x;
      __threadfence_system();
    }
  }
}

// ---------------------------------------------------------------------------
// "rw": three roles per CTA.  Warp 0 pops units into kSlots shared-memory slots
// (FULL[b]: a named barrier with the compute warps); warps 2..8 compute;
// warp 1 releases finished units (EMPTY[b]: an mbarrier the compute warps
// arrive on), up to kSlots at once on different lanes so their dependency
// RMWs overlap.  Popping, computing and releasing overlap; the pop warp only
// waits for a slot whose previous unit is released.  A CTA spinning for an
// unpublished unit never holds finished-but-unreleased work (the release warp
// runs independently), so it cannot starve the successor it waits for.
__global__ void __launch_bounds__(kBlock, BT_MIN_CTAS) scheduler_kernel_rw(EpochArgs a) {
  constexpr int kCompute = kComputeRW, kSlots = kSlotsRW;
  __shared__ unsigned long long s_unit[kSlots];
  __shared__ DItem s_item[kSlots];
  __shared__ __align__(8) uint64_t s_empty[kSlots];
  __shared__ __align__(16) float s_fac[kSlots][kMaxFactors];
  __shared__ DItem s_nitem[kSlots][2];              // in-slot continuation (compute warps)
  __shared__ float s_nfac[kSlots][2];
  __shared__ unsigned s_go[kSlots][2];
  __shared__ unsigned long long s_final[kSlots];    // last unit run in the slot
  __shared__ unsigned s_popped, s_released, s_mb_state, s_mb_staged, s_mb_expect;
  __shared__ __align__(8) uint64_t s_mb_bar;
  __shared__ unsigned long long s_mb_unit;
  __shared__ uint4 s_mb_item[2];
  __shared__ unsigned long long s_g0[kSlots];
  __shared__ long long s_popc[kSlots], s_c1[kSlots];
#if BT_TRACE_DETAIL
  __shared__ long long s_cst[kSlots], s_cen[kSlots];
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int b = 0; b < kSlots; ++b) mbar_init(&s_empty[b], kCompute / 32);
    s_popped = 0;
    s_released = 0;
    s_mb_state = 0;
    s_mb_staged = 0;
    s_mb_expect = 0;
    mbar_init(&s_mb_bar, 1);
  }
  __syncthreads();

  if (warp == 0) {
    // ================= pop warp =================
    unsigned long long ticket = 0;
    bool have_ticket = false;
    unsigned mb_taken = 0;   // mailbox entries taken (= phases of s_mb_bar consumed)
    for (unsigned u = 0;; ++u) {
      const int b = (int)(u % kSlots);
      if (u >= kSlots)   // the slot's previous unit must be released
        while (ld_acquire_cta_u32(&s_released) + kSlots <= u) __nanosleep(32);
      unsigned long long unit = kStop;
      unsigned staged = 0;
      if (lane == 0) {
        const uint64_t g0 = a.trace ? globaltimer() : 0;
        const long long c0 = a.trace ? clock64() : 0;
        // 1) a continuation from this CTA's release warp, 2) the unit at our
        // ticket (taken once, kept across continuations), 3) termination: no
        // queue work left for us and nothing of ours in flight, or every unit
        // of the epoch done.
        const uint64_t start = globaltimer();
        for (unsigned spin = 0;; ++spin) {
          // the mailbox first, with no global load outstanding (the block
          // fence below would wait for it: measured +0.35 us per chain link)
          if (*reinterpret_cast<volatile unsigned *>(&s_mb_state) == 1u) {
            __threadfence_block();
            unit = *reinterpret_cast<volatile unsigned long long *>(&s_mb_unit);
            staged = *reinterpret_cast<volatile unsigned *>(&s_mb_staged);
            if (staged) {   // copy the descriptor out before the mailbox is reused
              const volatile uint4 *src = s_mb_item;
              uint4 *dst = reinterpret_cast<uint4 *>(&s_item[b]);
              for (int q = 0; q < 2; ++q) {
                const uint4 w = {src[q].x, src[q].y, src[q].z, src[q].w};
                dst[q] = w;
              }
            }
            __threadfence_block();
            *reinterpret_cast<volatile unsigned *>(&s_mb_state) = 0u;
            ++mb_taken;
            break;
          }
          if (!have_ticket) {
            ticket = atomicAdd(&a.ctr->head, 1ull);
            have_ticket = true;
          }
          const bool poll = ticket < a.total_units;
          if (poll) {
            // relaxed poll (an acquire load would hold back the mailbox
            // checks behind its round trip); re-read with acquire once published
            unsigned long long v = ld_relaxed_u64(&a.queue[ticket]);
            if (v != Q_EMPTY) {
              v = ld_acquire_u64(&a.queue[ticket]);   // slots are written once: same value, now acquired
              unit = v;
              have_ticket = false;
              if ((unit >> 32) >= a.nitems) {
                raise_error(a, ERR_BAD_UNIT);
                unit = kStop;
              }
              break;
            }
          }
          // (the queue load above also paces this loop: a tight shared-memory
          // spin slows the CTA's barriers -- measured: chain 2.0 vs 1.4 us)
          const bool inflight = ld_acquire_cta_u32(&s_released) != u;   // a continuation may come
          if (!poll && !inflight && *reinterpret_cast<volatile unsigned *>(&s_mb_state) == 0u) {
            unit = kStop;      // all our units released, no continuation pending
            break;
          }
          if ((spin & 63) == 63) {
            if (ld_relaxed_u64(&a.ctr->done) == a.total_units) {
              unit = kStop;
              break;
            }
            if (ld_relaxed_u32(&a.ctr->abort)) {
              unit = kStop;
              break;
            }
            if (globaltimer() - start > a.watchdog_ns) {
              raise_error(a, ERR_WATCHDOG);
              unit = kStop;
              break;
            }
          }
          // a continuation is on its way (the release warp said so) and the
          // queue had nothing: sleep on the mailbox barrier, woken by the put;
          // with nothing of ours in flight back off; otherwise keep polling
          if (inflight && *reinterpret_cast<volatile unsigned *>(&s_mb_expect))
            mbar_try_wait_hint(&s_mb_bar, mb_taken & 1u, 1000u);
          else if (!inflight)
            __nanosleep(spin < 64 ? 32 : 256);
        }
        if (a.trace) {
          s_g0[b] = g0;
          s_c1[b] = clock64();
          s_popc[b] = s_c1[b] - c0;
        }
      }
      unit = __shfl_sync(0xffffffffu, unit, 0);
      staged = __shfl_sync(0xffffffffu, staged, 0);
      __syncwarp();   // memory order: lane 0's ld.acquire of the unit before the other lanes' descriptor loads
      if (!staged) {
        stage_unit(a, unit, &s_item[b], s_fac[b], lane);
      } else if (lane == 0 && s_item[b].kind() == K_SCAL) {
        s_fac[b][0] = __uint_as_float(s_item[b].arg);   // staged SCAL continuations have k == 1
      }
      if (lane == 0) s_unit[b] = unit;
      __syncwarp();
      if (lane == 0) st_release_cta_u32(&s_popped, u + 1);
      bar_arrive(kBarFull + b, 32 + kCompute);
      if (unit == kStop) break;
    }
  } else if (warp == 1) {
    // ================= release warp =================
    for (unsigned u = 0;;) {
      // the pop warp publishes within a few hundred cycles once it has a
      // unit: spin (a sleeping release warp delays the critical path of chains)
      for (unsigned spin = 0; ld_acquire_cta_u32(&s_popped) <= u; ++spin)
        if (spin >= 4096) __nanosleep(64);
      if (s_unit[u % kSlots] == kStop) break;
      // unit u's release metadata, loaded while it is being computed
      RelMeta pre{};
      if (lane == 0) {
        pre = release_meta(a, (uint32_t)(s_unit[u % kSlots] >> 32), &s_item[u % kSlots]);
        // this unit's release will hand a continuation to the pop warp (one
        // the compute warps run in the slot does not come through the mailbox)
        const bool cont = pre.nchunks == 1 && pre.nsucc > 0 && (pre.s0kind & K_SINGLE_PRED) && pre.s0nc == 1;
        const bool inslot = BT_INSLOT && !a.trace && pre.nchunks == 1 && pre.nsucc == 1 && pre.s0stage;
        *reinterpret_cast<volatile unsigned *>(&s_mb_expect) = cont && !inslot ? 1u : 0u;
      }
      mbar_wait(&s_empty[u % kSlots], (u / kSlots) & 1u);
      // batch the following units that are already done
      unsigned m = 1;
      if (lane == 0) {
        const unsigned popped = ld_acquire_cta_u32(&s_popped);
        while (m < kSlots) {
          const unsigned v = u + m;
          if (v >= popped || s_unit[v % kSlots] == kStop || !mbar_test(&s_empty[v % kSlots], (v / kSlots) & 1u))
            break;
          ++m;
        }
      }
      m = __shfl_sync(0xffffffffu, m, 0);
      if (lane < (int)m) {
        const unsigned v = u + lane;
        const int b = (int)(v % kSlots);
        const unsigned long long unit = s_final[b];   // the popped unit, or the end of an in-slot chain
        const long long c1 = a.trace ? clock64() : 0;
        release_unit(a, unit, Mailbox{&s_mb_unit, &s_mb_state, s_mb_item, &s_mb_staged, &s_mb_bar},
                     lane == 0 && unit == s_unit[b] ? &pre : nullptr);
        if (a.trace) {
          // the unit's own record (item's first record + chunk): no shared
          // counter in or around the measured window
          const long long c2r = clock64();
          const unsigned long long t = (unsigned long long)a.unit_base[(uint32_t)(unit >> 32)] + (uint32_t)unit;
          a.trace[4 * t + 0] = s_g0[b];
#if BT_TRACE_DETAIL
          // detail: [1] handoff pop -> compute start, [2] compute, [3] compute end -> release start
          a.trace[4 * t + 1] = (unsigned long long)(s_cst[b] - s_c1[b]);
          a.trace[4 * t + 2] = (unsigned long long)(s_cen[b] - s_cst[b]);
          a.trace[4 * t + 3] = (unsigned long long)(c1 - s_cen[b]);
#else
          a.trace[4 * t + 1] = (unsigned long long)s_popc[b];
          a.trace[4 * t + 2] = (unsigned long long)(c1 - s_c1[b]);
          a.trace[4 * t + 3] = (unsigned long long)(c2r - c1);
#endif
          a.trace_item[t] = (uint32_t)(unit >> 32);
        }
      }
      __syncwarp();
      u += m;
      if (lane == 0) {
        *reinterpret_cast<volatile unsigned *>(&s_mb_expect) = 0u;
        st_release_cta_u32(&s_released, u);
      }
    }
  } else {
#if BT_TRACE_DETAIL
    compute_loop_rw<kCompute, kSlots>(a, s_unit, s_item, s_fac, s_empty, s_nitem, s_nfac, s_go, s_final, lane, s_cst,
                                      s_cen);
#else
    compute_loop_rw<kCompute, kSlots>(a, s_unit, s_item, s_fac, s_empty, s_nitem, s_nfac, s_go, s_final, lane);
#endif
  }
  report_exit(a);
}

// "sw": one scheduler warp pops and releases, 8 compute warps, 2 slots.
template <bool PF>
__global__ void __launch_bounds__(kBlock, BT_MIN_CTAS) scheduler_kernel_sw(EpochArgs a) {
  constexpr int kCompute = kComputeSW;
  __shared__ unsigned long long s_unit[2];
  __shared__ DItem s_item[2];
  __shared__ __align__(8) uint64_t s_empty[2];
  __shared__ __align__(16) float s_fac[2][kMaxFactors];
#if BT_BULK
  __shared__ __align__(128) float s_bulk[kCompute / 32][2][kSB];
  __shared__ __align__(8) uint64_t s_bulk_bar[kCompute / 32][2];
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&s_empty[0], kCompute / 32);
    mbar_init(&s_empty[1], kCompute / 32);
#if BT_BULK
    for (int w = 0; w < kCompute / 32; ++w) {
      mbar_init(&s_bulk_bar[w][0], 1);
      mbar_init(&s_bulk_bar[w][1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#endif
  }
  __syncthreads();

  if (warp == 0) {
    // ================= scheduler warp (pop + release) =================
    // Invariant: the scheduler never spins on the queue while a finished unit
    // of this CTA is unreleased (it polls the other slot while waiting), so a
    // CTA cannot starve the very successor it is waiting for.
    SlotState st[2];
    for (int b = 0; b < 2; ++b) {
      st[b].unit = kStop;
      st[b].parity = 0;
      st[b].unreleased = false;
    }
    for (unsigned u = 0;; ++u) {
      const int b = u & 1;
      unsigned long long unit = kStop;
      if (lane == 0) {
        drain_slot(a, st[b], &s_empty[b]);        // slot b's previous unit (u-2)
        const uint64_t g0 = a.trace ? globaltimer() : 0;
        const long long c0 = a.trace ? clock64() : 0;
        const unsigned long long t = atomicAdd(&a.ctr->head, 1ull);
        if (t < a.total_units) {
          unit = ld_acquire_u64(&a.queue[t]);
          if (unit == Q_EMPTY) {
            const uint64_t start = globaltimer();
            for (unsigned spin = 0;; ++spin) {
              poll_slot(a, st[b ^ 1], &s_empty[b ^ 1]);
              __nanosleep(spin < 64 ? 32 : 256);
              unit = ld_acquire_u64(&a.queue[t]);
              if (unit != Q_EMPTY) break;
              if ((spin & 63) == 63) {
                if (ld_relaxed_u32(&a.ctr->abort)) {
                  unit = kStop;
                  break;
                }
                if (globaltimer() - start > a.watchdog_ns) {
                  raise_error(a, ERR_WATCHDOG);
                  unit = kStop;
                  break;
                }
              }
            }
          }
          if (unit != kStop && (unit >> 32) >= a.nitems) {
            raise_error(a, ERR_BAD_UNIT);
            unit = kStop;
          }
        }
        st[b].unit = unit;
        st[b].unreleased = unit != kStop;
        if (a.trace) {
          st[b].g0 = g0;
          st[b].body_c0 = clock64();
          st[b].pop_cyc = st[b].body_c0 - c0;
          st[b].ticket = t;
        }
      }
      unit = __shfl_sync(0xffffffffu, unit, 0);
      __syncwarp();   // memory order: lane 0's ld.acquire of the unit before the other lanes' descriptor loads
      stage_unit(a, unit, &s_item[b], s_fac[b], lane);
      if (lane == 0) s_unit[b] = unit;
      __syncwarp();
      bar_arrive(kBarFull + b, 32 + kCompute);
      if (unit == kStop) {
        if (lane == 0) drain_slot(a, st[b ^ 1], &s_empty[b ^ 1]);   // unit u-1 still in flight
        break;
      }
    }
  } else {
#if BT_BULK
    compute_loop<kCompute, kSlotsSW, PF>(a, nullptr, s_unit, s_item, s_fac, s_empty, lane, &s_bulk[0][0][0], &s_bulk_bar[0][0]);
#else
    compute_loop<kCompute, kSlotsSW, PF>(a, nullptr, s_unit, s_item, s_fac, s_empty, lane);
#endif
  }
  report_exit(a);
}

// "swp": "sw" with the priority ready queue (device_abi.h Bucket; SURVEY
// NEXT-3): lane 0 of the scheduler warp holds at most one ticket per level,
// takes a ticket on a level only while it has unclaimed units, and pops the
// most urgent published one; a CTA leaves when every level is exhausted for it.
template <bool PF>
__global__ void __launch_bounds__(kBlock, BT_MIN_CTAS) scheduler_kernel_swp(EpochArgs a) {
  constexpr int kCompute = kComputeSW;
  __shared__ unsigned long long s_unit[2];
  __shared__ DItem s_item[2];
  __shared__ __align__(8) uint64_t s_empty[2];
  __shared__ __align__(16) float s_fac[2][kMaxFactors];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = (int)a.nbuckets;
  if (threadIdx.x == 0) {
    mbar_init(&s_empty[0], kCompute / 32);
    mbar_init(&s_empty[1], kCompute / 32);
  }
  __syncthreads();

  if (warp == 0) {
    // warp-cooperative pop: lane l < nb serves level l (its ticket, its
    // exhaustion); lane 0 releases (slots, as in "sw")
    SlotState st[2];
    for (int b = 0; b < 2; ++b) {
      st[b].unit = kStop;
      st[b].parity = 0;
      st[b].unreleased = false;
    }
    const bool mine = lane < nb;
    Bucket *const bk = a.bk + (mine ? lane : 0);
    const uint32_t l_total = mine ? __ldcg(&bk->total) : 0, l_ready = mine ? __ldcg(&bk->ready) : 0;
    const uint32_t l_rbase = mine ? __ldcg(&bk->rbase) : 0, l_pbase = mine ? __ldcg(&bk->pbase) : 0;
    unsigned long long held = ~0ull;   // this lane's ticket on its level
    bool exhausted = !mine;
    for (unsigned u = 0;; ++u) {
      const int b = u & 1;
      if (lane == 0) drain_slot(a, st[b], &s_empty[b]);   // slot b's previous unit (u-2)
      __syncwarp();
      unsigned long long unit = kStop;
      const uint64_t start = globaltimer();
      for (unsigned spin = 0;; ++spin) {
        // 1) a ticket on each level with unclaimed units (no wait on a drained level)
        if (held == ~0ull && !exhausted &&
            ld_relaxed_u64(&bk->tail) > ld_relaxed_u64(&bk->head)) {
          const unsigned long long t = atomicAdd(&bk->head, 1ull);
          if (t >= l_total) exhausted = true;
          else held = t;
        }
        // 2) the most urgent level whose held ticket is published
        unsigned long long *q = nullptr, v = Q_EMPTY;
        if (held != ~0ull) {
          q = held < l_ready ? a.queue + l_rbase + held : a.queue + a.nready + l_pbase + (held - l_ready);
          v = ld_relaxed_u64(q);
        }
        const unsigned pubm = __ballot_sync(0xffffffffu, v != Q_EMPTY);
        if (pubm) {
          const int top = 31 - __clz((int)pubm);
          if (lane == top) {
            v = ld_acquire_u64(q);   // slots are written once: same value, now acquired
            held = ~0ull;
          }
          unit = __shfl_sync(0xffffffffu, v, top);
          break;
        }
        // 3) leave: every level exhausted with nothing held, or every unit done
        //    (tickets taken past the last publication of a level stay unfilled)
        if (__all_sync(0xffffffffu, exhausted && held == ~0ull)) break;
        int stop = 0;
        if (lane == 0) {
          if ((spin & 15) == 15 && ld_relaxed_u64(&a.ctr->done) == a.total_units) stop = 1;
          poll_slot(a, st[b ^ 1], &s_empty[b ^ 1]);
          if ((spin & 63) == 63) {
            if (ld_relaxed_u32(&a.ctr->abort)) stop = 1;
            else if (globaltimer() - start > a.watchdog_ns) {
              raise_error(a, ERR_WATCHDOG);
              stop = 1;
            }
          }
        }
        if (__shfl_sync(0xffffffffu, stop, 0)) break;
        __nanosleep(spin < 64 ? 32 : 256);
      }
      if (lane == 0) {
        if (unit != kStop && (unit >> 32) >= a.nitems) {
          raise_error(a, ERR_BAD_UNIT);
          unit = kStop;
        }
        st[b].unit = unit;
        st[b].unreleased = unit != kStop;
      }
      unit = __shfl_sync(0xffffffffu, unit, 0);
      __syncwarp();   // memory order: the acquiring lane's load before the other lanes' descriptor loads
      stage_unit(a, unit, &s_item[b], s_fac[b], lane);
      if (lane == 0) s_unit[b] = unit;
      __syncwarp();
      bar_arrive(kBarFull + b, 32 + kCompute);
      if (unit == kStop) {
        if (lane == 0) drain_slot(a, st[b ^ 1], &s_empty[b ^ 1]);   // unit u-1 still in flight
        break;
      }
    }
  } else {
    compute_loop<kCompute, kSlotsSW, PF>(a, nullptr, s_unit, s_item, s_fac, s_empty, lane);
  }
  report_exit(a);
}

// "sw" as a stream launch (StreamCtl, device_abi.h): the
// pipelined rounds of one SCAL run are sub-epochs of this single launch, built
// and published by the host while the kernel already runs the earlier ones.
// Identical to "sw" except that the scheduler warp maps each launch-wide ticket
// to (sub-epoch, position in its queue) and stages that sub-epoch's arguments
// in shared memory next to the unit (s_args[slot]), where the compute warps
// and the release path read them.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Give up ticket t at a close (device_abi.h, StreamCtl): the resume launch runs it.
__device__ __forceinline__ void abandon_ticket(StreamCtl *ctl, unsigned long long t) {
  const unsigned i = atomicAdd(&ctl->nabandoned, 1u);
  if (i < (unsigned)kMaxStreamGrid) ctl->abandoned[i] = t;
}

// resume = 0: the run's launch; 1: its resume launch (after the last
// publication), which runs what a closed first launch left.  quiesce_ns: how
// long every CTA must have waited for a publication before the launch closes.
template <bool PF>
__global__ void __launch_bounds__(kBlock, BT_MIN_CTAS) scheduler_kernel_sws(StreamCtl *ctl, uint64_t watchdog_ns,
                                                                             uint64_t quiesce_ns, int resume) {
  constexpr int kCompute = kComputeSW;
  __shared__ unsigned long long s_unit[2];
  __shared__ DItem s_item[2];
  __shared__ __align__(8) uint64_t s_empty[2];
  __shared__ __align__(16) float s_fac[2][kMaxFactors];
  __shared__ __align__(16) EpochArgs s_args[2];
  __shared__ unsigned s_go;
  static_assert(sizeof(EpochArgs) % 8 == 0, "EpochArgs layout");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&s_empty[0], kCompute / 32);
    mbar_init(&s_empty[1], kCompute / 32);
    // a resume launch after a first launch that ran every sub-epoch: nothing to do
    s_go = resume ? ld_acquire_u32(&ctl->resume) : 1u;
  }
  __syncthreads();
  if (!s_go) return;

  if (warp == 0) {
    SlotState st[2];
    for (int b = 0; b < 2; ++b) {
      st[b].unit = kStop;
      st[b].parity = 0;
      st[b].unreleased = false;
    }
    int slot_sub[2] = {-1, -1};   // warp-uniform: the sub-epoch whose arguments s_args[b] holds
    // lane 0: the sub-epoch this CTA's tickets have reached (fresh tickets only
    // grow; an abandoned one taken by the resume launch may lie lower: rescan)
    const unsigned nsub = __ldcg(&ctl->nsub);
    const unsigned nab = resume ? min(__ldcg(&ctl->nabandoned), (unsigned)kMaxStreamGrid) : 0u;
    bool fresh = !resume;            // lane 0: abandoned tickets exhausted
    unsigned cur = 0, pub = 0;
    unsigned long long base = 0, cur_units = ~0ull;   // ~0: not loaded yet
    unsigned long long *cur_queue = nullptr;
    uint32_t cur_nitems = 0;
    for (unsigned u = 0;; ++u) {
      const int b = u & 1;
      unsigned long long unit = kStop;
      unsigned sub = 0;
      if (lane == 0) {
        drain_slot<false>(s_args[b], st[b], &s_empty[b]);   // slot b's previous unit (u-2), with its sub-epoch's args
        unsigned long long t = 0;
        if (!fresh) {
          const unsigned i = atomicAdd(&ctl->ab_take, 1u);
          if (i < nab) t = __ldcg(&ctl->abandoned[i]);
          else fresh = true;
        }
        if (fresh) t = atomicAdd(&ctl->ticket, 1ull);
        if (t < base) {   // (resume) an abandoned ticket below the current sub-epoch
          cur = 0;
          base = 0;
          cur_units = ~0ull;
        }
        bool stop = false, waiting = false;
        uint64_t start = 0;
        // the sub-epoch holding ticket t (waiting for its publication)
        for (unsigned spin = 0;;) {
          if (cur >= nsub) {
            stop = true;
            break;
          }
          if (cur >= pub) {
            pub = ld_acquire_u32(&ctl->published);
            if (cur >= pub) {
              if (spin == 0) {
                start = globaltimer();
                if (!resume) {   // counted while waiting (closing needs every CTA here)
                  atomicAdd(&ctl->state, 1u);
                  waiting = true;
                }
              }
              poll_slot<false>(s_args[b ^ 1], st[b ^ 1], &s_empty[b ^ 1]);
              __nanosleep(spin < 64 ? 64 : 512);
              if ((++spin & 63) == 0) {
                const uint64_t waited = globaltimer() - start;
                if (waiting && waited > quiesce_ns) {
                  // every CTA waiting that long: close (one CAS), or join a close
                  unsigned s = ld_relaxed_u32(&ctl->state);
                  if (s == gridDim.x) s = atomicCAS(&ctl->state, gridDim.x, gridDim.x | kStreamClosed);
                  if ((s & kStreamClosed) || s == gridDim.x) {
                    abandon_ticket(ctl, t);
                    stop = true;
                    break;
                  }
                }
                if (ld_relaxed_u32(&ctl->abort) || waited > watchdog_ns) {
                  atomicExch(&ctl->abort, 1u);   // the host sees the unfinished sub-epochs
                  stop = true;
                  break;
                }
              }
              continue;
            }
          }
          if (waiting) {   // leaving the wait: unless the launch was closed meanwhile
            waiting = false;
            if (atomicSub(&ctl->state, 1u) & kStreamClosed) {
              abandon_ticket(ctl, t);
              stop = true;
              break;
            }
          }
          if (cur_units == ~0ull) {   // read past ld.acquire(published), L2 only
            cur_units = __ldcg(&ctl->subs[cur].total_units);
            cur_queue = reinterpret_cast<unsigned long long *>(
                __ldcg(reinterpret_cast<const unsigned long long *>(&ctl->subs[cur].queue)));
            cur_nitems = __ldcg(&ctl->subs[cur].nitems);
          }
          if (t < base + cur_units) break;
          base += cur_units;
          ++cur;
          cur_units = ~0ull;
        }
        if (!stop) {
          const unsigned long long lt = t - base;
          unit = ld_acquire_u64(&cur_queue[lt]);
          if (unit == Q_EMPTY) {
            const uint64_t t0 = globaltimer();
            for (unsigned spin = 0;; ++spin) {
              poll_slot<false>(s_args[b ^ 1], st[b ^ 1], &s_empty[b ^ 1]);
              __nanosleep(spin < 64 ? 32 : 256);
              unit = ld_acquire_u64(&cur_queue[lt]);
              if (unit != Q_EMPTY) break;
              if ((spin & 63) == 63) {
                if (ld_relaxed_u32(&ctl->abort)) {
                  unit = kStop;
                  break;
                }
                if (globaltimer() - t0 > watchdog_ns) {
                  raise_error(ctl->subs[cur], ERR_WATCHDOG);
                  unit = kStop;
                  break;
                }
              }
            }
          }
          if (unit != kStop && (unit >> 32) >= cur_nitems) {
            raise_error(ctl->subs[cur], ERR_BAD_UNIT);
            unit = kStop;
          }
        }
        sub = cur;
        st[b].unit = unit;
        st[b].unreleased = unit != kStop;
      }
      unit = __shfl_sync(0xffffffffu, unit, 0);
      sub = __shfl_sync(0xffffffffu, sub, 0);
      __syncwarp();   // memory order: lane 0's ld.acquire loads before the other lanes' reads of sub-epoch data
      if (unit != kStop && (int)sub != slot_sub[b]) {
        // stage the sub-epoch's arguments for slot b (its previous unit is
        // released); L2-only loads: subs[] is written during the launch
        const unsigned long long *src = reinterpret_cast<const unsigned long long *>(&ctl->subs[sub]);
        unsigned long long *dst = reinterpret_cast<unsigned long long *>(&s_args[b]);
        for (int i = lane; i < (int)(sizeof(EpochArgs) / 8); i += 32) dst[i] = __ldcg(src + i);
        __syncwarp();
        slot_sub[b] = (int)sub;
      }
      stage_unit<false>(s_args[b], unit, &s_item[b], s_fac[b], lane);
      if (lane == 0) s_unit[b] = unit;
      __syncwarp();
      bar_arrive(kBarFull + b, 32 + kCompute);
      if (unit == kStop) {
        if (lane == 0) drain_slot<false>(s_args[b ^ 1], st[b ^ 1], &s_empty[b ^ 1]);   // unit u-1 still in flight
        break;
      }
    }
  } else {
    compute_loop<kCompute, kSlotsSW, PF, true>(s_args[0], s_args, s_unit, s_item, s_fac, s_empty, lane);
  }
  // the last CTA to leave: after a close, hand over to the resume launch
  // (reset the launch-wide counts it reuses); otherwise copy every published
  // sub-epoch's counters to its mapped host copy (the host retires the
  // sub-epochs one by one)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ctl->exited, 1u) == gridDim.x - 1) {
      __threadfence();
      if (!resume && (atomicAdd(&ctl->state, 0u) & kStreamClosed)) {
        ctl->state = 0u;
        ctl->exited = 0u;
        ctl->ab_take = 0u;
        __threadfence();
        atomicExch(&ctl->resume, 1u);
        // sub-epoch 0's mapped record: the resume launch did work (its time counts)
        volatile Counters *h0 = reinterpret_cast<volatile Counters *>(
            __ldcg(reinterpret_cast<const unsigned long long *>(&ctl->subs[0].host_ctr)));
        if (h0) h0->pad = 1u;
        __threadfence_system();
      } else {
        const unsigned n = min(__ldcg(&ctl->nsub), ld_acquire_u32(&ctl->published));
        for (unsigned r = 0; r < n; ++r) {
          Counters *c = reinterpret_cast<Counters *>(
              __ldcg(reinterpret_cast<const unsigned long long *>(&ctl->subs[r].ctr)));
          volatile Counters *h = reinterpret_cast<volatile Counters *>(
              __ldcg(reinterpret_cast<const unsigned long long *>(&ctl->subs[r].host_ctr)));
          if (!c || !h) continue;   // published empty (close_stream)
          h->head = atomicAdd(&c->head, 0ull);
          h->tail = atomicAdd(&c->tail, 0ull);
          h->done = atomicAdd(&c->done, 0ull);
          h->error = atomicAdd(&c->error, 0u);
          h->exited = gridDim.x;
        }
        __threadfence_system();
      }
    }
  }
}

// Epoch set-up in one launch: copy the epoch blob from mapped pinned host
// memory with SM loads (optional: used for small blobs, and while chunked
// uploads occupy the host-to-device copy engine, where a memcpy would queue
// behind gigabytes), mark the not-yet-published queue slots EMPTY and zero
// the per-item chunk counters (replaces two memsets).
// Small blocks (64 threads, <= 32 registers) so that the set-up of round r+1
// fits beside round r's persistent CTAs (3 x 288 threads x 72 registers per
// SM) instead of waiting for them to exit.
__global__ void __launch_bounds__(64, 32) stage_kernel(uint4 *dst, const uint4 *src, size_t n16,
                                                    unsigned long long *q_empty, size_t nq, uint32_t *zero,
                                                    size_t nz) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (size_t i = tid; i < n16; i += stride) dst[i] = src[i];
  for (size_t i = tid; i < nq; i += stride) q_empty[i] = Q_EMPTY;
  for (size_t i = tid; i < nz; i += stride) zero[i] = 0u;
}

cudaError_t launch_stage(void *dst, const void *src_mapped, size_t bytes, unsigned long long *q_empty, size_t nq,
                         uint32_t *zero, size_t nz, cudaStream_t stream) {
  const size_t n16 = src_mapped ? (bytes + 15) / 16 : 0;
  size_t work = n16 > nq ? n16 : nq;
  if (nz > work) work = nz;
  const size_t blocks = (work + 63) / 64;
  const int grid = (int)(blocks < 296 ? (blocks > 0 ? blocks : 1) : 296);
  stage_kernel<<<grid, 64, 0, stream>>>(static_cast<uint4 *>(dst), static_cast<const uint4 *>(src_mapped), n16,
                                        q_empty, nq, zero, nz);
  return cudaGetLastError();
}

// Test hook (bt_debug_gate): one thread holds the stream until the host sets
// the mapped word; gives up after watchdog_ns (the stream then runs on).
__global__ void gate_kernel(const volatile unsigned *flag, uint64_t watchdog_ns) {
  const uint64_t t0 = globaltimer();
  while (*flag == 0u && globaltimer() - t0 < watchdog_ns) __nanosleep(1000);
}

cudaError_t launch_gate(const volatile unsigned *flag_dev, uint64_t watchdog_ns, cudaStream_t stream) {
  gate_kernel<<<1, 1, 0, stream>>>(flag_dev, watchdog_ns);
  return cudaGetLastError();
}

// Cross-rank flags (comm.hpp, device protocol) when the driver has no stream
// memory operations: one thread waits until *addr >= value (a peer's write
// into this GPU's flag page), or writes *addr = value after a system-wide
// fence (into a peer's page, after this stream's earlier work).
__global__ void flag_wait_kernel(const uint32_t *addr, uint32_t value, uint64_t watchdog_ns) {
  const uint64_t t0 = globaltimer();
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(addr) : "memory");
    if ((int32_t)(v - value) >= 0 || globaltimer() - t0 > watchdog_ns) break;
    __nanosleep(500);
  }
}
__global__ void flag_write_kernel(uint32_t *addr, uint32_t value) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(addr), "r"(value) : "memory");
}
cudaError_t launch_flag_wait(const uint32_t *addr, uint32_t value, uint64_t watchdog_ns, cudaStream_t stream) {
  flag_wait_kernel<<<1, 1, 0, stream>>>(addr, value, watchdog_ns);
  return cudaGetLastError();
}
cudaError_t launch_flag_write(uint32_t *addr, uint32_t value, cudaStream_t stream) {
  flag_write_kernel<<<1, 1, 0, stream>>>(addr, value);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// "wq": every warp is an independent worker (pop, body, release), for epochs of
// small units (<= 16 KiB): a CTA-wide unit of 4 KiB leaves most threads idle
// and keeps one unit's bytes in flight per CTA; eight warps per CTA each with
// its own unit keep eight (Little's law: the HBM / L2 latency is hidden by
// units in flight, not by threads per unit).  A warp whose release makes a
// single-unit successor ready runs it next itself (no queue round trip); the
// queue ticket for the next pop is taken while the body runs.
#ifndef BT_WQ_MIN_CTAS
#define BT_WQ_MIN_CTAS 4
#endif
#ifndef BT_WQ_U
#define BT_WQ_U 2   // 8-float vectors per lane in flight per step
#endif
constexpr int kBlockWQ = 256, kWarpsWQ = kBlockWQ / 32;
#ifndef BT_TICKET_BLOCK
#define BT_TICKET_BLOCK 4
#endif
constexpr unsigned kTicketBlock = BT_TICKET_BLOCK;   // queue positions per RMW on ctr->head
constexpr unsigned kDoneBatch = 16;                  // completions per RMW on ctr->done

// Release of one finished unit (item, ch) by its warp's lane 0 (the cases of
// release_unit, in one loop as there); returns a ready unit for this warp to
// run next, or kStop.  s0kind: the single successor's meta when prefetched
// (pre: this item and its only successor are single units), else ignored.
// The unit's completion is counted by the caller.
__device__ __forceinline__ unsigned long long release_wq(const EpochArgs &a, uint32_t item, uint32_t ch, const DItem &it,
                                                         uint32_t s0kind, bool pre) {
  const uint32_t nchunks = units_of(it.n, a.chunk_elems);
  bool item_done = true;
  if (nchunks > 1) item_done = atom_add_acq_rel(&a.chunk_done[item], 1u) + 1 == nchunks;
  unsigned long long cont = kStop;
  uint32_t nsucc, off;
  succ_list<true>(a, it.nsucc_field(), it.succ, nsucc, off);
  for (uint32_t i = 0; i < nsucc; ++i) {
    const uint32_t s = nsucc == 1 ? off : __ldg(&a.succ[off + i]);   // single successor inline
    const uint32_t skind = pre ? s0kind : __ldg(&a.items[s].meta);
    uint32_t c0 = 0, c1 = 1;   // units [c0, c1) of s lose this predecessor
    int32_t *cnt = a.pending + s;
    if (nchunks > 1 || !(skind & K_ONE_UNIT)) {
      const uint32_t sn = __ldg(&a.items[s].n);
      const bool chunkwise = nchunks > 1 && !(skind & (K_ONE_UNIT | K_ITEM_DEPS)) && sn == it.n;
      if (chunkwise) {
        c0 = ch;
        c1 = ch + 1;
      } else if (!item_done) {
        continue;
      } else if (!(skind & K_ONE_UNIT)) {
        c1 = units_of(sn, a.chunk_elems);
      }
      if (!(skind & (K_ONE_UNIT | K_SINGLE_PRED))) cnt = a.cpending + __ldg(&a.unit_base[s]);
    }
    const bool one = c1 - c0 == 1;   // a single ready unit: this warp may run it next
    for (uint32_t c = c0; c < c1; ++c) {
      if (!(skind & K_SINGLE_PRED) && atom_add_acq_rel(reinterpret_cast<unsigned *>(cnt + c), 0xFFFFFFFFu) != 1u)
        continue;
      if (one && cont == kStop) {   // run it here next
        cont = ((unsigned long long)s << 32) | c;
        continue;
      }
      const uint32_t e = (skind & K_SINGLE_PRED) ? c1 : c + 1;   // no counters: all at once
      publish_units(a, s, skind, c, e);
      c = e - 1;
    }
  }
  return cont;
}

__global__ void __launch_bounds__(kBlockWQ, BT_WQ_MIN_CTAS) scheduler_kernel_wq(EpochArgs a) {
  __shared__ DItem s_wi[kWarpsWQ];
  __shared__ __align__(16) float s_wf[kWarpsWQ][kMaxFactors];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  DItem *my = &s_wi[w];
  float *fac = s_wf[w];
  unsigned long long ticket = 0;      // lane 0: the queue position this warp pops next
  unsigned tickets = 0;               // lane 0: positions left in its block [ticket, ticket + tickets)
  unsigned ndone = 0;                 // lane 0: units completed, not yet added to ctr->done
  bool grow = false, chained = true;  // lane 0: last popped unit continued / not (ticket block size;
                                      // the first pop takes one position: chains may follow)
  unsigned long long cont = kStop;    // uniform: a local continuation
  bool cont_staged = false;           // uniform: its descriptor is already in *my
  const uint64_t start = globaltimer();
  for (;;) {
    uint64_t g0 = 0;
    long long c0 = 0, c1 = 0, c2 = 0;
    if (a.trace) {
      g0 = globaltimer();
      c0 = clock64();
    }
    unsigned long long unit = cont;
    if (unit == kStop && lane == 0) {
      grow = !chained;
      chained = false;
      for (unsigned spin = 0;; ++spin) {
        if (!tickets) {
          // queue positions are taken kTicketBlock at a time (one RMW on head
          // per block) after a unit that did not continue; one at a time after
          // one that started a chain (a held block would serialise chains)
          const unsigned nb = grow ? kTicketBlock : 1u;
          ticket = atomicAdd(&a.ctr->head, (unsigned long long)nb);
          tickets = nb;
        }
        if (ticket >= a.total_units) break;   // no queue work left for this warp
        unsigned long long v = ld_relaxed_u64(&a.queue[ticket]);
        if (v != Q_EMPTY) {
          v = ld_acquire_u64(&a.queue[ticket]);   // slots are written once: same value, now acquired
          ++ticket;
          --tickets;
          if ((v >> 32) >= a.nitems) {
            raise_error(a, ERR_BAD_UNIT);
            break;
          }
          unit = v;
          break;
        }
        if (ndone) {   // about to wait: account our finished units first (termination reads the sum)
          atomicAdd(&a.ctr->done, (unsigned long long)ndone);
          ndone = 0;
        }
        if ((spin & 15) == 15) {
          // every unit done (the rest ran as continuations): no publication will come
          if (ld_relaxed_u64(&a.ctr->done) == a.total_units) break;
          if (ld_relaxed_u32(&a.ctr->abort)) break;
          if (globaltimer() - start > a.watchdog_ns) {
            raise_error(a, ERR_WATCHDOG);
            break;
          }
        }
        __nanosleep(spin < 32 ? 64 : 256);
      }
      if (unit == kStop && ndone) {
        atomicAdd(&a.ctr->done, (unsigned long long)ndone);
        ndone = 0;
      }
    }
    unit = __shfl_sync(0xffffffffu, unit, 0);
    if (unit == kStop) break;
    cont = kStop;
    // stage the descriptor (lanes 0-2, 16 bytes each; a continuation's was
    // prefetched) and the factor list
    const uint32_t item = (uint32_t)(unit >> 32);
    if (!cont_staged && lane < 2)
      reinterpret_cast<uint4 *>(my)[lane] = __ldg(reinterpret_cast<const uint4 *>(a.items + item) + lane);
    __syncwarp();
    const DItem it = *my;
    const uint32_t kk = it.k();
    // prefetch the single successor's descriptor under the body (lanes 0-1)
    const bool pre = it.nsucc_field() == 1 && (uint64_t)it.n <= a.chunk_elems;
    uint4 nd = {};
    if (pre && lane < 2) nd = __ldg(reinterpret_cast<const uint4 *>(a.items + it.succ) + lane);
    if (it.kind() == K_SCAL) {
      if (kk == 1) {
        if (lane == 0) fac[0] = __uint_as_float(it.arg);   // a single factor travels inline
      } else {
        for (uint32_t j = lane; j < kk; j += 32) fac[j] = __ldg(a.factors + it.arg + j);
      }
      __syncwarp();
    }
    if (a.trace) c1 = clock64();
    const uint32_t chunk = (uint32_t)unit;
    const uint64_t lo = (uint64_t)chunk * a.chunk_elems;
    const uint64_t hi = min((uint64_t)it.n, lo + a.chunk_elems);
    switch (it.kind()) {
      case K_SCAL:
        scal_range<BT_WQ_U, 32>(reinterpret_cast<float *>(it.x) + lo, hi - lo, fac, kk, lane);
        break;
      case K_AXPY:
        axpy_range<32>(reinterpret_cast<const float *>(it.x) + lo, reinterpret_cast<float *>(it.y) + lo, hi - lo,
                       __uint_as_float(it.arg), lane);
        break;
      case K_COPY:
        copy_range<32>(reinterpret_cast<const float *>(it.x) + lo, reinterpret_cast<float *>(it.y) + lo, hi - lo,
                       lane);
        break;
      default:
        if (lane == 0) raise_error(a, ERR_BAD_KIND);
        break;
    }
    // the warp's stores precede lane 0's release (__syncwarp orders memory
    // among the warp's lanes; lane 0's acq_rel operations are cumulative)
    __syncwarp();
    if (a.trace) c2 = clock64();
    const uint32_t s0kind = __shfl_sync(0xffffffffu, nd.y, 1);                          // word 1: n, meta, arg, succ
    if (lane == 0) {
      cont = release_wq(a, item, chunk, it, s0kind, pre);
      chained |= cont != kStop;
      if (++ndone == kDoneBatch) {
        atomicAdd(&a.ctr->done, (unsigned long long)ndone);
        ndone = 0;
      }
    }
    cont = __shfl_sync(0xffffffffu, cont, 0);
    // the continuation is the prefetched successor: its descriptor is ready
    cont_staged = pre && cont != kStop;
    if (a.trace && lane == 0) {
      const long long c3 = clock64();
      const unsigned long long t = (unsigned long long)a.unit_base[item] + chunk;   // the unit's own record
      a.trace[4 * t + 0] = g0;
      a.trace[4 * t + 1] = (unsigned long long)(c1 - c0);
      a.trace[4 * t + 2] = (unsigned long long)(c2 - c1);
      a.trace[4 * t + 3] = (unsigned long long)(c3 - c2);
      a.trace_item[t] = item;
    }
    // the next unit's descriptor overwrites this one's: every lane has read it
    __syncwarp();
    if (cont_staged && lane < 2) reinterpret_cast<uint4 *>(my)[lane] = nd;
  }
  report_exit(a);
}

// Stream launch (runtime.cpp, flush_epoch): the "sw" kernel over the
// sub-epochs the host publishes in *ctl.
cudaError_t launch_stream(StreamCtl *ctl, uint64_t watchdog_ns, uint64_t quiesce_ns, int grid, cudaStream_t stream,
                          bool prefetch, bool resume) {
  if (prefetch) scheduler_kernel_sws<true><<<grid, kBlock, 0, stream>>>(ctl, watchdog_ns, quiesce_ns, resume ? 1 : 0);
  else scheduler_kernel_sws<false><<<grid, kBlock, 0, stream>>>(ctl, watchdog_ns, quiesce_ns, resume ? 1 : 0);
  return cudaGetLastError();
}

// Direct launch (device_abi.h DirectArgs): block (x, y) runs elements
// [x * chunk, (x + 1) * chunk) of item y with the same bodies and the same
// per-element arithmetic as the persistent kernels.
template <class Args>
__global__ void __launch_bounds__(256) direct_kernel(const __grid_constant__ Args p) {
  __shared__ __align__(16) float sf[sizeof(p.factors) / sizeof(float)];
  // item blockIdx.y's group: the last one whose first item is <= it
  uint32_t g0 = 0, g1 = p.nitems - 1;
  while (g0 < g1) {
    const uint32_t mid = (g0 + g1 + 1) >> 1;
    if (p.items[mid].first <= blockIdx.y) g0 = mid;
    else g1 = mid - 1;
  }
  const DirectItem &it = p.items[g0];   // read in place (parameter space): registers for the bodies
  const uint64_t step = (uint64_t)(blockIdx.y - it.first) * it.stride;
  const uint64_t lo = (uint64_t)blockIdx.x * p.chunk;
  if (lo >= it.n) return;
  const uint64_t n = min(it.n - lo, (uint64_t)p.chunk);
  float *const x = reinterpret_cast<float *>(it.x + step) + lo;
  const int tid = threadIdx.x;
  switch (it.kind) {
    case K_SCAL:
      for (uint32_t j = tid; j < it.k; j += blockDim.x) sf[j] = p.factors[it.arg + j];
      __syncthreads();
      // short chains are HBM-bound: keep the next step's loads in flight (as "sws")
      if (it.k < 32) scal_range_pf<2, 256>(x, n, sf, it.k, tid);
      else scal_range<4, 256>(x, n, sf, it.k, tid);
      break;
    case K_AXPY:
      axpy_range<256>(x, reinterpret_cast<float *>(it.y + step) + lo, n, __uint_as_float(it.arg), tid);
      break;
    case K_COPY:
      copy_range<256>(x, reinterpret_cast<float *>(it.y + step) + lo, n, tid);
      break;
    default:
      break;
  }
}

// The smallest parameter block that holds the epoch (the launch copies the
// whole block: C2's 256 items in the 24.6 KB block cost ~20 us of launch).
template <class Small>
bool launch_direct_as(const DirectArgs &args, uint32_t nf, unsigned grid_x, unsigned nall, cudaStream_t stream) {
  constexpr uint32_t kI = sizeof(Small::items) / sizeof(DirectItem), kF = sizeof(Small::factors) / sizeof(float);
  if (args.nitems > kI || nf > kF) return false;
  Small sm;
  sm.nitems = args.nitems;
  sm.chunk = args.chunk;
  memcpy(sm.items, args.items, sizeof(DirectItem) * args.nitems);
  memcpy(sm.factors, args.factors, 4 * nf);
  direct_kernel<Small><<<dim3(grid_x, nall), 256, 0, stream>>>(sm);
  return true;
}

// nall: items (grid.y); args.nitems: their groups
cudaError_t launch_direct(const DirectArgs &args, unsigned grid_x, unsigned nall, cudaStream_t stream) {
  uint32_t nf = 0;   // factors used
  for (uint32_t i = 0; i < args.nitems; ++i)
    if (args.items[i].kind == K_SCAL) nf = max(nf, args.items[i].arg + args.items[i].k);
  if (!launch_direct_as<DirectArgsSmall>(args, nf, grid_x, nall, stream) &&
      !launch_direct_as<DirectArgsT<64, 256>>(args, nf, grid_x, nall, stream) &&
      !launch_direct_as<DirectArgsT<256, 256>>(args, nf, grid_x, nall, stream))
    direct_kernel<DirectArgs><<<dim3(grid_x, nall), 256, 0, stream>>>(args);
  return cudaGetLastError();
}

// Host-side launcher (called from runtime.cpp).
// kernel: 0 = sw, 1 = rw, 2 = wq, 3 = sw with prefetching SCAL bodies (short
// chains); grid in CTAs of that kernel's block size.
cudaError_t launch_epoch(const EpochArgs &args, int grid, cudaStream_t stream, int kernel) {
  if (args.bk) {   // priority ready queue ("sw" bodies)
    if (kernel == 3) scheduler_kernel_swp<true><<<grid, kBlock, 0, stream>>>(args);
    else scheduler_kernel_swp<false><<<grid, kBlock, 0, stream>>>(args);
    return cudaGetLastError();
  }
  if (kernel == 2) scheduler_kernel_wq<<<grid, kBlockWQ, 0, stream>>>(args);
  else if (kernel == 1) scheduler_kernel_rw<<<grid, kBlock, 0, stream>>>(args);
  else if (kernel == 3) scheduler_kernel_sw<true><<<grid, kBlock, 0, stream>>>(args);
  else scheduler_kernel_sw<false><<<grid, kBlock, 0, stream>>>(args);
  return cudaGetLastError();
}

cudaError_t scheduler_occupancy_wq(int *blocks_per_sm, int *block) {
  *block = kBlockWQ;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, scheduler_kernel_wq, kBlockWQ, 0);
}

cudaError_t scheduler_occupancy(int *blocks_per_sm, int *block) {
  *block = kBlock;
  int a = 0, b = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, scheduler_kernel_rw, kBlock, 0);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, scheduler_kernel_sw<false>, kBlock, 0);
  int c = 0;
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, scheduler_kernel_sw<true>, kBlock, 0);
  if (c < b) b = c;
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, scheduler_kernel_swp<false>, kBlock, 0);
  if (c < b) b = c;
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, scheduler_kernel_swp<true>, kBlock, 0);
  if (c < b) b = c;
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, scheduler_kernel_sws<false>, kBlock, 0);
  if (c < b) b = c;
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, scheduler_kernel_sws<true>, kBlock, 0);
  if (c < b) b = c;
  *blocks_per_sm = a < b ? a : b;
  return e;
}

int max_factors() { return kMaxFactors; }

}  // namespace bt
