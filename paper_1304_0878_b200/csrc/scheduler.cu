// scheduler.cu -- the persistent sm_100a scheduler kernel and its task bodies.
//
// One launch executes one epoch: a DAG of work items built on the host from
// the submission order (runtime.cpp).  Every resident CTA loops:
//
//   pop    t = atomicAdd(head, 1); spin on ld.acquire(queue[t]) until the unit
//          (item, chunk) is published; t >= total_units ends the CTA.
//   body   run the item's task body on its chunk of elements:
//            SCAL   x[i] = x[i]*f_1*...*f_k   (k sequential RN multiplies,
//                   submission order: PAPER.md:157-158; a fused chain of k
//                   vector_scal tasks is exactly k roundings per element)
//            AXPY   y[i] = fl(fl(a*x[i]) + y[i])
//            COPY   y[i] = x[i]
//   release when the item's last chunk is done, decrement each successor's
//          pending counter; a successor reaching 0 is ready: its chunks are
//          appended to the queue (atomicAdd(tail, nchunks) + stores after a
//          gpu-scope fence).
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

constexpr int kBlock = 256;
constexpr int kMaxFactors = 1024;      // upper bound of bt_config.max_fused
constexpr unsigned long long kStop = ~0ull - 1;

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
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

__device__ void scal_range(float *x, uint64_t n, const float *sf, uint32_t k) {
  const int tid = threadIdx.x;
  const uint64_t head = head_elems(x, n);
  for (uint64_t i = tid; i < head; i += kBlock) __stcg(x + i, chain_scalar(__ldcg(x + i), sf, k));
  float *xv = x + head;
  const uint64_t nv = (n - head) >> 3;
  constexpr int U = 2;
  uint64_t i = tid;
  for (; i + (U - 1) * kBlock < nv; i += U * kBlock) {
    float v[U][8];
#pragma unroll
    for (int a = 0; a < U; ++a) ld8(xv + 8 * (i + a * kBlock), v[a]);
    chain_apply<U>(v, sf, k);
#pragma unroll
    for (int a = 0; a < U; ++a) st8(xv + 8 * (i + a * kBlock), v[a]);
  }
  for (; i < nv; i += kBlock) {
    float v[1][8];
    ld8(xv + 8 * i, v[0]);
    chain_apply<1>(v, sf, k);
    st8(xv + 8 * i, v[0]);
  }
  for (uint64_t t = head + 8 * nv + tid; t < n; t += kBlock) __stcg(x + t, chain_scalar(__ldcg(x + t), sf, k));
}

// AXPY: y[i] = fl(fl(a*x[i]) + y[i]) (two roundings, no FFMA).
__device__ __forceinline__ float axpy1(float a, float x, float y) { return __fadd_rn(__fmul_rn(a, x), y); }

__device__ void axpy_range(const float *x, float *y, uint64_t n, float a) {
  const int tid = threadIdx.x;
  if (((reinterpret_cast<uintptr_t>(x) ^ reinterpret_cast<uintptr_t>(y)) & 31u) != 0) {
    for (uint64_t i = tid; i < n; i += kBlock) __stcg(y + i, axpy1(a, __ldcg(x + i), __ldcg(y + i)));
    return;
  }
  const uint64_t head = head_elems(y, n);
  for (uint64_t i = tid; i < head; i += kBlock) __stcg(y + i, axpy1(a, __ldcg(x + i), __ldcg(y + i)));
  const float *xv = x + head;
  float *yv = y + head;
  const uint64_t nv = (n - head) >> 3;
  for (uint64_t i = tid; i < nv; i += kBlock) {
    float xr[8], yr[8];
    ld8(xv + 8 * i, xr);
    ld8(yv + 8 * i, yr);
#pragma unroll
    for (int q = 0; q < 8; ++q) yr[q] = axpy1(a, xr[q], yr[q]);
    st8(yv + 8 * i, yr);
  }
  for (uint64_t t = head + 8 * nv + tid; t < n; t += kBlock) __stcg(y + t, axpy1(a, __ldcg(x + t), __ldcg(y + t)));
}

__device__ void copy_range(const float *x, float *y, uint64_t n) {
  const int tid = threadIdx.x;
  if (x == y) return;
  if (((reinterpret_cast<uintptr_t>(x) ^ reinterpret_cast<uintptr_t>(y)) & 31u) != 0) {
    for (uint64_t i = tid; i < n; i += kBlock) __stcg(y + i, __ldcg(x + i));
    return;
  }
  const uint64_t head = head_elems(y, n);
  for (uint64_t i = tid; i < head; i += kBlock) __stcg(y + i, __ldcg(x + i));
  const float *xv = x + head;
  float *yv = y + head;
  const uint64_t nv = (n - head) >> 3;
  uint64_t i = tid;
  for (; i + kBlock < nv; i += 2 * kBlock) {
    float a[8], b[8];
    ld8(xv + 8 * i, a);
    ld8(xv + 8 * (i + kBlock), b);
    st8(yv + 8 * i, a);
    st8(yv + 8 * (i + kBlock), b);
  }
  for (; i < nv; i += kBlock) {
    float a[8];
    ld8(xv + 8 * i, a);
    st8(yv + 8 * i, a);
  }
  for (uint64_t t = head + 8 * nv + tid; t < n; t += kBlock) __stcg(y + t, __ldcg(x + t));
}

// ---- release: completion of one unit (called by thread 0 after bar.sync) --
// Memory-model pattern (as in cooperative-groups grid sync): the CTA's stores
// are ordered before thread 0's gpu-scope fence by bar.sync; fence + relaxed
// RMW = release; RMW observing the last decrement + fence = acquire.
__device__ __forceinline__ void release_unit(const EpochArgs &a, uint32_t item, const DItem &it) {
  __threadfence();
  if (it.nchunks > 1) {
    const unsigned c = atomicAdd(&a.chunk_done[item], 1u);
    if (c + 1 != it.nchunks) return;
    __threadfence();  // acquire the other chunks' stores before releasing them on
  }
  for (uint32_t i = 0; i < it.nsucc; ++i) {
    const uint32_t s = __ldg(&a.succ[it.succ_off + i]);
    if (atomicSub(&a.pending[s], 1) == 1) {
      __threadfence();
      const uint32_t nc = __ldg(&a.items[s].nchunks);
      const unsigned long long pos = atomicAdd(&a.ctr->tail, (unsigned long long)nc);
      for (uint32_t c = 0; c < nc; ++c)
        st_relaxed_u64(&a.queue[pos + c], ((unsigned long long)s << 32) | c);
    }
  }
}

__device__ __forceinline__ void raise_error(const EpochArgs &a, unsigned code) {
  atomicCAS(&a.ctr->error, 0u, code);
  atomicExch(&a.ctr->abort, 1u);
}

__global__ void __launch_bounds__(kBlock) scheduler_kernel(EpochArgs a) {
  __shared__ unsigned long long s_unit;
  __shared__ unsigned long long s_ticket;
  __shared__ __align__(16) float s_fac[kMaxFactors];
  const int tid = threadIdx.x;
  uint64_t g0 = 0;
  long long c0 = 0, c1 = 0, c2 = 0;

  for (;;) {
    if (tid == 0) {
      if (a.trace) { g0 = globaltimer(); c0 = clock64(); }
      unsigned long long u = kStop;
      const unsigned long long t = atomicAdd(&a.ctr->head, 1ull);
      if (t < a.total_units) {
        u = ld_acquire_u64(&a.queue[t]);
        if (u == Q_EMPTY) {
          const uint64_t start = globaltimer();
          for (unsigned spin = 0;; ++spin) {
            __nanosleep(spin < 64 ? 32 : 256);
            u = ld_acquire_u64(&a.queue[t]);
            if (u != Q_EMPTY) break;
            if ((spin & 63) == 63) {
              if (ld_volatile_u32(&a.ctr->abort)) { u = kStop; break; }
              if (globaltimer() - start > a.watchdog_ns) { raise_error(a, ERR_WATCHDOG); u = kStop; break; }
            }
          }
        }
        if (u != kStop && (u >> 32) >= a.nitems) { raise_error(a, ERR_BAD_UNIT); u = kStop; }
      }
      s_unit = u;
      s_ticket = t;
      if (a.trace) c1 = clock64();
    }
    __syncthreads();
    const unsigned long long u = s_unit;
    if (u == kStop) break;
    const uint32_t item = (uint32_t)(u >> 32);
    const uint32_t chunk = (uint32_t)u;
    const DItem it = a.items[item];
    const uint64_t b = (uint64_t)chunk * a.chunk_elems;
    const uint64_t e = min(it.n, b + a.chunk_elems);
    switch (it.kind) {
      case K_SCAL: {
        const uint32_t k = it.k;
        for (uint32_t j = tid; j < k; j += kBlock) s_fac[j] = __ldg(a.factors + it.arg + j);
        __syncthreads();
        scal_range(reinterpret_cast<float *>(it.x) + b, e - b, s_fac, k);
        break;
      }
      case K_AXPY:
        axpy_range(reinterpret_cast<const float *>(it.x) + b, reinterpret_cast<float *>(it.y) + b, e - b,
                   __uint_as_float(it.arg));
        break;
      case K_COPY:
        copy_range(reinterpret_cast<const float *>(it.x) + b, reinterpret_cast<float *>(it.y) + b, e - b);
        break;
      default:
        if (tid == 0) raise_error(a, ERR_BAD_KIND);
        break;
    }
    __syncthreads();
    if (tid == 0) {
      if (a.trace) c2 = clock64();
      release_unit(a, item, it);
      if (a.trace) {
        const unsigned long long t = s_ticket;
        const long long c3 = clock64();
        a.trace[4 * t + 0] = g0;
        a.trace[4 * t + 1] = (unsigned long long)(c1 - c0);
        a.trace[4 * t + 2] = (unsigned long long)(c2 - c1);
        a.trace[4 * t + 3] = (unsigned long long)(c3 - c2);
        a.trace_item[t] = item;
      }
    }
  }
}

// Host-side launcher (called from runtime.cpp).
cudaError_t launch_epoch(const EpochArgs &args, int grid, cudaStream_t stream) {
  scheduler_kernel<<<grid, kBlock, 0, stream>>>(args);
  return cudaGetLastError();
}

cudaError_t scheduler_occupancy(int *blocks_per_sm, int *block) {
  *block = kBlock;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, scheduler_kernel, kBlock, 0);
}

int max_factors() { return kMaxFactors; }

}  // namespace bt
