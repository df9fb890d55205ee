// Probe: C3's data movement without its dependencies.  The jobs are the C3
// tasks' 64 KiB work units (SCAL in place / AXPY / COPY over 64 x 4 MiB
// buffers), in submission order or shuffled, dispatched to persistent CTAs
// from one atomic counter -- no DAG, no release.  Its time bounds what C3 can
// reach with this unit size and access pattern (C3).  Measurement
// tool only: not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -lineinfo \
//        tools/chunk_probe.cu -o tools/chunk_probe
//   python tools/chunk_probe.py        (writes the job list from workloads.c3_random_dag, runs it)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

struct Job { uint32_t kind, x, y, chunk; float a; };   // kind 1 SCAL, 2 AXPY, 3 COPY

constexpr int kThreads = 256;
constexpr int kChunk = 16384;   // floats (64 KiB)

__global__ void __launch_bounds__(kThreads) run_jobs(const Job *jobs, uint32_t njobs, float *const *bufs,
                                                     unsigned *next) {
  __shared__ uint32_t s_j;
  for (;;) {
    if (threadIdx.x == 0) s_j = atomicAdd(next, 1u);
    __syncthreads();
    const uint32_t j = s_j;
    __syncthreads();
    if (j >= njobs) return;
    const Job jb = jobs[j];
    const float4 *x = reinterpret_cast<const float4 *>(bufs[jb.x] + (size_t)jb.chunk * kChunk);
    float4 *y = reinterpret_cast<float4 *>(bufs[jb.y] + (size_t)jb.chunk * kChunk);
    float4 *xs = reinterpret_cast<float4 *>(bufs[jb.x] + (size_t)jb.chunk * kChunk);
    constexpr int n4 = kChunk / 4;   // 4096 float4 = 16 per thread
#pragma unroll 4
    for (int i = threadIdx.x; i < n4; i += kThreads) {
      if (jb.kind == 1) {
        float4 v = __ldcg(xs + i);
        v.x = __fmul_rn(v.x, jb.a); v.y = __fmul_rn(v.y, jb.a); v.z = __fmul_rn(v.z, jb.a); v.w = __fmul_rn(v.w, jb.a);
        __stcg(xs + i, v);
      } else if (jb.kind == 2) {
        const float4 u = __ldcg(x + i);
        float4 v = __ldcg(y + i);
        v.x = __fadd_rn(__fmul_rn(jb.a, u.x), v.x); v.y = __fadd_rn(__fmul_rn(jb.a, u.y), v.y);
        v.z = __fadd_rn(__fmul_rn(jb.a, u.z), v.z); v.w = __fadd_rn(__fmul_rn(jb.a, u.w), v.w);
        __stcg(y + i, v);
      } else {
        __stcg(y + i, __ldcg(x + i));
      }
    }
  }
}

// The same, with the next job claimed one step ahead and its operands
// prefetched into L2 by one bulk prefetch per operand (no registers, no shared
// memory) while the current job runs.
__device__ __forceinline__ void prefetch_l2(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__(kThreads) run_jobs_pf(const Job *jobs, uint32_t njobs, float *const *bufs,
                                                        unsigned *next, int pf_bytes) {
  __shared__ uint32_t s_j[2];
  if (threadIdx.x == 0) {
    s_j[0] = atomicAdd(next, 1u);
    s_j[1] = atomicAdd(next, 1u);
  }
  __syncthreads();
  for (unsigned it = 0;; ++it) {
    const uint32_t j = s_j[it & 1], jn = s_j[(it + 1) & 1];
    if (j >= njobs) return;
    if (threadIdx.x == 0 && jn < njobs) {
      const Job n = jobs[jn];
      prefetch_l2(bufs[n.x] + (size_t)n.chunk * kChunk, pf_bytes);
      if (n.kind == 2) prefetch_l2(bufs[n.y] + (size_t)n.chunk * kChunk, pf_bytes);
    }
    const Job jb = jobs[j];
    const float4 *x = reinterpret_cast<const float4 *>(bufs[jb.x] + (size_t)jb.chunk * kChunk);
    float4 *y = reinterpret_cast<float4 *>(bufs[jb.y] + (size_t)jb.chunk * kChunk);
    float4 *xs = reinterpret_cast<float4 *>(bufs[jb.x] + (size_t)jb.chunk * kChunk);
    constexpr int n4 = kChunk / 4;
#pragma unroll 4
    for (int i = threadIdx.x; i < n4; i += kThreads) {
      if (jb.kind == 1) {
        float4 v = __ldcg(xs + i);
        v.x = __fmul_rn(v.x, jb.a); v.y = __fmul_rn(v.y, jb.a); v.z = __fmul_rn(v.z, jb.a); v.w = __fmul_rn(v.w, jb.a);
        __stcg(xs + i, v);
      } else if (jb.kind == 2) {
        const float4 u = __ldcg(x + i);
        float4 v = __ldcg(y + i);
        v.x = __fadd_rn(__fmul_rn(jb.a, u.x), v.x); v.y = __fadd_rn(__fmul_rn(jb.a, u.y), v.y);
        v.z = __fadd_rn(__fmul_rn(jb.a, u.z), v.z); v.w = __fadd_rn(__fmul_rn(jb.a, u.w), v.w);
        __stcg(y + i, v);
      } else {
        __stcg(y + i, __ldcg(x + i));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_j[it & 1] = atomicAdd(next, 1u);   // the job after jn
    __syncthreads();
  }
}

// The same with the operands staged through shared memory by cp.async
// (LDGSTS: no registers hold the bytes in flight): NS stages of SB float4 per
// operand, NS-1 stages in flight while one is consumed.
__device__ __forceinline__ void cp16(void *smem, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NS, int SB>   // SB float4 per stage and operand (multiple of kThreads)
__global__ void __launch_bounds__(kThreads) run_jobs_cp(const Job *jobs, uint32_t njobs, float *const *bufs,
                                                        unsigned *next) {
  extern __shared__ float4 sm[];   // [NS][2][SB]
  __shared__ uint32_t s_j;
  constexpr int n4 = kChunk / 4, nst = n4 / SB, per = SB / kThreads;
  for (;;) {
    if (threadIdx.x == 0) s_j = atomicAdd(next, 1u);
    __syncthreads();
    const uint32_t j = s_j;
    __syncthreads();
    if (j >= njobs) return;
    const Job jb = jobs[j];
    const float4 *x = reinterpret_cast<const float4 *>(bufs[jb.x] + (size_t)jb.chunk * kChunk);
    float4 *y = reinterpret_cast<float4 *>(bufs[jb.y] + (size_t)jb.chunk * kChunk);
    const bool two = jb.kind == 2;
    auto issue = [&](int st) {
      float4 *bx = sm + (size_t)(st % NS) * 2 * SB, *by = bx + SB;
#pragma unroll
      for (int q = 0; q < per; ++q) {
        const int i = st * SB + q * kThreads + threadIdx.x;
        cp16(bx + q * kThreads + threadIdx.x, x + i);
        if (two) cp16(by + q * kThreads + threadIdx.x, y + i);
      }
    };
#pragma unroll
    for (int st = 0; st < NS - 1; ++st) {
      if (st < nst) issue(st);
      cp_commit();
    }
    for (int st = 0; st < nst; ++st) {
      if (st + NS - 1 < nst) issue(st + NS - 1);
      cp_commit();
      cp_wait<NS - 1>();   // stage st has landed (each thread reads only what it copied)
      const float4 *bx = sm + (size_t)(st % NS) * 2 * SB, *by = bx + SB;
#pragma unroll
      for (int q = 0; q < per; ++q) {
        const int k = q * kThreads + threadIdx.x, i = st * SB + k;
        float4 v = bx[k];
        if (jb.kind == 1) {
          v.x = __fmul_rn(v.x, jb.a); v.y = __fmul_rn(v.y, jb.a); v.z = __fmul_rn(v.z, jb.a); v.w = __fmul_rn(v.w, jb.a);
          __stcg(y + i, v);
        } else if (two) {
          float4 w = by[k];
          w.x = __fadd_rn(__fmul_rn(jb.a, v.x), w.x); w.y = __fadd_rn(__fmul_rn(jb.a, v.y), w.y);
          w.z = __fadd_rn(__fmul_rn(jb.a, v.z), w.z); w.w = __fadd_rn(__fmul_rn(jb.a, v.w), w.w);
          __stcg(y + i, w);
        } else {
          __stcg(y + i, v);
        }
      }
    }
    cp_wait<0>();
  }
}

// read-only L2 eviction (a written scratch would leave dirty lines behind)
__global__ void touch(const float4 *p, size_t n4, float *out) {
  float s = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = __ldcg(p + i);
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 1234.5f) *out = s;
}

int main(int argc, char **argv) {
  if (argc < 2) {
    printf("usage: chunk_probe jobs.bin [reps]\n");
    return 2;
  }
  FILE *f = fopen(argv[1], "rb");
  if (!f) return 2;
  uint32_t nbuf, njobs;
  if (fread(&nbuf, 4, 1, f) != 1 || fread(&njobs, 4, 1, f) != 1) return 2;
  std::vector<Job> jobs(njobs);
  if (fread(jobs.data(), sizeof(Job), njobs, f) != njobs) return 2;
  fclose(f);
  const int reps = argc > 2 ? atoi(argv[2]) : 5;
  int sms = 0, occ = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, run_jobs, kThreads, 0));
  std::vector<float *> hb(nbuf);
  for (uint32_t b = 0; b < nbuf; ++b) {
    CK(cudaMalloc(&hb[b], (size_t)4 << 20));
    CK(cudaMemset(hb[b], 0x3f, (size_t)4 << 20));
  }
  float **db;
  Job *dj;
  unsigned *next;
  CK(cudaMalloc(&db, nbuf * sizeof(float *)));
  CK(cudaMemcpy(db, hb.data(), nbuf * sizeof(float *), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&dj, njobs * sizeof(Job)));
  CK(cudaMemcpy(dj, jobs.data(), njobs * sizeof(Job), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&next, 4));
  // evict L2 between reps by reading 512 MiB
  float *flush;
  CK(cudaMalloc(&flush, (size_t)512 << 20));
  CK(cudaMemset(flush, 0, (size_t)512 << 20));
  double bytes = 0;
  for (const Job &j : jobs) bytes += (j.kind == 2 ? 12.0 : 8.0) * kChunk;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int grid_mul : {occ, 3, 2}) {
    const int grid = sms * grid_mul;
    std::vector<float> ms;
    for (int r = 0; r < reps + 1; ++r) {
      touch<<<sms * 4, 256>>>(reinterpret_cast<const float4 *>(flush), ((size_t)512 << 20) / 16, flush);
      CK(cudaMemset(next, 0, 4));
      CK(cudaEventRecord(e0));
      run_jobs<<<grid, kThreads>>>(dj, njobs, db, next);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float t;
      CK(cudaEventElapsedTime(&t, e0, e1));
      if (r) ms.push_back(t);
    }
    std::vector<float> s = ms;
    std::sort(s.begin(), s.end());
    const float med = s[s.size() / 2];
    printf("{\"probe\":\"c3_jobs_no_deps\",\"file\":\"%s\",\"jobs\":%u,\"ctas_per_sm\":%d,\"grid\":%d,\"ms\":%.3f,"
           "\"algorithmic_GBps\":%.1f}\n",
           argv[1], njobs, grid_mul, grid, med, bytes / med / 1e6);
  }
  auto run_cp = [&](auto kern, int ns, int sb, int grid_mul) -> int {
    const size_t smem = (size_t)ns * 2 * sb * 16;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ2 = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, kern, kThreads, smem));
    const int gm = std::min(grid_mul, occ2);
    std::vector<float> ms;
    for (int r = 0; r < reps + 1; ++r) {
      touch<<<sms * 4, 256>>>(reinterpret_cast<const float4 *>(flush), ((size_t)512 << 20) / 16, flush);
      CK(cudaMemset(next, 0, 4));
      CK(cudaEventRecord(e0));
      kern<<<sms * gm, kThreads, smem>>>(dj, njobs, db, next);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float t;
      CK(cudaEventElapsedTime(&t, e0, e1));
      if (r) ms.push_back(t);
    }
    std::sort(ms.begin(), ms.end());
    const float med = ms[ms.size() / 2];
    printf("{\"probe\":\"c3_jobs_no_deps_cp_async\",\"file\":\"%s\",\"stages\":%d,\"stage_bytes_per_operand\":%d,"
           "\"ctas_per_sm\":%d,\"ms\":%.3f,\"algorithmic_GBps\":%.1f}\n",
           argv[1], ns, sb * 16, gm, med, bytes / med / 1e6);
    return 0;
  };
  run_cp(run_jobs_cp<4, 512>, 4, 512, 3);     // 4 x 8 KiB per operand: 64 KiB per CTA
  run_cp(run_jobs_cp<3, 1024>, 3, 1024, 3);   // 3 x 16 KiB: 96 KiB (2 CTAs/SM fit)
  run_cp(run_jobs_cp<8, 256>, 8, 256, 3);     // 8 x 4 KiB: 64 KiB
  run_cp(run_jobs_cp<4, 256>, 4, 256, 3);     // 4 x 4 KiB: 32 KiB
  for (int grid_mul : {3, 2}) {
    for (int pf : {16384, 65536}) {
      const int grid = sms * grid_mul;
      std::vector<float> ms;
      for (int r = 0; r < reps + 1; ++r) {
        touch<<<sms * 4, 256>>>(reinterpret_cast<const float4 *>(flush), ((size_t)512 << 20) / 16, flush);
        CK(cudaMemset(next, 0, 4));
        CK(cudaEventRecord(e0));
        run_jobs_pf<<<grid, kThreads>>>(dj, njobs, db, next, pf);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float t;
        CK(cudaEventElapsedTime(&t, e0, e1));
        if (r) ms.push_back(t);
      }
      std::sort(ms.begin(), ms.end());
      const float med = ms[ms.size() / 2];
      printf("{\"probe\":\"c3_jobs_no_deps_l2_prefetch\",\"file\":\"%s\",\"prefetch_bytes\":%d,\"ctas_per_sm\":%d,"
             "\"grid\":%d,\"ms\":%.3f,\"algorithmic_GBps\":%.1f}\n",
             argv[1], pf, grid_mul, grid, med, bytes / med / 1e6);
    }
  }
  return 0;
}
