// One-off B200 probe: device properties, FP32 multiply throughput (FMUL vs
// packed FMUL2), streaming-scale bandwidth with 128/256-bit accesses and the
// canonical NaN pattern.  Measurement tool only -- not part of the product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -lineinfo \
//        tools/probe_b200.cu -o tools/probe_b200 && tools/probe_b200
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

// ---- FP32 multiply throughput -------------------------------------------
template <int NV>
__global__ void fmul_tput(float *out, const float *fac, int iters) {
  float v[NV];
#pragma unroll
  for (int i = 0; i < NV; i++) v[i] = 1.0f + threadIdx.x * 1e-7f + i * 1e-6f;
  float f0 = fac[0], f1 = fac[1];
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NV; i++) v[i] = __fmul_rn(v[i], (it & 1) ? f1 : f0);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NV; i++) s += v[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}

template <int NV>
__global__ void fmul2_tput(float *out, const float *fac, int iters) {
  float2 v[NV];
#pragma unroll
  for (int i = 0; i < NV; i++) v[i] = make_float2(1.0f + threadIdx.x * 1e-7f + i * 1e-6f, 1.0f + i * 1e-5f);
  float2 f0 = make_float2(fac[0], fac[0]), f1 = make_float2(fac[1], fac[1]);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NV; i++) v[i] = __fmul2_rn(v[i], (it & 1) ? f1 : f0);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NV; i++) s += v[i].x + v[i].y;
  if (s == 12345.f) out[threadIdx.x] = s;
}

// ---- streaming scale: x[i] = x[i]*f_1*...*f_k ---------------------------
__device__ __forceinline__ void ld8(const float *p, float (&r)[8]) {
  asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void st8(float *p, const float (&r)[8]) {
  asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
               : "memory");
}

template <bool PACKED>
__global__ void __launch_bounds__(256) scal_v8(float *x, size_t n8, const float *fac, int k) {
  __shared__ float sf[256];
  for (int i = threadIdx.x; i < k; i += blockDim.x) sf[i] = fac[i];
  __syncthreads();
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n8; i += 2 * stride) {
    float a[8], b[8];
    bool hb = i + stride < n8;
    ld8(x + 8 * i, a);
    if (hb) ld8(x + 8 * (i + stride), b);
    for (int j = 0; j < k; j++) {
      float f = sf[j];
      if (PACKED) {
        float2 ff = make_float2(f, f);
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          float2 t = __fmul2_rn(make_float2(a[q], a[q + 1]), ff); a[q] = t.x; a[q + 1] = t.y;
          float2 u = __fmul2_rn(make_float2(b[q], b[q + 1]), ff); b[q] = u.x; b[q + 1] = u.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; q++) { a[q] = __fmul_rn(a[q], f); b[q] = __fmul_rn(b[q], f); }
      }
    }
    st8(x + 8 * i, a);
    if (hb) st8(x + 8 * (i + stride), b);
  }
}

__global__ void __launch_bounds__(256) scal_v4(float4 *x, size_t n4, float f) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 v = __ldcg(x + i);
    v.x = __fmul_rn(v.x, f); v.y = __fmul_rn(v.y, f); v.z = __fmul_rn(v.z, f); v.w = __fmul_rn(v.w, f);
    __stcg(x + i, v);
  }
}

__global__ void nan_probe(const float *in, unsigned *out) {
  out[0] = __float_as_uint(__fmul_rn(in[0], in[1]));   // inf * 0
  out[1] = __float_as_uint(__fadd_rn(in[0], -in[0]));  // inf - inf
  out[2] = __float_as_uint(__fmul_rn(in[2], in[3]));   // subnormal * 3.14f
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0, memclk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, 0);
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_per_sm\":%zu,\"smem_optin\":%zu,"
         "\"regs_per_sm\":%d,\"max_thr_per_sm\":%d,\"clock_khz\":%d,\"mem_clock_khz\":%d,\"bus_bits\":%d,"
         "\"global_mem\":%zu,\"cc\":\"%d.%d\",\"persisting_l2_max\":%d}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerMultiprocessor,
         p.sharedMemPerBlockOptin, p.regsPerMultiprocessor, p.maxThreadsPerMultiProcessor, clk, memclk,
         p.memoryBusWidth, p.totalGlobalMem, p.major, p.minor, p.persistingL2CacheMaxSize);
  int sms = p.multiProcessorCount;

  float *dout, *dfac;
  CK(cudaMalloc(&dout, 4096));
  CK(cudaMalloc(&dfac, 256 * 4));
  float hfac[256];
  for (int i = 0; i < 256; i++) hfac[i] = (i & 1) ? 1.0000001f : 0.9999999f;
  CK(cudaMemcpy(dfac, hfac, sizeof hfac, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;

  // FMUL throughput: blocks = 8*SMs, 256 threads, NV=16 independent chains
  {
    int iters = 4096, blocks = sms * 8, thr = 256;
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      fmul_tput<16><<<blocks, thr>>>(dout, dfac, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    double muls = (double)blocks * thr * 16 * iters;
    printf("{\"probe\":\"fmul\",\"ms\":%.4f,\"Tmul_per_s\":%.2f}\n", ms, muls / ms / 1e9);
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      fmul2_tput<8><<<blocks, thr>>>(dout, dfac, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("{\"probe\":\"fmul2\",\"ms\":%.4f,\"Tmul_per_s\":%.2f}\n", ms, muls / ms / 1e9);
  }

  // streaming scale over 4 GiB
  size_t n = (size_t)1 << 30;
  float *x;
  CK(cudaMalloc(&x, n * 4));
  CK(cudaMemset(x, 0, n * 4));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, scal_v8<true>, 256, 0);
  printf("{\"probe\":\"occ_scal_v8\",\"blocks_per_sm\":%d}\n", occ);
  for (int grid_mult : {2, 4, 8}) {
    int blocks = sms * grid_mult;
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(e0);
      scal_v4<<<blocks, 256>>>((float4 *)x, n / 4, 0.5f);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("{\"probe\":\"scal_v4\",\"grid\":%d,\"ms\":%.4f,\"GBps\":%.1f}\n", blocks, ms, 8.0 * n / ms / 1e6);
  }
  for (int k : {1, 16, 32, 64}) {
    for (int packed = 0; packed < 2; packed++) {
      int blocks = sms * occ;
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        if (packed) scal_v8<true><<<blocks, 256>>>(x, n / 8, dfac, k);
        else scal_v8<false><<<blocks, 256>>>(x, n / 8, dfac, k);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      }
      printf("{\"probe\":\"scal_v8\",\"k\":%d,\"packed\":%d,\"grid\":%d,\"ms\":%.4f,\"GBps\":%.1f,\"Tmul_per_s\":%.2f}\n",
             k, packed, blocks, ms, 8.0 * n / ms / 1e6, (double)n * k / ms / 1e9);
    }
  }
  CK(cudaGetLastError());

  float hin[4];
  unsigned hout[3];
  float inf = __builtin_inff();
  hin[0] = inf; hin[1] = 0.f;
  unsigned sub = 1; memcpy(&hin[2], &sub, 4); hin[3] = 3.14f;
  float *din; unsigned *dno;
  CK(cudaMalloc(&din, 16)); CK(cudaMalloc(&dno, 12));
  CK(cudaMemcpy(din, hin, 16, cudaMemcpyHostToDevice));
  nan_probe<<<1, 1>>>(din, dno);
  CK(cudaMemcpy(hout, dno, 12, cudaMemcpyDeviceToHost));
  printf("{\"probe\":\"nan\",\"inf_x_0\":\"0x%08X\",\"inf_minus_inf\":\"0x%08X\",\"sub1_x_3.14\":\"0x%08X\"}\n",
         hout[0], hout[1], hout[2]);
  return 0;
}
