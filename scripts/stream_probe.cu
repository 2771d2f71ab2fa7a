// stream_probe.cu -- microbenchmark of HBM streaming schemes on sm_100a
// (how to move W through shared memory at the HBM roofline).  Not part of the
// product; results go to profiles/.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sp scripts/stream_probe.cu && /tmp/sp
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(phase) : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// persistent ring: S stages of TB bytes, each stage filled by `pieces` bulk copies
__global__ void k_ring(const double* __restrict__ w, int64_t n, int S, int TB, int pieces, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[16];
  const int64_t per = TB / 8;
  const int64_t nt = n / per;
  const int64_t tb = nt * blockIdx.x / gridDim.x, te = nt * (blockIdx.x + 1) / gridDim.x;
  auto issue = [&](int64_t k) {
    const int st = (int)(k % S);
    mbar_expect_tx(&full[st], (uint32_t)TB);
    const int pb = TB / pieces;
    for (int p = 0; p < pieces; ++p)
      bulk_g2s(sm + (size_t)st * TB + p * pb, (const unsigned char*)(w + k * per) + p * pb, (uint32_t)pb, &full[st]);
  };
  if (threadIdx.x == 0) {
    for (int q = 0; q < S; ++q) mbar_init(&full[q], 1);
    for (int64_t k = tb; k < te && k < tb + S; ++k) issue(k);
  }
  __syncthreads();
  double acc = 0.0;
  uint32_t ph = 0;
  for (int64_t k = tb; k < te; ++k) {
    const int st = (int)(k % S);
    mbar_wait(&full[st], (ph >> st) & 1u);
    ph ^= 1u << st;
    const double* t = (const double*)(sm + (size_t)st * TB);
    acc += t[threadIdx.x] + t[per - 1 - threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && k + S < te) issue(k + S);
  }
  if (acc == 12345.0) sink[0] = acc;
}

// one tile per CTA (the old merge kernel's scheme)
__global__ void k_one(const double* __restrict__ w, int64_t n, int TB, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  const int64_t per = TB / 8;
  const int64_t k = blockIdx.x;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, (uint32_t)TB);
    bulk_g2s(sm, w + k * per, (uint32_t)TB, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  const double* t = (const double*)sm;
  double acc = t[threadIdx.x] + t[per - 1 - threadIdx.x];
  if (acc == 12345.0) sink[0] = acc;
}

// plain 128-bit loads, grid-stride, U-way unrolled
template <int U>
__global__ void k_ldg(const double2* __restrict__ w, int64_t n2, double* sink) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(w + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
  }
  for (; i < n2; i += stride) acc += w[i].x;
  if (acc == 12345.0) sink[0] = acc;
}

int main() {
  const int64_t n = (int64_t)1 << 26;  // 512 MiB of doubles
  double *w, *sink;
  unsigned char* flush;
  cudaMalloc(&w, n * 8);
  cudaMalloc(&sink, 8);
  cudaMalloc(&flush, 256 << 20);
  cudaMemset(w, 0, n * 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k_one, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](const char* name, auto launch) {
    float best = 1e9f;
    for (int r = 0; r < 6; ++r) {
      cudaMemsetAsync(flush, r, 256 << 20);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r > 0 && ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("%-44s %8.1f us  %7.0f GB/s  %s\n", name, best * 1e3, n * 8 / (best * 1e-3) / 1e9,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  char nm[128];
  for (int TBk : {16, 32, 64}) {
    for (int S : {2, 3, 4, 6, 8, 12}) {
      if ((size_t)S * TBk * 1024 > 200 * 1024) continue;
      for (int pieces : {1, 4}) {
        for (int per_sm : {1, 2}) {
          if ((size_t)per_sm * S * TBk * 1024 > 220 * 1024) continue;
          snprintf(nm, sizeof nm, "ring S=%d TB=%dK pieces=%d ctas/sm=%d", S, TBk, pieces, per_sm);
          time(nm, [&] { k_ring<<<sms * per_sm, 256, (size_t)S * TBk * 1024>>>(w, n, S, TBk * 1024, pieces, sink); });
        }
      }
    }
  }
  for (int TBk : {16, 32, 64}) {
    snprintf(nm, sizeof nm, "one-tile-per-CTA TB=%dK", TBk);
    time(nm, [&] { k_one<<<(unsigned)(n * 8 / (TBk * 1024)), 256, (size_t)TBk * 1024>>>(w, n, TBk * 1024, sink); });
  }
  time("ldg128 x4 grid=sms*8 256thr", [&] { k_ldg<4><<<sms * 8, 256>>>((const double2*)w, n / 2, sink); });
  time("ldg128 x8 grid=sms*8 256thr", [&] { k_ldg<8><<<sms * 8, 256>>>((const double2*)w, n / 2, sink); });
  time("ldg128 x8 grid=sms*4 512thr", [&] { k_ldg<8><<<sms * 4, 512>>>((const double2*)w, n / 2, sink); });
  time("ldg128 x16 grid=sms*4 256thr", [&] { k_ldg<16><<<sms * 4, 256>>>((const double2*)w, n / 2, sink); });
  return 0;
}
