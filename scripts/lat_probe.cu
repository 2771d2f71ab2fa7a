// Latency probe: dependent fp64 add chain, dependent L2 load chain, globaltimer tick.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, const double* buf, unsigned long long* gt) {
  double a = out[0], b = out[1];
  long long t0 = clock64();
#pragma unroll 1
  for (int r = 0; r < 4; ++r) {
#pragma unroll
    for (int i = 0; i < 32; ++i) a = __dadd_rn(a, b);
  }
  long long t1 = clock64();
  out[2] = a;
  // dependent loads (pointer chase in buf, L2-resident)
  long long idx = 0;
  long long t2 = clock64();
  for (int i = 0; i < 64; ++i) idx = __double_as_longlong(__ldcg(buf + idx));
  long long t3 = clock64();
  out[3] = (double)idx;
  float f = out[4], g = out[5];
  long long t4 = clock64();
#pragma unroll
  for (int i = 0; i < 128; ++i) f = __fadd_rn(f, g);
  long long t5 = clock64();
  out[6] = f;
  cyc[0] = (t1 - t0) / 128; cyc[1] = (t3 - t2) / 64; cyc[2] = (t5 - t4) / 128;
  unsigned long long g0, g1; int changes = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  unsigned long long first = g0, last = g0;
  long long c0 = clock64();
  while (changes < 20) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1)); if (g1 != last) { ++changes; last = g1; } }
  long long c1 = clock64();
  gt[0] = last - first; gt[1] = c1 - c0;
}
int main() {
  double *out, *buf; long long* cyc; unsigned long long* gt;
  cudaMalloc(&out, 64); cudaMalloc(&buf, 1 << 20); cudaMallocManaged(&cyc, 64); cudaMallocManaged(&gt, 64);
  double h[8] = {1.0, 1e-9, 0, 0, 1.0f, 1e-6f, 0, 0};
  cudaMemcpy(out, h, 64, cudaMemcpyHostToDevice);
  // chase: buf[i] holds the next index (as bits) with a 4 KB stride
  static double hb[1 << 17];
  for (int i = 0; i < (1 << 17); ++i) { long long nx = (i + 512) % (1 << 17); hb[i] = *(double*)&nx; }
  cudaMemcpy(buf, hb, 1 << 20, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) { k<<<1, 1>>>(out, cyc, buf, gt); cudaDeviceSynchronize(); }
  printf("dadd dependent latency %lld cycles; L2 dependent load %lld cycles; fadd %lld cycles\n", cyc[0], cyc[1], cyc[2]);
  printf("globaltimer: 20 changes spanned %llu ns over %llu cycles -> tick %.1f ns\n", gt[0], gt[1], gt[0] / 20.0);
  return 0;
}
