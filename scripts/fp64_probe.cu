// fp64 dependent-chain latency and throughput with W warps per SM (one CTA per SM).
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void k(double* out, long long* cyc, int iters) {
  double a[ILP], b = out[1];
#pragma unroll
  for (int j = 0; j < ILP; ++j) a[j] = out[0] + j;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < iters; ++r) {
#pragma unroll
    for (int i = 0; i < 32; ++i)
#pragma unroll
      for (int j = 0; j < ILP; ++j) a[j] = __dadd_rn(a[j], b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += a[j];
  out[2 + threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x % 32 == 0) atomicMax((unsigned long long*)&cyc[0], (unsigned long long)(t1 - t0));
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, (2 + 148 * 1024) * 8); cudaMallocManaged(&cyc, 64);
  double h[2] = {1.0, 1e-9};
  cudaMemcpy(out, h, 16, cudaMemcpyHostToDevice);
  int iters = 64;
  for (int warps : {1, 4, 8, 16, 32}) {
    for (int ilp : {1, 2, 4}) {
      cyc[0] = 0;
      if (ilp == 1) k<1><<<148, warps * 32>>>(out, cyc, iters);
      if (ilp == 2) k<2><<<148, warps * 32>>>(out, cyc, iters);
      if (ilp == 4) k<4><<<148, warps * 32>>>(out, cyc, iters);
      cudaDeviceSynchronize();
      cyc[0] = 0;
      if (ilp == 1) k<1><<<148, warps * 32>>>(out, cyc, iters);
      if (ilp == 2) k<2><<<148, warps * 32>>>(out, cyc, iters);
      if (ilp == 4) k<4><<<148, warps * 32>>>(out, cyc, iters);
      cudaDeviceSynchronize();
      const double per = (double)cyc[0] / (iters * 32);
      printf("warps/SM %2d ILP %d: %.1f cycles per dependent step; %.2f warp-DADD/clk/SM\n", warps, ilp, per,
             warps * ilp / per);
    }
  }
  return 0;
}
