// GPU-side launch gap: events around one kernel enqueued right after a 256 MB
// memset (the bench's L2 flush), for an empty kernel and for kernels that need
// large dynamic shared memory.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(int* p) { if (p && threadIdx.x == 1023) p[0] = 1; }
__global__ void k_smem(int* p) {
  extern __shared__ int s[];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (p && threadIdx.x == 1023) p[0] = s[5];
}
int main() {
  void* flush; cudaMalloc(&flush, 256 << 20);
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"empty 129x256", "smem 8KB 129x256", "smem 200KB 129x256", "smem 200KB coop 129x256"};
  for (int v = 0; v < 4; ++v) {
    float best = 1e9, sum = 0; int reps = 50;
    for (int r = 0; r < reps; ++r) {
      cudaMemsetAsync(flush, r, 256 << 20);
      cudaEventRecord(a);
      if (v == 0) k_empty<<<129, 256>>>(nullptr);
      else if (v == 1) k_smem<<<129, 256, 8192>>>(nullptr);
      else if (v == 2) k_smem<<<129, 256, 200 * 1024>>>(nullptr);
      else { int* np = nullptr; void* args[] = {&np}; cudaLaunchCooperativeKernel((void*)k_smem, 129, 256, args, 200 * 1024, 0); }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (r > 2) { best = ms < best ? ms : best; sum += ms; }
    }
    printf("%-26s events: min %.2f us, mean %.2f us\n", names[v], best * 1e3, sum / (reps - 3) * 1e3);
  }
  // the same empty kernel after no flush / a 4 KB memset / a busy kernel
  for (int v = 0; v < 3; ++v) {
    float best = 1e9, sum = 0; int reps = 50;
    for (int r = 0; r < reps; ++r) {
      if (v == 1) cudaMemsetAsync(flush, r, 4096);
      if (v == 2) k_smem<<<148 * 4, 1024, 8192>>>(nullptr);
      cudaEventRecord(a);
      k_empty<<<129, 256>>>(nullptr);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (r > 2) { best = ms < best ? ms : best; sum += ms; }
    }
    const char* nm[] = {"empty, nothing before", "empty, after 4 KB memset", "empty, after a kernel"};
    printf("%-26s events: min %.2f us, mean %.2f us\n", nm[v], best * 1e3, sum / (reps - 3) * 1e3);
  }
  // two events back to back
  {
    float best = 1e9;
    for (int r = 0; r < 20; ++r) {
      cudaMemsetAsync(flush, r, 256 << 20);
      cudaEventRecord(a); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
    }
    printf("%-26s events: min %.2f us\n", "no kernel (after flush)", best * 1e3);
  }
  return 0;
}
