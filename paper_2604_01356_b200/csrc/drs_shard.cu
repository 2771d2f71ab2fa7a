// drs_shard.cu -- W sharded in contiguous ranges over G GPUs (config 5).
//
// Rank g owns W[g*M/G, (g+1)*M/G).  dr_shard_scan (drs_scan.cu) gives the
// local chained prefix S and local total T_g; the caller all-gathers the G
// totals (one double per rank, NCCL over NVLink); every rank then folds
// O_g = T_0 + ... + T_{g-1} and T = O_G in rank order, so each shard's lower
// boundary fl(O_g/T) is bit-identical to the previous shard's last W.
// Sampling regenerates the same U on every rank and each rank matches only
// the u's in (fl(O_g/T), fl(O_{g+1}/T)] -- no further communication.
#include "drs_common.cuh"

namespace drs {

IndexDesc make_index_desc(int64_t M);
int launch_build_index(const double* W, int64_t M, double* idx, cudaStream_t st);

__device__ __forceinline__ void fold_offsets(const double* totals, int G, int g, double& Og,
                                             double& Og1, double& T) {
  double o = 0.0;
  Og = 0.0;
  Og1 = 0.0;
  for (int h = 0; h < G; ++h) {
    if (h == g) Og = o;
    o = __dadd_rn(o, totals[h]);
    if (h == g) Og1 = o;
  }
  T = o;
}

__global__ void k_shard_finalize(double* __restrict__ S, int64_t Mg, const double* __restrict__ totals,
                                 int G, int g) {
  double Og, Og1, T;
  fold_offsets(totals, G, g, Og, Og1, T);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < Mg; j += stride) {
    double v = fmin(__ddiv_rn(__dadd_rn(Og, S[j]), T), 1.0);
    if (g == G - 1 && j == Mg - 1) v = 1.0;
    S[j] = v;
  }
}

__device__ __forceinline__ int64_t warp_count_le_s(const double* __restrict__ U, int64_t N, double key) {
  const int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = N;
  while (hi - lo > 32) {
    const int64_t step = cdiv(hi - lo, 32);
    const int64_t p = lo + (int64_t)(lane + 1) * step - 1;
    const bool pred = (p < hi) && (__ldg(U + p) <= key);
    const int cnt = __popc(__ballot_sync(FULL, pred));
    const int64_t nhi = lo + (int64_t)(cnt + 1) * step - 1;
    lo = lo + (int64_t)cnt * step;
    hi = nhi < hi ? nhi : hi;
  }
  const int64_t p = lo + lane;
  const bool pred = (p < hi) && (__ldg(U + p) <= key);
  return lo + __popc(__ballot_sync(FULL, pred));
}

__global__ void k_shard_range(const double* __restrict__ U, int64_t N, const double* __restrict__ totals,
                              int G, int g, int64_t* range) {
  double Og, Og1, T;
  fold_offsets(totals, G, g, Og, Og1, T);
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    const int64_t v = (g == 0) ? 0 : warp_count_le_s(U, N, fmin(__ddiv_rn(Og, T), 1.0));
    if ((threadIdx.x & 31) == 0) range[0] = v;
  } else if (warp == 1) {
    const int64_t v = (g == G - 1) ? N : warp_count_le_s(U, N, fmin(__ddiv_rn(Og1, T), 1.0));
    if ((threadIdx.x & 31) == 0) range[1] = v;
  }
}

__global__ void __launch_bounds__(256) k_shard_match(const double* __restrict__ W,
                                                     const double* __restrict__ idx, IndexDesc d,
                                                     int64_t shard_start, const double* __restrict__ U,
                                                     const int64_t* __restrict__ range,
                                                     int64_t* __restrict__ out) {
  const int64_t a = range[0], b = range[1];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = a + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += stride)
    out[i] = shard_start + index_lower_bound(W, idx, d, __ldg(U + i));
}

}  // namespace drs

using namespace drs;

extern "C" {

int dr_shard_finalize(double* S_to_W, int64_t Mg, const double* totals, int32_t G, int32_t g,
                      double* idx, void* stream) {
  if (Mg < 1 || !S_to_W || !totals || G < 1 || g < 0 || g >= G) return DRS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t blocks = cdiv(Mg, 256) < 148 * 16 ? cdiv(Mg, 256) : 148 * 16;
  k_shard_finalize<<<(unsigned)blocks, 256, 0, st>>>(S_to_W, Mg, totals, G, g);
  if (cudaGetLastError() != cudaSuccess) return DRS_ERR_LAUNCH;
  return launch_build_index(S_to_W, Mg, idx, st);
}

int dr_shard_range(const double* U, int64_t N, const double* totals, int32_t G, int32_t g,
                   int64_t* range, void* stream) {
  if (N < 0 || !totals || !range || G < 1 || g < 0 || g >= G || (N > 0 && !U)) return DRS_ERR_ARG;
  k_shard_range<<<1, 64, 0, (cudaStream_t)stream>>>(U, N, totals, G, g, range);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

int dr_shard_match(const double* W, const double* idx, int64_t Mg, int64_t shard_start,
                   const double* U, int64_t N, const int64_t* range, int64_t* out, void* stream) {
  if (Mg < 1 || !W || !range || (N > 0 && (!U || !out))) return DRS_ERR_ARG;
  if ((uintptr_t)W & 31) return DRS_ERR_ALIGN;
  if (N == 0) return DRS_OK;
  const IndexDesc d = make_index_desc(Mg);
  if (d.levels > 0 && !idx) return DRS_ERR_ARG;
  const int64_t blocks = cdiv(N, 256) < 148 * 16 ? cdiv(N, 256) : 148 * 16;
  k_shard_match<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(W, idx, d, shard_start, U, range, out);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

}  // extern "C"
