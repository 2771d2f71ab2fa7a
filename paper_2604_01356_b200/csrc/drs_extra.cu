// drs_extra.cu -- the steps either side of the resampling path.
//
//   gather          the step after resampling: particle states by index
//                   ("trivial"; EnGMF rows of d = 40 fp64,
//                   weightgen.py:37), out[i] = states[idx[i] / divisor].
//   histogram       np.bincount(indices, minlength=M) (bench.py:241) on the
//                   device: warp-aggregated atomics (equal indices of a warp
//                   -- sorted samplers produce long runs -- add once).
//   chi_square      chi_square_statistic(counts, n * weights) (bench.py:221-225,
//                   expected from table.weights() = diff(W, prepend 0),
//                   cdf.py:51-53), reduced deterministically (fixed tree).
#include "drs_common.cuh"

namespace drs {

static int launch_rc_x() {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

// one thread per 16-byte (or 8-byte) element of the output: stores fully
// coalesced, each source row read as one contiguous run
template <typename V>
__global__ void __launch_bounds__(256) k_gather_rows(const V* __restrict__ states, int64_t K, int64_t dv,
                                                     const int64_t* __restrict__ idx, int64_t N,
                                                     int64_t divisor, V* __restrict__ out, int32_t* status) {
  // flat over the N x dv destination elements: consecutive threads write
  // consecutive elements, and a sorted index vector reads rows in order (a
  // warp-per-64-rows variant with batched row reads measured 2x slower here
  // at 1 CTA/SM; the fused sampler uses that scheme, gather_warp_rows)
  const int64_t total = N * dv;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t i = e / dv, k = e - i * dv;
    const int64_t x = __ldg(idx + i);
    const int64_t src = x / divisor;
    if (x < 0 || src >= K) {
      if (k == 0) atomicOr(status, DRS_ST_OUT_OF_SUPPORT);
      continue;
    }
    out[e] = __ldg(states + src * dv + k);
  }
}

__global__ void __launch_bounds__(256) k_histogram(const int64_t* __restrict__ idx, int64_t N, int64_t M,
                                                   unsigned long long* __restrict__ counts, int32_t* status) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < N; base += stride) {
    const int64_t i = base + threadIdx.x;
    const int64_t j = (i < N) ? __ldg(idx + i) : -1;
    const bool ok = (i < N) && j >= 0 && j < M;
    if (i < N && !ok) atomicOr(status, DRS_ST_OUT_OF_SUPPORT);
    const unsigned act = __ballot_sync(FULL, ok);
    if (!ok) continue;
    // lanes holding the same index: the lowest adds the group size
    const unsigned peers = __match_any_sync(act, (unsigned long long)j);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(counts + j, (unsigned long long)__popc(peers));
  }
}

// per-bin Pearson terms, then a fixed two-level tree: 256-thread blocks over
// contiguous bins, block partials summed in block order by one thread
constexpr int CHI_THREADS = 256;

__global__ void __launch_bounds__(CHI_THREADS) k_chi_partial(const unsigned long long* __restrict__ counts,
                                                             const double* __restrict__ W, int64_t M,
                                                             double n, double* __restrict__ partial) {
  __shared__ double red[CHI_THREADS];
  const int64_t per = (int64_t)gridDim.x;
  double acc = 0.0;
  // block b takes bins [b*M/g, (b+1)*M/g); thread t folds its strided bins in order
  const int64_t b0 = M * blockIdx.x / per, b1 = M * (blockIdx.x + 1) / per;
  for (int64_t j = b0 + threadIdx.x; j < b1; j += CHI_THREADS) {
    const double wj = (j == 0) ? W[0] : __dsub_rn(W[j], W[j - 1]);
    const double e = __dmul_rn(n, wj);
    const double dlt = __dsub_rn((double)counts[j], e);
    acc = __dadd_rn(acc, __ddiv_rn(__dmul_rn(dlt, dlt), e));
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = CHI_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void k_chi_final(const double* __restrict__ partial, int nb, double* out) {
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s = __dadd_rn(s, partial[b]);
  *out = s;
}

// ---------------------------------------------------------- op counts ----
// The reference's OpStats for its instrumented CPU twins (samplers.py:40-46,
// 178-188, 213-232, 249-252; cdf.py:116-125), reproduced EXACTLY from the
// device result: every count is a function of W, u and the lower bounds.
//   ccf     comparisons = out[n-1] + n (the cursor advances to out[n-1], one
//           closing comparison per u: samplers.py:178-186);
//   binary  probes = sum over u of the bisection steps of upper_bound_search
//           on [0, M-1] (samplers.py:249-252);
//   dac     the work list of _dac_instrumented visits the implicit median
//           tree of [0, n-1]; the scope of median m is [a_u, b_u] (its tree
//           node) with W range [out[a_u-1] or 0, out[b_u+1] or M-1] (each
//           bound is an ancestor's match), m is visited iff its parent's W
//           range is not a single index (else the parent filled it), and a
//           visited m costs the bisection steps over its W range (0 when the
//           range is one index); max_depth = the deepest visited node.
// counts[0] comparisons, [1] probes, [2] max_depth (accumulated with atomics).
__device__ __forceinline__ unsigned long long bisect_probes(const double* __restrict__ W, int64_t a, int64_t b,
                                                            double x) {
  unsigned long long p = 0;
  while (a != b) {
    const int64_t m = (a + b) >> 1;  // floor((a + b) / 2) for a, b >= 0
    ++p;
    if (__ldg(W + m) < x) a = m + 1;
    else b = m;
  }
  return p;
}

__global__ void __launch_bounds__(256) k_op_counts(int kind, const double* __restrict__ W, int64_t M,
                                                   const double* __restrict__ u, int64_t n,
                                                   const int64_t* __restrict__ out,
                                                   unsigned long long* counts) {
  unsigned long long probes = 0, depth = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; kind != 1 && m < n; m += stride) {
    if (kind == 2) {  // binary
      probes += bisect_probes(W, 0, M - 1, __ldg(u + m));
      continue;
    }
    // the node of median m in the tree of [0, n-1], and its parent's scope
    int64_t a = 0, b = n - 1, pa = -1, pb = -1;
    unsigned long long d = 1;
    while (true) {
      const int64_t mid = (a + b) >> 1;
      if (mid == m) break;
      pa = a;
      pb = b;
      if (m < mid) b = mid - 1;
      else a = mid + 1;
      ++d;
    }
    if (pa >= 0) {  // visited only when the parent's W range was not one index
      const int64_t paw = pa > 0 ? __ldg(out + pa - 1) : 0;
      const int64_t pbw = pb < n - 1 ? __ldg(out + pb + 1) : M - 1;
      if (paw == pbw) continue;
    }
    const int64_t aw = a > 0 ? __ldg(out + a - 1) : 0;
    const int64_t bw = b < n - 1 ? __ldg(out + b + 1) : M - 1;
    probes += bisect_probes(W, aw, bw, __ldg(u + m));
    depth = d > depth ? d : depth;
  }
  // warp reduce, one atomic per warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    probes += __shfl_xor_sync(FULL, probes, o);
    const unsigned long long od = __shfl_xor_sync(FULL, depth, o);
    depth = od > depth ? od : depth;
  }
  if ((threadIdx.x & 31) == 0) {
    if (probes) atomicAdd(counts + 1, probes);
    if (depth) atomicMax(counts + 2, depth);
  }
  if (kind == 1 && blockIdx.x == 0 && threadIdx.x == 0 && n > 0)
    atomicAdd(counts + 0, (unsigned long long)__ldg(out + n - 1) + (unsigned long long)n);
}

// the gather after a match (status untouched unless an index has no row)
int launch_gather_rows(const double* states, int64_t K, int64_t d, const int64_t* idx, int64_t N, int64_t divisor,
                       double* out, int32_t* status, cudaStream_t st) {
  if (N == 0) return DRS_OK;
  const bool vec2 = ((d & 1) == 0) && ((((uintptr_t)states) | ((uintptr_t)out)) & 15) == 0;
  const int64_t total = vec2 ? N * (d / 2) : N * d;
  const int64_t blocks = cdiv(total, 256) < 148 * 16 ? cdiv(total, 256) : 148 * 16;
  if (vec2)
    k_gather_rows<double2><<<(unsigned)blocks, 256, 0, st>>>((const double2*)states, K, d / 2, idx, N, divisor,
                                                             (double2*)out, status);
  else
    k_gather_rows<double><<<(unsigned)blocks, 256, 0, st>>>(states, K, d, idx, N, divisor, out, status);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

}  // namespace drs

using namespace drs;

extern "C" {

int dr_gather_rows(const double* states, int64_t K, int64_t d, const int64_t* idx, int64_t N, int64_t divisor,
                   double* out, int32_t* status, void* stream) {
  if (K < 1 || d < 1 || N < 0 || divisor < 1 || !status || (N > 0 && (!states || !idx || !out)))
    return DRS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(status, 0, sizeof(int32_t), st) != cudaSuccess) return DRS_ERR_LAUNCH;
  const int rc = launch_gather_rows(states, K, d, idx, N, divisor, out, status, st);
  return rc ? rc : launch_rc_x();
}

int dr_histogram(const int64_t* idx, int64_t N, int64_t M, uint64_t* counts, int32_t* status, void* stream) {
  if (N < 0 || M < 1 || !counts || !status || (N > 0 && !idx)) return DRS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(status, 0, sizeof(int32_t), st) != cudaSuccess) return DRS_ERR_LAUNCH;
  if (cudaMemsetAsync(counts, 0, sizeof(uint64_t) * (size_t)M, st) != cudaSuccess) return DRS_ERR_LAUNCH;
  if (N == 0) return DRS_OK;
  const int64_t blocks = cdiv(N, 256) < 148 * 8 ? cdiv(N, 256) : 148 * 8;
  k_histogram<<<(unsigned)blocks, 256, 0, st>>>(idx, N, M, (unsigned long long*)counts, status);
  return launch_rc_x();
}

size_t dr_chi_square_workspace(int64_t M) {
  (void)M;
  return sizeof(double) * 1024;
}

int dr_chi_square(const uint64_t* counts, const double* W, int64_t M, int64_t n, double* out, void* ws,
                  size_t ws_bytes, void* stream) {
  if (M < 1 || n < 0 || !counts || !W || !out || !ws || ws_bytes < dr_chi_square_workspace(M)) return DRS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = (int)(cdiv(M, 4096) < 1024 ? cdiv(M, 4096) : 1024);
  k_chi_partial<<<nb, CHI_THREADS, 0, st>>>((const unsigned long long*)counts, W, M, (double)n, (double*)ws);
  k_chi_final<<<1, 1, 0, st>>>((const double*)ws, nb, out);
  return launch_rc_x();
}

int dr_op_counts(int32_t kind, const double* W, int64_t M, const double* u, int64_t N, const int64_t* out,
                 uint64_t* counts, void* stream) {
  if (kind < 0 || kind > 2 || M < 1 || N < 0 || !W || !counts || (N > 0 && (!u || !out))) return DRS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(counts, 0, 3 * sizeof(uint64_t), st) != cudaSuccess) return DRS_ERR_LAUNCH;
  if (N == 0) return DRS_OK;
  const int64_t blocks = cdiv(N, 256) < 148 * 8 ? cdiv(N, 256) : 148 * 8;
  k_op_counts<<<(unsigned)blocks, 256, 0, st>>>(kind, W, M, u, N, out, (unsigned long long*)counts);
  return launch_rc_x();
}

}  // extern "C"
