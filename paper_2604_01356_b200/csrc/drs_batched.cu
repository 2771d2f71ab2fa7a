// drs_batched.cu -- many independent filters in one launch (config 4).
//
// The reference resamples a batch of filters with a Python loop of
// build_weight_table (cdf.py:59-89) + dac_sampler (samplers.py:262-266) per
// filter.  Here one CTA owns one filter end to end: its raw weights arrive by
// one TMA bulk copy, the table is scanned in shared memory with the same
// chained association as dr_build_table (so W is bit-identical to the
// single-filter path), the N_f+1 spacings are generated and scanned in
// registers/shared memory exactly like dr_sorted_uniforms, and the N_f
// lower bounds are found by bisection in shared memory.  Global traffic is
// the raw weights once plus U and the indices.  Filters shard across GPUs
// with no collective (the caller slices w/keys/out by filter).
#include "drs_common.cuh"

namespace drs {

constexpr int64_t TS_TABLE = (int64_t)THREADS * K_TABLE;
constexpr int64_t TS_UNIF = (int64_t)THREADS * K_UNIF;
constexpr int MAX_TABLE_TILES = 3;  // Mf <= 25344 (shared memory bound)

__device__ __forceinline__ double chain_fold_b(double tau, double* s_g, double& Q, double& R) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0.0;
  Q = 0.0;
#pragma unroll
  for (int k = 0; k < LANES; ++k) {
    if (lane == k) Q = acc;
    acc = __dadd_rn(acc, __shfl_sync(FULL, tau, k));
  }
  if (lane == 0) s_g[warp] = acc;
  __syncthreads();
  double r = 0.0;
  R = 0.0;
#pragma unroll
  for (int v = 0; v < WARPS; ++v) {
    if (v == warp) R = r;
    r = __dadd_rn(r, s_g[v]);
  }
  __syncthreads();  // s_g is reused by the next tile
  return r;
}

__device__ __forceinline__ int smem_lb(const double* a, int n, double x) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (a[m] < x) lo = m + 1;
    else hi = m;
  }
  return lo;
}

__global__ void __launch_bounds__(THREADS, 1)
    k_resample_batched(const double* __restrict__ w, int64_t Mf, int64_t Nf,
                       const uint64_t* __restrict__ keys, double* __restrict__ Wout,
                       double* __restrict__ Uout, int64_t* __restrict__ out, int32_t* status) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double s_g[WARPS];
  __shared__ unsigned long long s_min;
  __shared__ int s_bad;
  const int64_t f = blockIdx.x;
  const int ntt = (int)cdiv(Mf, TS_TABLE);
  const int64_t padM = (int64_t)ntt * TS_TABLE;
  double* sw = sm;
  double* su = sm + padM;  // Nf + 1 scanned spacings, then U
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* wf = w + f * Mf;

  // ---- stage the filter's raw weights (TMA bulk copy when 16-byte aligned)
  const bool aligned = (((uintptr_t)wf) & 15) == 0;
  const int64_t bulk = aligned ? (Mf & ~(int64_t)1) : 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, (uint32_t)(bulk * 8));
    if (bulk > 0) bulk_g2s(sw, wf, (uint32_t)(bulk * 8), &bar);
    s_min = 0x7FF0000000000000ULL;
    s_bad = 0;
  }
  for (int64_t i = bulk + threadIdx.x; i < padM; i += THREADS) sw[i] = (i < Mf) ? wf[i] : 0.0;
  __syncthreads();
  mbar_wait(&bar, 0);

  // ---- table: sweep 1 (tile totals and the chained tile prefixes)
  double Pt[MAX_TABLE_TILES];
  double P = 0.0;
  bool bad = false;
  for (int t = 0; t < ntt; ++t) {
    const double* chunk = sw + t * TS_TABLE + (warp * LANES + lane) * K_TABLE;
    double s = chunk[0];
    bad |= !(s >= 0.0 && s < dinf());
#pragma unroll
    for (int i = 1; i < K_TABLE; ++i) {
      const double x = chunk[i];
      bad |= !(x >= 0.0 && x < dinf());
      s = __dadd_rn(s, x);
    }
    double Q, R;
    const double A = chain_fold_b(s, s_g, Q, R);
    Pt[t] = P;
    P = __dadd_rn(P, A);
  }
  const double T = P;
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, DRS_ST_INVALID_WEIGHT);
  if (threadIdx.x == 0) {
    int st = 0;
    if (T == 0.0) st |= DRS_ST_DEGENERATE;
    if (!(T < dinf())) st |= DRS_ST_ACCUM_OVERFLOW;
    if (st) atomicOr(status, st);
  }
  // ---- table: sweep 2 (W in place)
  for (int t = 0; t < ntt; ++t) {
    double* chunk = sw + t * TS_TABLE + (warp * LANES + lane) * K_TABLE;
    double s = chunk[0];
#pragma unroll
    for (int i = 1; i < K_TABLE; ++i) s = __dadd_rn(s, chunk[i]);
    double Q, R;
    chain_fold_b(s, s_g, Q, R);
    const int64_t jb = t * TS_TABLE + (warp * LANES + lane) * K_TABLE;
    double s2 = 0.0;
#pragma unroll
    for (int i = 0; i < K_TABLE; ++i) {
      const double x = chunk[i];
      s2 = (i == 0) ? x : __dadd_rn(s2, x);
      const double S = __dadd_rn(Pt[t], __dadd_rn(R, __dadd_rn(Q, s2)));
      double v = fmin(__ddiv_rn(S, T), 1.0);
      if (jb + i == Mf - 1) v = 1.0;
      chunk[i] = v;
    }
  }

  // ---- sorted uniforms: Nf+1 spacings, chained scan over 1024-element tiles
  const uint64_t k0 = keys[3 * f], k1 = keys[3 * f + 1], off = keys[3 * f + 2];
  const int64_t ne = Nf + 1;
  const int ntu = (int)cdiv(ne, TS_UNIF);
  double Pu = 0.0;
  unsigned long long mn = 0x7FF0000000000000ULL;
  for (int t = 0; t < ntu; ++t) {
    const int64_t e0 = t * TS_UNIF + (int64_t)(warp * LANES + lane) * K_UNIF;
    const uint64_t d0 = off + (uint64_t)e0;
    const uint64_t b0 = d0 >> 2, b1 = (d0 + 3) >> 2;
    const U64x4 v0 = philox_block(k0, k1, b0);
    U64x4 v1 = v0;
    if (b1 != b0) v1 = philox_block(k0, k1, b1);
    double z[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint64_t dd = d0 + (uint64_t)i;
      const uint64_t raw = ((dd >> 2) == b0) ? pick(v0, (int)(dd & 3)) : pick(v1, (int)(dd & 3));
      z[i] = (e0 + i < ne) ? neglog(u01(raw)) : 0.0;
      if (e0 + i < ne) mn = min(mn, (z[i] > 0.0) ? (unsigned long long)__double_as_longlong(z[i]) : 0ull);
    }
    double sc[4];
    sc[0] = z[0];
#pragma unroll
    for (int i = 1; i < 4; ++i) sc[i] = __dadd_rn(sc[i - 1], z[i]);
    double Q, R;
    const double A = chain_fold_b(sc[3], s_g, Q, R);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (e0 + i < ne) su[e0 + i] = __dadd_rn(Pu, __dadd_rn(R, __dadd_rn(Q, sc[i])));
    Pu = __dadd_rn(Pu, A);
  }
  atomicMin(&s_min, mn);
  __syncthreads();
  const double total = Pu;
  for (int64_t i = threadIdx.x; i < Nf; i += THREADS) su[i] = __ddiv_rn(su[i], total);
  __syncthreads();
  const double zmin = __longlong_as_double((long long)s_min);
  if (!(zmin > __dmul_rn(1e-14, total)) && threadIdx.x == 0 && Nf > 0) {
    // exact check and repair (randkit.py:95-116), serial: rare and Nf is small
    bool b2 = (su[0] <= 0.0) || (su[Nf - 1] >= 1.0);
    for (int64_t i = 1; !b2 && i < Nf; ++i) b2 = !(__dsub_rn(su[i], su[i - 1]) > 0.0);
    if (b2) {
      double lo = 0.0;
      for (int64_t i = 0; i < Nf; ++i) {
        if (su[i] <= lo) su[i] = nextafter(lo, 1.0);
        lo = su[i];
      }
      double hi = 1.0;
      for (int64_t i = Nf - 1; i >= 0; --i) {
        if (su[i] >= hi) su[i] = nextafter(hi, 0.0);
        hi = su[i];
      }
      atomicOr(status, DRS_ST_REPAIRED);
    }
  }
  __syncthreads();

  // ---- match (bisection in shared memory) and write back
  for (int64_t i = threadIdx.x; i < Nf; i += THREADS) {
    const double x = su[i];
    out[f * Nf + i] = smem_lb(sw, (int)Mf, x);
    if (Uout) Uout[f * Nf + i] = x;
  }
  if (Wout)
    for (int64_t i = threadIdx.x; i < Mf; i += THREADS) Wout[f * Mf + i] = sw[i];
}

}  // namespace drs

using namespace drs;

extern "C" int dr_resample_batched(const double* w, int64_t B, int64_t Mf, int64_t Nf,
                                   const uint64_t* keys, double* W, double* U, int64_t* out,
                                   int32_t* status, void* stream) {
  if (B < 0 || Mf < 1 || Nf < 0 || !status) return DRS_ERR_ARG;
  if (B > 0 && (!w || !keys || (Nf > 0 && !out))) return DRS_ERR_ARG;
  if (cdiv(Mf, TS_TABLE) > MAX_TABLE_TILES) return DRS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(status, 0, sizeof(int32_t), st) != cudaSuccess) return DRS_ERR_LAUNCH;
  if (B == 0) return DRS_OK;
  const int64_t smem = (cdiv(Mf, TS_TABLE) * TS_TABLE + Nf + 1) * 8;
  if (smem > 227 * 1024 - 1024) return DRS_ERR_ARG;
  cudaFuncSetAttribute(k_resample_batched, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_resample_batched<<<(unsigned)B, THREADS, (size_t)smem, st>>>(w, Mf, Nf, keys, W, U, out, status);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}
