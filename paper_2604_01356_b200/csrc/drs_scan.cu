// drs_scan.cu -- the two fp64 scans of the resampling path on sm_100a.
//
//   K1 build_table     (cdf.py:59-89)      raw w -> W = S/T, W[M-1] == 1, + search index
//   K2 sorted_uniforms (randkit.py:70-101) Philox draws -> -log -> Z -> U = Z/Z[n], + repair
//
// Both are reduce-then-scan over tiles of THREADS*K elements, with the
// deterministic chained association of DESIGN.md section 4:
//   pass 1       : tile totals A_t (in-tile chained fold) -- fully parallel;
//   chain groups : one CTA folds the tile totals serially inside groups of
//                  GROUP_TILES tiles (D_t) and the group totals serially (C_g);
//                  no look-back, so no serial chain of inter-CTA round trips;
//   pass 2       : S = C_g + (D_t + (R + (Q + s))) and the epilogue.
// Every fold is a left fold from 0.0 and every group's last value is the next
// group's base, so S is monotone and S[last] == T exactly.
// The table pass reads w twice and writes W once (24 bytes per entry); the
// uniform pass generates each draw once, writes the in-tile sums in pass 1 and
// turns them into U in pass 2 (24 bytes per u).
#include <algorithm>
#include <cstdlib>

#include "drs_common.cuh"

namespace drs {

// ------------------------------------------------------ workspace layout ----
static constexpr size_t kHdr = 64;

__host__ inline size_t ws_fixed_bytes() { return kHdr + 8 * (size_t)SITE_CAP + 8 * (size_t)FLAG_CAP + 64; }

// The layout depends only on ws_bytes, so flag slots never alias value slots
// across calls with different tile counts.
__host__ inline int64_t ws_tile_capacity(size_t ws_bytes) {
  if (ws_bytes < ws_fixed_bytes()) return 0;
  return (int64_t)((ws_bytes - ws_fixed_bytes()) / 20);
}

__host__ inline ScanWS carve(void* ws, size_t ws_bytes) {
  const int64_t C = ws_tile_capacity(ws_bytes);
  unsigned char* b = (unsigned char*)ws;
  ScanWS s;
  s.hdr = (ScanHdr*)b;
  size_t o = kHdr;
  s.grp = (double*)(b + o);  // 4 bytes per tile hold the 8-byte group bases (GROUP_TILES >= 2)
  o += 4 * (size_t)C;
  o = (o + 15) & ~(size_t)15;
  s.agg = (double*)(b + o);
  o += 8 * (size_t)C;
  s.incl = (double*)(b + o);
  o += 8 * (size_t)C;
  s.sites = (long long*)(b + o);
  o += 8 * (size_t)SITE_CAP;
  s.tflag = (unsigned long long*)(b + o);
  return s;
}

__global__ void k_ws_init(ScanHdr* h) {
  h->done = 0;
  h->status = 0; h->nsites = 0; h->top = 0; h->bar_count = 0; h->bar_gen = 0;
  h->zmin_bits = 0x7FF0000000000000ULL;
  h->total = 0.0;
}

// The tile chain: one CTA folds the nt tile totals.  Thread g folds group g
// serially (D_t, exclusive) and leaves the group total; thread 0 then folds
// the group totals serially (C_g, exclusive) and writes T = C_ng.  It also
// finishes what needs every tile: for a table (mode 0) the status word (and
// T for a shard scan); for sorted uniforms (mode 1) the minimum spacing
// (pass 1 left each tile's minimum in incl[t]) and the reference's
// exactness trigger zmin <= 1e-14 T (randkit.py:95).
constexpr int CHAIN_THREADS = 512;
constexpr int64_t CHAIN_CHUNK = 16384;    // tiles staged in shared memory per round (a multiple of GROUP_TILES)
constexpr int CHAIN_MAX_GROUPS = 8192;    // nt <= 2^18 tiles
constexpr size_t CHAIN_SMEM = (size_t)(CHAIN_CHUNK + CHAIN_CHUNK / 32) * 8 + (size_t)CHAIN_MAX_GROUPS * 8;

__global__ void __launch_bounds__(CHAIN_THREADS) k_chain_groups(ScanWS ws, int64_t nt, int mode,
                                                               int32_t* status_out, double* total_out,
                                                               int64_t chunk) {
  extern __shared__ __align__(16) double csm[];
  STAMPK(1, 0);
  pdl_wait();
  STAMPK(1, 1);
  STAMP1(0);
  pdl_trigger();  // one CTA: the next grid may take the other SMs now
  // [chunk + chunk / 32] tile totals -> exclusive in-group folds, one pad slot
  // per group of 32 so that the per-group folds (thread g reads group g) hit
  // different banks; then [ng] group totals -> group bases
  double* sa = csm;
  double* sE = csm + chunk + chunk / GROUP_TILES;
  __shared__ unsigned long long s_min;
  if (threadIdx.x == 0) s_min = 0x7FF0000000000000ULL;
  const int64_t ng = cdiv(nt, GROUP_TILES);
  unsigned long long mn = 0x7FF0000000000000ULL;
  for (int64_t c0 = 0; c0 < nt; c0 += chunk) {
    const int64_t c1 = (c0 + chunk < nt) ? c0 + chunk : nt;
    // 1. stage the chunk's tile totals (coalesced; eight loads per thread in
    // flight before the first store, so the staging costs one round trip per
    // eight rather than one per tile)
    for (int64_t tb = c0 + threadIdx.x; tb < c1; tb += 8 * CHAIN_THREADS) {
      double v[8], m[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t t = tb + (int64_t)k * CHAIN_THREADS;
        v[k] = (t < c1) ? __ldcg(ws.agg + t) : 0.0;
        m[k] = (mode == 1 && t < c1) ? __ldcg(ws.incl + t) : __longlong_as_double(0x7FF0000000000000LL);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t t = tb + (int64_t)k * CHAIN_THREADS;
        if (t < c1) sa[(t - c0) + ((t - c0) >> 5)] = v[k];
        mn = min(mn, (unsigned long long)__double_as_longlong(m[k]));
      }
    }
    __syncthreads();
    STAMP(1);
    // 2. one thread per group: serial left fold from shared memory
    const int64_t g0 = c0 / GROUP_TILES, g1 = cdiv(c1, GROUP_TILES);
    static_assert(CHAIN_CHUNK % GROUP_TILES == 0, "chunks hold whole groups");
    for (int64_t g = g0 + threadIdx.x; g < g1; g += CHAIN_THREADS) {
      const int64_t gl = g - g0;  // group within the chunk: its 32 tiles start at 33 gl
      const int len = (int)(((g + 1) * GROUP_TILES < c1 ? (g + 1) * GROUP_TILES : c1) - g * GROUP_TILES);
      double* ga = sa + gl * (GROUP_TILES + 1);
      double D = 0.0;
      int t = 0;
      for (; t + 8 <= len; t += 8) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = ga[t + k];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          ga[t + k] = D;
          D = __dadd_rn(D, v[k]);
        }
      }
      for (; t < len; ++t) {
        const double v = ga[t];
        ga[t] = D;
        D = __dadd_rn(D, v);
      }
      sE[g] = D;
    }
    __syncthreads();
    STAMP(2);
    // 3. write the exclusive in-group folds back (coalesced)
    for (int64_t t = c0 + threadIdx.x; t < c1; t += CHAIN_THREADS) ws.incl[t] = sa[(t - c0) + ((t - c0) >> 5)];
    __syncthreads();
  }
  STAMP(3);
  if (mode == 1) block_min_u64(&s_min, mn);
  __syncthreads();
  if (threadIdx.x == 0) {
    // serial left fold of the group totals; eight loads ahead of the adds,
    // so the chain costs one fp64 add latency per group, not a shared load
    double C = 0.0;
    int64_t g = 0;
    for (; g + 8 <= ng; g += 8) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = sE[g + k];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        sE[g + k] = C;
        C = __dadd_rn(C, v[k]);
      }
    }
    for (; g < ng; ++g) {
      const double e = sE[g];
      sE[g] = C;
      C = __dadd_rn(C, e);
    }
    const double T = C;
    ws.hdr->total = T;
    if (mode == 0) {
      uint32_t st = ws.hdr->status;
      if (T == 0.0) st |= DRS_ST_DEGENERATE;
      if (!(T < dinf())) st |= DRS_ST_ACCUM_OVERFLOW;
      if (status_out) *status_out = (int32_t)st;
      if (total_out) *total_out = T;
      ws.hdr->status = 0;
    } else {
      const double zmin = __longlong_as_double((long long)s_min);
      ws.hdr->need = !(zmin > __dmul_rn(1e-14, T)) ? 1u : 0u;
    }
  }
  __syncthreads();
  STAMP1(4);
  for (int64_t g = threadIdx.x; g < ng; g += CHAIN_THREADS) ws.grp[g] = sE[g];
  STAMP(5);
  STAMPK(1, 3);
}

#ifdef DRS_PHASE_TIMING
extern "C" int dr_debug_phase_times_scan(unsigned long long* host, int n) {
  return cudaMemcpyFromSymbol(host, g_phase, sizeof(unsigned long long) * (size_t)n) == cudaSuccess ? 0 : -1;
}
extern "C" int dr_debug_phase_clear_scan(void) {
  void* p = nullptr;
  if (cudaGetSymbolAddress(&p, g_phase) != cudaSuccess) return -1;
  return cudaMemset(p, 0, sizeof(g_phase)) == cudaSuccess ? 0 : -1;
}
#endif

void launch_chain(const ScanWS& s, int64_t nt, int mode, int32_t* status, double* total,
                  cudaStream_t st) {
  static SmemLimit lim;
  lim.raise((const void*)k_chain_groups, CHAIN_SMEM);
  // shared memory sized to the call (whole groups of tiles, then the group
  // totals): small chains launch without reconfiguring a 192 KB carve-out
  const int64_t chunk = std::min<int64_t>(CHAIN_CHUNK, cdiv(nt, GROUP_TILES) * GROUP_TILES);
  const size_t smem = (size_t)(chunk + chunk / GROUP_TILES + cdiv(nt, GROUP_TILES)) * 8;
  launch_pdl(k_chain_groups, dim3(1), dim3(CHAIN_THREADS), smem, st, s, nt, mode, status, total, chunk);
}

// exclusive chained prefix of tile t applied to an in-tile value y
__device__ __forceinline__ double chain_apply(const ScanWS& ws, int64_t t, double y) {
  return __dadd_rn(ws.grp[t / GROUP_TILES], __dadd_rn(ws.incl[t], y));
}

// ------------------------------------------------------------ K1 table ----
// Stage tile t of src (zero padded) into shared memory with one TMA bulk copy.
template <int K>
__device__ __forceinline__ int64_t stage_tile(const double* __restrict__ src, int64_t n, int64_t t,
                                              double* sm, uint64_t* bar) {
  constexpr int64_t TS = (int64_t)THREADS * K;
  const int64_t j0 = t * TS;
  const int64_t len = (n - j0 < TS) ? (n - j0) : TS;
  const int64_t len_even = len & ~(int64_t)1;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_expect_tx(bar, (uint32_t)(len_even * 8));
    if (len_even > 0) bulk_g2s(sm, src + j0, (uint32_t)(len_even * 8), bar);
  }
  for (int64_t i = len_even + threadIdx.x; i < TS; i += THREADS) sm[i] = (i < len) ? src[j0 + i] : 0.0;
  __syncthreads();
  mbar_wait(bar, 0);
  return len;
}

// ------------------------------------------------- log-weight tables ----
// max over the log-weights (order-independent, exact) with NaN propagation:
// per-CTA maxima in agg[], the last CTA folds them into hdr->wmax.
__device__ __forceinline__ unsigned long long ord_key(double x) {  // total order on non-NaN doubles
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k));
}

__global__ void __launch_bounds__(256) k_max_logw(const double* __restrict__ lw, int64_t n, ScanWS ws) {
  __shared__ unsigned long long s_key;
  __shared__ int s_nan;
  __shared__ bool s_last;
  pdl_wait();
  if (threadIdx.x == 0) { s_key = 0; s_nan = 0; }
  __syncthreads();
  unsigned long long key = 0;
  bool nan = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double x = __ldg(lw + i);
    if (x != x) nan = true;
    else key = max(key, ord_key(x));
  }
  atomicMax(&s_key, key);
  if (nan) s_nan = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    ws.agg[blockIdx.x] = __longlong_as_double((long long)(s_nan ? ~0ULL : s_key));
    __threadfence();
    s_last = atomicAdd(&ws.hdr->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    unsigned long long k = 0;
    bool anynan = false;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      const unsigned long long v = (unsigned long long)__double_as_longlong(ld_relaxed_f64(&ws.agg[b]));
      if (v == ~0ULL) anynan = true;
      else k = max(k, v);
    }
    ws.hdr->wmax = anynan ? __longlong_as_double(0x7FF8000000000000LL) : ord_val(k);
    ws.hdr->done = 0;
  }
}

// the staged tile of log-weights -> w = exp(lw - max) in place (padding stays 0)
__device__ __forceinline__ void exp_shift_tile(double* sm, int64_t len, double mx) {
  const int c0 = threadIdx.x * K_TABLE;
#pragma unroll 3
  for (int i = 0; i < K_TABLE; ++i)
    if (c0 + i < len) sm[c0 + i] = dexp(__dsub_rn(sm[c0 + i], mx));
  __syncwarp();
}

// LOGW: the staged log-weights become w = exp(lw - max) in place and the
// tile of w is stored to wout (the table buffer), which pass 2 then scans:
// each exp is evaluated once
template <bool LOGW>
__global__ void __launch_bounds__(THREADS) k_table_pass1(const double* __restrict__ w, int64_t n,
                                                         ScanWS ws, double* __restrict__ wout) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ FoldSmem fs;
  const int64_t t = blockIdx.x;
  pdl_wait();
  const int64_t len = stage_tile<K_TABLE>(w, n, t, sm, &bar);
  if (LOGW) {
    exp_shift_tile(sm, len, ws.hdr->wmax);  // each thread transforms its own chunk
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t j0 = t * (int64_t)THREADS * K_TABLE;
      const int64_t le = len & ~(int64_t)1;
      if (le > 0) bulk_s2g(wout + j0, sm, (uint32_t)(le * 8));
      if (len & 1) wout[j0 + len - 1] = sm[len - 1];
    }
  }
  const int c0 = threadIdx.x * K_TABLE;
  const double* chunk = sm + c0;
  // valid weight <=> 0 <= x < inf: screened from the high words (integer
  // pipe); a set sign bit gets the exact check (-0.0 is a valid weight)
  uint32_t any_sign = 0, max_mag = 0;
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < K_TABLE; ++i) {
    const double x = chunk[i];
    const uint32_t hi = (uint32_t)__double2hiint(x);
    any_sign |= hi;
    max_mag = max(max_mag, hi & 0x7FFFFFFFu);
    s = (i == 0) ? x : __dadd_rn(s, x);
  }
  bool bad = max_mag >= 0x7FF00000u;
  if (any_sign & 0x80000000u)
    for (int i = 0; i < K_TABLE; ++i) bad |= !(chunk[i] >= 0.0);
  double Q, R;
  const double A = block_fold(s, fs, Q, R);
  pdl_trigger();
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&ws.hdr->status, (uint32_t)DRS_ST_INVALID_WEIGHT);
  if (threadIdx.x == 0) ws.agg[t] = A;
  if (LOGW && threadIdx.x == 0) bulk_commit_wait();  // smem stays valid until the store has read it
}

// RAW = false: W = min(S/T, 1) with W[n-1] = 1 and the index levels (dr_build_table)
// RAW = true:  the unnormalised local prefix S and *total_out = T (dr_shard_scan)
template <bool RAW, bool LOGW>
__global__ void __launch_bounds__(THREADS) k_table_pass2(const double* __restrict__ w, int64_t n,
                                                         int64_t nt, ScanWS ws,
                                                         double* __restrict__ W,
                                                         double* __restrict__ idx, IndexDesc d,
                                                         int32_t* status_out, double* total_out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ FoldSmem fs;
  constexpr int64_t TS = (int64_t)THREADS * K_TABLE;
  const int64_t t = blockIdx.x;
  const int64_t len = stage_tile<K_TABLE>(w, n, t, sm, &bar);
  if (LOGW) exp_shift_tile(sm, len, ws.hdr->wmax);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* chunk = sm + (warp * LANES + lane) * K_TABLE;
  double s = chunk[0];
#pragma unroll
  for (int i = 1; i < K_TABLE; ++i) s = __dadd_rn(s, chunk[i]);
  double Q, R;
  block_fold(s, fs, Q, R);
  // everything above reads only the weights (produced before the previous
  // launch): under programmatic launch it overlaps the chain kernel
  pdl_wait();
  pdl_trigger();
  const double C = ws.grp[t / GROUP_TILES], D = ws.incl[t];
  const double T = ws.hdr->total;
  const int64_t jb = t * TS + (int64_t)(warp * LANES + lane) * K_TABLE;
  double s2 = 0.0;
#pragma unroll
  for (int i = 0; i < K_TABLE; ++i) {
    const double x = chunk[i];
    s2 = (i == 0) ? x : __dadd_rn(s2, x);
    const double S = __dadd_rn(C, __dadd_rn(D, __dadd_rn(R, __dadd_rn(Q, s2))));
    const int64_t j = jb + i;
    if (RAW) {
      chunk[i] = S;
      continue;
    }
    double v = fmin(__ddiv_rn(S, T), 1.0);
    if (j == n - 1) v = 1.0;
    chunk[i] = v;
  }
  fence_proxy_async_smem();
  __syncthreads();
  const int64_t len_even = len & ~(int64_t)1;
  const int64_t j0 = t * TS;
  if (threadIdx.x == 0) {
    if (len_even > 0) bulk_s2g(W + j0, sm, (uint32_t)(len_even * 8));
    if (len & 1) W[j0 + len - 1] = sm[len - 1];
  }
  if (!RAW) {
    // index entries ending in this tile, written cooperatively: level k holds
    // W at every 16^k-block end (the last block ends at n-1), padded with +inf
    static_assert(FANOUT == 16, "index levels use shifts by 4 bits per level");
    const int64_t jl = j0 + len - 1;
    for (int k = 1, sh = 4; k <= d.levels; ++k, sh += 4) {
      const int64_t m0 = (j0 + 1 + ((int64_t)1 << sh) - 1) >> sh;  // (m0 + 1) << sh > j0: m0 - 1 ends at/after j0
      const int64_t m1 = (jl + 1) >> sh;                             // blocks ending at or before jl
      for (int64_t m = m0 - 1 + threadIdx.x; m < m1; m += THREADS)
        if (m >= 0) idx[d.off[k] + m] = sm[((m + 1) << sh) - 1 - j0];
      if (jl == n - 1) {  // the last, possibly partial, block and the padding
        const int64_t mlast = (n - 1) >> sh;
        const int64_t padded = cdiv(d.n[k], FANOUT) * FANOUT;
        for (int64_t p = mlast + threadIdx.x; p < padded; p += THREADS)
          idx[d.off[k] + p] = (p == mlast) ? sm[len - 1] : dinf();
      }
    }
  }
  if (threadIdx.x == 0 && len_even > 0) bulk_commit_wait();
  (void)status_out;
  (void)total_out;
}

// ------------------------------------------- K1 in one pass (deferred) ----
// dr_build_table_deferred: ONE pass over w.  Each tile's in-tile chained sums
// L = R + (Q + s) -- k_table_pass2's association without the tile prefix
// C_g + D_t, which needs every tile before it -- are stored as the table's
// values, the tile's level-1 index entries likewise, the tile total to
// agg[t]; validation as in pass 1.  k_chain_groups then folds the tile
// totals, and k_table_levels stores each tile's pair {C_g, D_t} and T in the
// index header, turns level 1 into W and writes the levels above it.  Reads
// w once and writes the table once: 16 bytes per entry instead of 24.
template <bool LOGW>
__global__ void __launch_bounds__(THREADS) k_table_local(const double* __restrict__ w, int64_t n, ScanWS ws,
                                                         double* __restrict__ L, double* __restrict__ lvl1,
                                                         double* __restrict__ lvl2) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ FoldSmem fs;
  constexpr int64_t TS = (int64_t)THREADS * K_TABLE;
  const int64_t t = blockIdx.x;
  STAMPK(4, 0);
  pdl_wait();
  STAMPK(4, 1);
  const int64_t len = stage_tile<K_TABLE>(w, n, t, sm, &bar);
  STAMPK(4, 2);
  if (LOGW) exp_shift_tile(sm, len, ws.hdr->wmax);
  double* chunk = sm + threadIdx.x * K_TABLE;
  uint32_t any_sign = 0, max_mag = 0;
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < K_TABLE; ++i) {
    const double x = chunk[i];
    const uint32_t hi = (uint32_t)__double2hiint(x);
    any_sign |= hi;
    max_mag = max(max_mag, hi & 0x7FFFFFFFu);
    s = (i == 0) ? x : __dadd_rn(s, x);
  }
  bool bad = max_mag >= 0x7FF00000u;
  if (any_sign & 0x80000000u)
    for (int i = 0; i < K_TABLE; ++i) bad |= !(chunk[i] >= 0.0);
  double Q, R;
  const double A = block_fold(s, fs, Q, R);
  pdl_trigger();
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&ws.hdr->status, (uint32_t)DRS_ST_INVALID_WEIGHT);
  if (threadIdx.x == 0) ws.agg[t] = A;
  double s2 = 0.0;
#pragma unroll
  for (int i = 0; i < K_TABLE; ++i) {
    const double x = chunk[i];
    s2 = (i == 0) ? x : __dadd_rn(s2, x);
    chunk[i] = __dadd_rn(R, __dadd_rn(Q, s2));
  }
  fence_proxy_async_smem();
  __syncthreads();
  const int64_t len_even = len & ~(int64_t)1;
  const int64_t j0 = t * TS;
  if (threadIdx.x == 0) {
    if (len_even > 0) bulk_s2g(L + j0, sm, (uint32_t)(len_even * 8));
    if (len & 1) L[j0 + len - 1] = sm[len - 1];
  }
  if (lvl1) {  // level 1: the value at every 16-entry block end (the last block ends at n-1)
    static_assert(TS % FANOUT == 0, "level-1 blocks never straddle table tiles");
    const int64_t jl = j0 + len - 1;
    for (int64_t m = j0 / FANOUT + threadIdx.x; m < (jl + 1) / FANOUT; m += THREADS)
      lvl1[m] = sm[(m + 1) * FANOUT - 1 - j0];
    if (jl == n - 1 && (n % FANOUT) && threadIdx.x == 0) lvl1[(n - 1) / FANOUT] = sm[len - 1];
  }
  if (lvl2) {
    // the sources of level 2 (the in-tile value at every 256-entry block end,
    // 33 per tile), left in level 2's own slots: the kernel after the chain
    // turns them into W in place with coalesced accesses instead of gathering
    // one sector per 128-byte line of level 1
    constexpr int64_t B2 = (int64_t)FANOUT * FANOUT;
    static_assert(TS % B2 == 0, "level-2 blocks never straddle table tiles");
    const int64_t jl = j0 + len - 1;
    for (int64_t m = j0 / B2 + threadIdx.x; m < (jl + 1) / B2; m += THREADS) lvl2[m] = sm[(m + 1) * B2 - 1 - j0];
    if (jl == n - 1 && (n % B2) && threadIdx.x == 0) lvl2[(n - 1) / B2] = sm[len - 1];
  }
  if (threadIdx.x == 0 && len_even > 0) bulk_commit_wait();
  STAMPK(4, 3);
}

// after the chain: level 1 (in-tile values) -> W = min(S / T, 1), the last
// entry pinned to 1, exactly what k_table_pass2 / k_shard_finalize store; an
// entry that ends a block of a higher level is stored there too; +inf padding
// of every level to whole nodes.  FROM_WS (dr_build_table_deferred): the tile
// pairs come from the chain's workspace and are stored with the header
// {T, 1, 0, 1}; otherwise (a shard: dr_shard_finalize_deferred) the header and
// pairs are already in idx.  A persistent grid, two level-1 entries per
// thread per step (16-byte accesses), the division by T as a multiply and two
// FMAs (div_rn, bit-identical).
template <bool FROM_WS>
__global__ void __launch_bounds__(256) k_table_levels(int64_t M, int64_t nt, ScanWS ws, double* __restrict__ idx,
                                                      IndexDesc d) {
  STAMPK(5, 0);
  pdl_wait();
  STAMPK(5, 1);
  pdl_trigger();
  double* aux = idx + d.aoff;
  const double2* P = reinterpret_cast<const double2*>(aux + TAB_HDR);
  const int64_t e0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double T, O = 0.0;
  bool shard = false, pin = true;
  const bool l1 = d.kt >= 2;  // level 1 keeps its in-tile values (TAB_L1)
  if (FROM_WS) {
    T = ws.hdr->total;
    for (int64_t e = e0; e < nt; e += stride)
      reinterpret_cast<double2*>(aux + TAB_HDR)[e] = make_double2(ws.grp[e / GROUP_TILES], ws.incl[e]);
    if (e0 == 0) {
      aux[0] = T;
      aux[1] = (double)(TAB_DEFERRED | (l1 ? TAB_L1 : 0));
      aux[2] = 0.0;
      aux[3] = 1.0;
    }
  } else {
    const TabAux ta = load_aux(aux);
    T = ta.T;
    O = ta.O;
    shard = ta.shard;
    pin = ta.pin;
  }
  if (d.levels == 0) return;
  if (e0 < (int64_t)FANOUT * d.levels) {
    const int k = 1 + (int)(e0 / FANOUT);
    const int64_t p = d.n[k] + e0 % FANOUT;
    if (p < cdiv(d.n[k], FANOUT) * FANOUT) idx[d.off[k] + p] = dinf();
  }
  const DivBy byT = div_by(T);
  // level-1 entry m ends W block m (position 16 m + 15, the last one M - 1),
  // which lies in table tile m / 528 (TABLE_TILE = 528 blocks); a pair
  // (m, m + 1), m even, never straddles two tiles (528 is even)
  static_assert(TABLE_TILE % (2 * FANOUT) == 0, "pairs of level-1 entries share a table tile");
  constexpr uint32_t BLOCKS_PER_TILE = (uint32_t)(TABLE_TILE / FANOUT);
  const int64_t n1 = d.n[1];  // level 1 starts at offset 0 (16-byte aligned); n1 < 2^32
  if (l1) {
    // level 1 stays in-tile: only the entries of level 2 and above, each the
    // W of its level-1 source entry m = 16 m2 + 15 (the last: n1 - 1)
    for (int64_t m2 = e0; m2 < d.n[2]; m2 += stride) {
      const int64_t m = (m2 * FANOUT + FANOUT - 1 < n1 - 1) ? m2 * FANOUT + FANOUT - 1 : n1 - 1;
      const uint32_t tt = (uint32_t)m / BLOCKS_PER_TILE;
      const double2 cd = FROM_WS ? make_double2(ws.grp[tt / GROUP_TILES], ws.incl[tt]) : __ldg(P + tt);
      // the source value: left in level 2's slot by k_table_local (FROM_WS), else level-1 entry m
      const double sl = __dadd_rn(cd.x, __dadd_rn(cd.y, FROM_WS ? idx[d.off[2] + m2] : idx[m]));
      const double S = shard ? __dadd_rn(O, sl) : sl;
      const bool lastm = m == n1 - 1;
      const double v = (lastm && pin) ? 1.0 : fmin(div_rn(S, byT), 1.0);
      idx[d.off[2] + m2] = v;
      for (int k = 3, sh = 8; k <= d.levels; ++k, sh += 4) {
        if (!lastm && ((m + 1) & (((int64_t)1 << sh) - 1)) != 0) break;
        idx[d.off[k] + (m >> sh)] = v;
      }
    }
    return;
  }
  for (int64_t e = 2 * e0; e < n1; e += 2 * stride) {
    const bool two = e + 1 < n1;
    double2 l;
    if (two) l = *reinterpret_cast<const double2*>(idx + e);
    else l = make_double2(idx[e], 0.0);
    const uint32_t tt = (uint32_t)e / BLOCKS_PER_TILE;
    const double2 cd = FROM_WS ? make_double2(ws.grp[tt / GROUP_TILES], ws.incl[tt]) : __ldg(P + tt);
    double v[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double sl = __dadd_rn(cd.x, __dadd_rn(cd.y, h ? l.y : l.x));
      const double S = shard ? __dadd_rn(O, sl) : sl;
      const bool last = e + h == n1 - 1;  // block n1 - 1 ends at M - 1
      v[h] = (last && pin) ? 1.0 : fmin(div_rn(S, byT), 1.0);
    }
    if (two) *reinterpret_cast<double2*>(idx + e) = make_double2(v[0], v[1]);
    else idx[e] = v[0];
    // the higher levels: entry m ends a level-k block when (m + 1) is a
    // multiple of 16^(k-1) (only an odd m can), or m is the last entry
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t m = e + h;
      if (h == 1 && !two) break;
      const bool lastm = m == n1 - 1;
      if (!lastm && ((m + 1) & (FANOUT - 1)) != 0) continue;
      for (int k = 2, sh = 4; k <= d.levels; ++k, sh += 4) {
        if (!lastm && ((m + 1) & (((int64_t)1 << sh) - 1)) != 0) break;
        idx[d.off[k] + (m >> sh)] = v[h];
      }
    }
  }
}

// The chain and the levels in ONE launch (dr_build_table_deferred, tables
// whose level 1 stays in-tile and whose tile totals fit in shared memory:
// 2^18 < M <= TAIL_MAX_TILES * 8448).  One 1024-thread CTA per SM; every CTA
// folds the whole tile chain itself out of shared memory -- the nt totals are
// L2-resident (k_table_local has just written them), thread g folds group g,
// thread 0 the group totals: k_chain_groups' fold, bit for bit -- instead of
// waiting for a one-CTA kernel to do it and write it back: the chain launch,
// its drain and its round trip through the workspace leave the critical path.
// Each thread loads the sources of its level-2 entries (the in-tile values
// k_table_local left in level 2's slots) behind the totals, then forms W in
// place and stores the levels above;
// the CTA's slice of the tile pairs goes to the header from shared memory.
// CTA 0 finishes what k_chain_groups (mode 0) finishes: T, the status word.
constexpr int TAIL_THREADS = 1024;
constexpr int64_t TAIL_MAX_TILES = 16384;  // (nt + nt / 32 + ng) * 8 bytes of shared memory: <= 140 KB
constexpr int TAIL_PRE = 4;                // level-2 entries per thread loaded ahead of the fold

__global__ void __launch_bounds__(TAIL_THREADS) k_table_tail(int64_t M, int64_t nt, ScanWS ws, double* __restrict__ idx,
                                                             IndexDesc d, int32_t* status_out) {
  extern __shared__ __align__(16) double tsm[];
  STAMPK(5, 0);
  pdl_wait();
  STAMPK(5, 1);
  pdl_trigger();
  const int64_t ng = cdiv(nt, GROUP_TILES);
  double* sa = tsm;                          // [nt + nt / 32 (+1)] tile totals -> D_t, one pad slot per group
  double* sE = tsm + nt + nt / GROUP_TILES + 1;  // [ng] group totals -> C_g
  const int64_t e0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n1 = d.n[1], n2 = d.n[2];
  // 1. stage the tile totals (eight loads per thread in flight), and behind
  // them the sources of this thread's first level-2 entries
  double pre[TAIL_PRE];
  for (int64_t tb = threadIdx.x; tb < nt || tb == threadIdx.x; tb += 8 * TAIL_THREADS) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int64_t t = tb + (int64_t)k * TAIL_THREADS;
      v[k] = (t < nt) ? __ldcg(ws.agg + t) : 0.0;
    }
    if (tb == threadIdx.x) {
#pragma unroll
      for (int k = 0; k < TAIL_PRE; ++k) {
        // an always-valid address (no select on the loaded value, which would wait for it here)
        const int64_t m2 = (e0 + k * stride < n2) ? e0 + k * stride : n2 - 1;
        pre[k] = __ldcg(idx + d.off[2] + m2);
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int64_t t = tb + (int64_t)k * TAIL_THREADS;
      if (t < nt) sa[t + (t >> 5)] = v[k];
    }
  }
  __syncthreads();
  STAMPK(7, 0);
  // 2. thread g folds group g (exclusive, left to right from 0.0)
  static_assert(TAIL_MAX_TILES / GROUP_TILES <= TAIL_THREADS, "one thread per group");
  if (threadIdx.x < ng) {
    const int64_t g = threadIdx.x;
    const int len = (int)(((g + 1) * GROUP_TILES < nt ? (g + 1) * GROUP_TILES : nt) - g * GROUP_TILES);
    double* ga = sa + g * (GROUP_TILES + 1);
    double D = 0.0;
    int t = 0;
    for (; t + 8 <= len; t += 8) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = ga[t + k];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        ga[t + k] = D;
        D = __dadd_rn(D, v[k]);
      }
    }
    for (; t < len; ++t) {
      const double v = ga[t];
      ga[t] = D;
      D = __dadd_rn(D, v);
    }
    sE[g] = D;
  }
  __syncthreads();
  STAMPK(7, 1);
  // 3. thread 0 folds the group totals (eight loads ahead of the adds)
  __shared__ double s_T;
  if (threadIdx.x == 0) {
    double C = 0.0;
    int64_t g = 0;
    for (; g + 8 <= ng; g += 8) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = sE[g + k];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        sE[g + k] = C;
        C = __dadd_rn(C, v[k]);
      }
    }
    for (; g < ng; ++g) {
      const double e = sE[g];
      sE[g] = C;
      C = __dadd_rn(C, e);
    }
    s_T = C;
    if (blockIdx.x == 0) {
      ws.hdr->total = C;
      uint32_t st = ws.hdr->status;
      if (C == 0.0) st |= DRS_ST_DEGENERATE;
      if (!(C < dinf())) st |= DRS_ST_ACCUM_OVERFLOW;
      if (status_out) *status_out = (int32_t)st;
      ws.hdr->status = 0;
    }
  }
  __syncthreads();
  STAMPK(5, 2);
  const double T = s_T;
  // 4. the header, the tile pairs, the +inf padding of every level
  double* aux = idx + d.aoff;
  for (int64_t e = e0; e < nt; e += stride)
    reinterpret_cast<double2*>(aux + TAB_HDR)[e] = make_double2(sE[e / GROUP_TILES], sa[e + (e >> 5)]);
  if (e0 == 0) {
    aux[0] = T;
    aux[1] = (double)(TAB_DEFERRED | TAB_L1);
    aux[2] = 0.0;
    aux[3] = 1.0;
  }
  if (e0 < (int64_t)FANOUT * d.levels) {
    const int k = 1 + (int)(e0 / FANOUT);
    const int64_t p = d.n[k] + e0 % FANOUT;
    if (p < cdiv(d.n[k], FANOUT) * FANOUT) idx[d.off[k] + p] = dinf();
  }
  STAMPK(7, 2);
  // 5. level 2 and above: the W of level-1 entry m = 16 m2 + 15 (the last: n1 - 1)
  const DivBy byT = div_by(T);
  constexpr uint32_t BLOCKS_PER_TILE = (uint32_t)(TABLE_TILE / FANOUT);
  int k = 0;
  for (int64_t m2 = e0; m2 < n2; m2 += stride, ++k) {
    const int64_t m = (m2 * FANOUT + FANOUT - 1 < n1 - 1) ? m2 * FANOUT + FANOUT - 1 : n1 - 1;
    double l;
    switch (k) {  // the first TAIL_PRE are in registers
      case 0: l = pre[0]; break;
      case 1: l = pre[1]; break;
      case 2: l = pre[2]; break;
      case 3: l = pre[3]; break;
      default: l = __ldcg(idx + d.off[2] + m2); break;
    }
    static_assert(TAIL_PRE == 4, "the switch above names the preloaded entries");
    const uint32_t tt = (uint32_t)m / BLOCKS_PER_TILE;
    const double S = __dadd_rn(sE[tt / GROUP_TILES], __dadd_rn(sa[tt + (tt >> 5)], l));
    const bool lastm = m == n1 - 1;
    const double v = lastm ? 1.0 : fmin(div_rn(S, byT), 1.0);
    idx[d.off[2] + m2] = v;
    for (int kk = 3, sh = 8; kk <= d.levels; ++kk, sh += 4) {
      if (!lastm && ((m + 1) & (((int64_t)1 << sh) - 1)) != 0) break;
      idx[d.off[kk] + (m >> sh)] = v;
    }
  }
  STAMPK(5, 3);
}

// a shard's scan (dr_shard_scan_deferred): the tile pairs from the chain's
// workspace into idx (the header follows once the shard totals are known)
__global__ void k_table_pairs(int64_t nt, ScanWS ws, double* __restrict__ aux) {
  pdl_wait();
  pdl_trigger();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nt; e += stride)
    reinterpret_cast<double2*>(aux + TAB_HDR)[e] = make_double2(ws.grp[e / GROUP_TILES], ws.incl[e]);
}

// a table's cumulative weights: W itself (direct) or formed (deferred)
__global__ void __launch_bounds__(256) k_table_materialize(const double* __restrict__ V, int64_t M,
                                                           const double* __restrict__ aux, double* __restrict__ W) {
  const TabAux ta = load_aux(aux);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += stride) {
    const double v = V[j];
    W[j] = ta.def ? tab_w(ta, __ldg(ta.P + j / TABLE_TILE), v, j == M - 1) : v;
  }
}

// ------------------------------------------------- K2 sorted uniforms ----
__device__ __forceinline__ unsigned long long zmin_key(double z) {
  // positive doubles order like their bit patterns; NaN / <= 0 force the exact check
  if (!(z > 0.0)) return 0ull;
  return (unsigned long long)__double_as_longlong(z);
}

// pass 1: every spacing generated ONCE; the in-tile chained sums
// R + (Q + sc) written to U (the tile prefix is applied in pass 2); the tile
// total to agg[t]; the spacing minimum to the header.
template <class Src>
__global__ void __launch_bounds__(THREADS) k_unif_pass1(Src src, int64_t n, ScanWS ws, double* __restrict__ Z) {
  __shared__ FoldSmem fs;
  __shared__ unsigned long long s_min;
  __shared__ uint64_t s_words[Src::SMEM_WORDS];
  STAMPK(0, 0);
  pdl_wait();
  STAMPK(0, 1);
  if (threadIdx.x == 0) s_min = 0x7FF0000000000000ULL;
  const int64_t t = blockIdx.x;
  constexpr int64_t TS = (int64_t)THREADS * K_UNIF;
  const int64_t e0 = t * TS + (int64_t)threadIdx.x * K_UNIF;
  double z[K_UNIF];
  src.tile(t, n + 1, src.position(), s_words, z);  // contains __syncthreads
  unsigned long long mn = 0x7FF0000000000000ULL;
#pragma unroll
  for (int i = 0; i < K_UNIF; ++i)
    if (e0 + i <= n) mn = min(mn, zmin_key(z[i]));
  double sc[K_UNIF];
  sc[0] = z[0];
#pragma unroll
  for (int i = 1; i < K_UNIF; ++i) sc[i] = __dadd_rn(sc[i - 1], z[i]);
  block_min_u64(&s_min, mn);
  double Q, R;
  const double A = block_fold(sc[K_UNIF - 1], fs, Q, R);  // contains __syncthreads
  if (threadIdx.x == 0) {
    ws.agg[t] = A;
    ws.incl[t] = __longlong_as_double((long long)s_min);  // folded by k_chain_groups
  }
  STAMPK(0, 2);
  pdl_trigger();
  double v[K_UNIF];
#pragma unroll
  for (int i = 0; i < K_UNIF; ++i) v[i] = __dadd_rn(R, __dadd_rn(Q, sc[i]));
  if (e0 + K_UNIF <= n && vec_ok(Z + e0)) {
    store_k(Z + e0, v);
  } else {
#pragma unroll
    for (int i = 0; i < K_UNIF; ++i)
      if (e0 + i < n) Z[e0 + i] = v[i];
  }
  STAMPK(0, 3);
}

// pass 2: U = Z / Z[n] in place (memory-bound: 16 bytes per u), collapse
// sites recorded when the reference's exactness check fires (the repair and
// the device stream advance follow in k_unif_finalize).
__global__ void __launch_bounds__(THREADS) k_unif_pass2(int64_t n, int64_t nt, ScanWS ws, double* __restrict__ U) {
  __shared__ double s_last[WARPS];
  STAMPK(2, 0);
  pdl_wait();
  STAMPK(2, 1);
  constexpr int64_t TS = (int64_t)THREADS * K_UNIF;
  const int64_t t = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e0 = t * TS + (int64_t)threadIdx.x * K_UNIF;
  const double total = ws.hdr->total;
  const double C = ws.grp[t / GROUP_TILES], D = ws.incl[t];
  const bool need = ws.hdr->need != 0u;
  double u[K_UNIF];
  if (e0 + K_UNIF <= n && vec_ok(U + e0)) {
    double v[K_UNIF];
    load_k(U + e0, v);
#pragma unroll
    for (int i = 0; i < K_UNIF; ++i) u[i] = __ddiv_rn(__dadd_rn(C, __dadd_rn(D, v[i])), total);
    store_k(U + e0, u);
  } else {
#pragma unroll
    for (int i = 0; i < K_UNIF; ++i) {
      u[i] = (e0 + i < n) ? __ddiv_rn(__dadd_rn(C, __dadd_rn(D, U[e0 + i])), total) : 2.0;
      if (e0 + i < n) U[e0 + i] = u[i];
    }
  }
  pdl_trigger();
  if (need) {
    // previous U for each element: inside the chunk, from lane-1, from the
    // previous warp, or from the previous tile's last Z
    double prev_lane = __shfl_up_sync(FULL, u[K_UNIF - 1], 1);
    if (lane == 31) s_last[warp] = u[K_UNIF - 1];
    __syncthreads();
    if (lane == 0) {
      // the previous tile's last Z is its inclusive prefix, C + D of tile t
      // (or, at a group boundary, C_g = C_{g-1} + E_{g-1}: the same value)
      if (warp > 0) prev_lane = s_last[warp - 1];
      else prev_lane = (t == 0) ? 0.0 : __ddiv_rn(__dadd_rn(C, D), total);
    }
#pragma unroll
    for (int i = 0; i < K_UNIF; ++i) {
      const int64_t e = e0 + i;
      if (e < n) {
        const double pv = (i == 0) ? prev_lane : u[i - 1];
        if (u[i] <= pv) {
          const uint32_t slot = atomicAdd(&ws.hdr->nsites, 1u);
          if (slot < (uint32_t)SITE_CAP) ws.sites[slot] = (long long)e;
        }
        if (e == n - 1 && u[i] >= 1.0) atomicOr(&ws.hdr->top, 1u);
      }
    }
  }
  STAMPK(2, 3);
}

// after pass 2: the repair when pass 2 found collapse sites, the status word,
// the device stream advance, counters back to zero
__global__ void k_unif_finalize(ScanWS ws, int64_t n, double* U, int32_t* status_out, uint64_t* offset_dev) {
  STAMPK(3, 0);
  pdl_wait();
  STAMPK(3, 1);
  pdl_trigger();
  const uint32_t nsites = *(volatile uint32_t*)&ws.hdr->nsites;
  const uint32_t top = *(volatile uint32_t*)&ws.hdr->top;
  int32_t st = 0;
  if (ws.hdr->need && (nsites > 0 || top)) {
    repair_sites(U, n, ws, nsites, true);  // the backward pass stops at the first untouched entry
    st |= DRS_ST_REPAIRED;
  }
  *status_out = st;
  if (offset_dev) *offset_dev += (uint64_t)(n + 1);  // every pass-1 CTA has read it
  ws.hdr->nsites = 0;
  ws.hdr->top = 0;
  STAMPK(3, 3);
}

// ------------------------------------------------------------- uniforms ----
__global__ void k_uniforms(uint64_t k0, uint64_t k1, uint64_t offset, int64_t k, double* __restrict__ u) {
  const int64_t b = (int64_t)(offset >> 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t first = (int64_t)(offset >> 2);
  const int64_t last = (int64_t)((offset + (uint64_t)k - 1) >> 2);
  if (b > last) return;
  const U64x4 v = philox_block(k0, k1, (uint64_t)b);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t d = 4 * b + i - (int64_t)offset;
    if (d >= 0 && d < k) u[d] = u01(pick(v, i));
  }
  (void)first;
}

// --------------------------------------------------------------- host ----
int launch_top_guide(int64_t M, double* idx, cudaStream_t st);  // drs_match.cu

IndexDesc make_index_desc(int64_t M) {
  IndexDesc d{};
  d.n[0] = M;
  d.off[0] = 0;
  int64_t n = M, off = 0;
  int L = 0;
  while (n > FANOUT && L < MAX_LEVELS) {
    n = cdiv(n, FANOUT);
    ++L;
    d.n[L] = n;
    d.off[L] = off;
    off += cdiv(n, FANOUT) * FANOUT;
  }
  d.levels = L;
  d.kt = 0;
  d.tshift = 0;
  d.toff = 0;
  d.aoff = 0;
  if (L > 0) {
    int k = 1;
    while (d.n[k] > DRS_TG_ENTRIES) ++k;  // n[L] <= FANOUT, so k <= L
    int sh = 0;
    while (((int64_t)2 << sh) < d.n[k]) ++sh;  // 2^(sh+1) >= n[kt]
    d.kt = k;
    d.tshift = sh < 4 ? 4 : sh;
    d.toff = off;
    d.aoff = off + tg_doubles(d);  // a multiple of 16 doubles
  }
  return d;
}

static int launch_rc() {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

static void set_attrs() {
  static SmemLimit l1, l2, l3, l4, l5, l6;
  const size_t smem = (size_t)THREADS * K_TABLE * 8;
  l1.raise((const void*)k_table_pass1<false>, smem);
  l2.raise((const void*)k_table_pass1<true>, smem);
  l3.raise((const void*)k_table_pass2<false, false>, smem);
  l4.raise((const void*)k_table_pass2<true, false>, smem);
  l5.raise((const void*)k_table_local<false>, smem);
  l6.raise((const void*)k_table_local<true>, smem);
}

int write_direct_header(double* idx, int64_t M, cudaStream_t st);  // drs_match.cu

// dr_build_table_deferred / dr_build_table_log_deferred
static int build_deferred(const double* w, bool logw, int64_t M, double* L, double* idx, int32_t* status, void* ws,
                          size_t ws_bytes, cudaStream_t st) {
  if (M < 1 || !w || !L || !idx || !status || !ws) return DRS_ERR_ARG;
  if (((uintptr_t)w | (uintptr_t)L | (uintptr_t)idx) & 15) return DRS_ERR_ALIGN;
  const IndexDesc d = make_index_desc(M);
  const int64_t nt = cdiv(M, (int64_t)THREADS * K_TABLE);
  if (nt > ws_tile_capacity(ws_bytes)) return DRS_ERR_WORKSPACE;
  if (nt > (int64_t)CHAIN_MAX_GROUPS * GROUP_TILES) return DRS_ERR_ARG;
  set_attrs();
  const ScanWS s = carve(ws, ws_bytes);
  const int smem = THREADS * K_TABLE * 8;
  double* lvl1 = d.levels > 0 ? idx + d.off[1] : nullptr;
  double* lvl2 = d.kt >= 2 ? idx + d.off[2] : nullptr;  // level 1 stays in-tile: level 2's sources
  if (logw) {
    const int64_t mb = cdiv(M, 256 * 8);
    const unsigned mgrid = (unsigned)(mb < nt ? (mb < 1 ? 1 : mb) : nt);  // partials fit in agg[nt]
    launch_pdl(k_max_logw, dim3(mgrid < 1184 ? mgrid : 1184), dim3(256), 0, st, w, M, s);
    launch_pdl(k_table_local<true>, dim3((unsigned)nt), dim3(THREADS), smem, st, w, M, s, L, lvl1, lvl2);
  } else {
    launch_pdl(k_table_local<false>, dim3((unsigned)nt), dim3(THREADS), smem, st, w, M, s, L, lvl1, lvl2);
  }
  if (d.kt >= 2 && nt <= TAIL_MAX_TILES && !getenv("DRS_NO_TABLE_TAIL")) {
    // the chain and the levels in one launch (k_table_tail), then the guide
    static SmemLimit lim_t;
    const size_t tsmem = (size_t)(nt + nt / GROUP_TILES + 1 + cdiv(nt, GROUP_TILES)) * 8;
    lim_t.raise((const void*)k_table_tail, (size_t)(TAIL_MAX_TILES + TAIL_MAX_TILES / GROUP_TILES + 1 +
                                                     TAIL_MAX_TILES / GROUP_TILES) * 8);
    const int64_t tgrid = std::min<int64_t>(cdiv(std::max<int64_t>(d.n[2], nt), TAIL_THREADS), drs_sm_count());
    launch_pdl(k_table_tail, dim3((unsigned)tgrid), dim3(TAIL_THREADS), tsmem, st, M, nt, s, idx, d, status);
    if (launch_rc()) return DRS_ERR_LAUNCH;
    return launch_top_guide(M, idx, st);
  }
  launch_chain(s, nt, 0, status, nullptr, st);
  int64_t work = nt;
  if (d.levels > 0)
    work = std::max<int64_t>(work, std::max<int64_t>(d.kt >= 2 ? d.n[2] : cdiv(d.n[1], 2), (int64_t)FANOUT * d.levels));
  static OccupancyCache occ_l;
  const int64_t lgrid = std::min<int64_t>(cdiv(work, 256), (int64_t)drs_sm_count() * occ_l.get((const void*)k_table_levels<true>, 256, 0));
  launch_pdl(k_table_levels<true>, dim3((unsigned)lgrid), dim3(256), 0, st, M, nt, s, idx, d);
  if (launch_rc()) return DRS_ERR_LAUNCH;
  return launch_top_guide(M, idx, st);
}

// levels, top guide, then the table header and the per-tile pairs (TabAux)
int64_t index_entries(int64_t M) {
  const IndexDesc d = make_index_desc(M);
  return d.aoff + TAB_HDR + 2 * table_tiles(M);
}

int64_t ws_capacity_tiles(size_t ws_bytes) { return ws_tile_capacity(ws_bytes); }
ScanWS carve_ws(void* ws, size_t ws_bytes) { return carve(ws, ws_bytes); }

template <class Src>
static int sorted_impl(const Src& src, int64_t n, double* U, int32_t* status, void* ws,
                       size_t ws_bytes, uint64_t* offset_dev, cudaStream_t st) {
  const int64_t nt = cdiv(n + 1, (int64_t)THREADS * K_UNIF);
  if (nt > ws_tile_capacity(ws_bytes)) return DRS_ERR_WORKSPACE;
  if (nt > (int64_t)CHAIN_MAX_GROUPS * GROUP_TILES) return DRS_ERR_ARG;
  const ScanWS s = carve(ws, ws_bytes);
  launch_pdl(k_unif_pass1<Src>, dim3((unsigned)nt), dim3(THREADS), 0, st, src, n, s, U);
  launch_chain(s, nt, 1, nullptr, nullptr, st);
  launch_pdl(k_unif_pass2, dim3((unsigned)nt), dim3(THREADS), 0, st, n, nt, s, U);
  launch_pdl(k_unif_finalize, dim3(1), dim3(1), 0, st, s, n, U, status, offset_dev);
  return launch_rc();
}

int sorted_uniforms_launch(uint64_t k0, uint64_t k1, uint64_t offset, const uint64_t* offset_dev,
                           int64_t n, double* U, int32_t* status, void* ws, size_t ws_bytes,
                           cudaStream_t st) {
  PhiloxSpacings src{k0, k1, offset, offset_dev};
  return sorted_impl(src, n, U, status, ws, ws_bytes, const_cast<uint64_t*>(offset_dev), st);
}

int sorted_uniforms_from_launch(const double* raw, int64_t n, double* U, int32_t* status, void* ws,
                                size_t ws_bytes, cudaStream_t st) {
  ArraySpacings src{raw};
  return sorted_impl(src, n, U, status, ws, ws_bytes, nullptr, st);
}

// the levels of a shard whose header is in place (dr_shard_finalize_deferred, drs_shard.cu)
int launch_table_levels_from_aux(int64_t M, double* idx, cudaStream_t st) {
  const IndexDesc d = make_index_desc(M);
  const ScanWS none{};
  int64_t work = 1;
  if (d.levels > 0) work = std::max<int64_t>(d.kt >= 2 ? d.n[2] : cdiv(d.n[1], 2), (int64_t)FANOUT * d.levels);
  static OccupancyCache occ_l;
  const int64_t lgrid = std::min<int64_t>(cdiv(work, 256), (int64_t)drs_sm_count() * occ_l.get((const void*)k_table_levels<false>, 256, 0));
  launch_pdl(k_table_levels<false>, dim3((unsigned)lgrid), dim3(256), 0, st, M, (int64_t)0, none, idx, d);
  if (launch_rc()) return DRS_ERR_LAUNCH;
  return launch_top_guide(M, idx, st);
}

// one cooperative launch when the spacings fit a co-resident grid, else the pipeline above (drs_fused.cu)
int sorted_uniforms_auto(uint64_t k0, uint64_t k1, uint64_t offset, uint64_t* offset_dev, const double* raw,
                         int64_t n, double* U, int32_t* status, void* ws, size_t ws_bytes, cudaStream_t st);

}  // namespace drs

using namespace drs;

extern "C" {

const char* dr_version(void) { return "drs 0.1.0 (sm_100a)"; }

const char* dr_strerror(int code) {
  switch (code) {
    case DRS_OK: return "ok";
    case DRS_ERR_ARG: return "invalid argument";
    case DRS_ERR_WORKSPACE: return "workspace too small";
    case DRS_ERR_LAUNCH: return "CUDA launch failed";
    case DRS_ERR_ALIGN: return "pointer misaligned";
    case DRS_ERR_MODE: return "unknown mode";
    default: return "unknown error";
  }
}

int dr_stream_synchronize(void* stream) {
  return cudaStreamSynchronize((cudaStream_t)stream) == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

int dr_device_accessible(const void* p) {
  cudaPointerAttributes a;
  if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return 1;
  return (a.type == cudaMemoryTypeHost && a.devicePointer == p) ? 1 : 0;
}

void dr_scan_geometry(int32_t g[6]) {
  g[0] = LANES; g[1] = WARPS; g[2] = K_TABLE; g[3] = K_UNIF; g[4] = FANOUT; g[5] = GROUP_TILES;
}

size_t dr_workspace_bytes(int op, int64_t M, int64_t N, int64_t B) {
  (void)B;
  int64_t nt = 1;
  if (op == DRS_OP_TABLE) nt = cdiv(M > 0 ? M : 1, (int64_t)THREADS * K_TABLE);
  else if (op == DRS_OP_SORTED) nt = cdiv((N > 0 ? N : 0) + 1, (int64_t)THREADS * K_UNIF);
  return ws_fixed_bytes() + 20 * (size_t)nt + 64;
}

int dr_workspace_init(void* ws, size_t ws_bytes, void* stream) {
  if (!ws || ws_bytes < ws_fixed_bytes()) return DRS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(ws, 0, ws_bytes, st) != cudaSuccess) return DRS_ERR_LAUNCH;
  k_ws_init<<<1, 1, 0, st>>>((ScanHdr*)ws);
  return launch_rc();
}

int64_t dr_index_entries(int64_t M) { return M > 0 ? index_entries(M) : 0; }

int dr_build_table(const double* w, int64_t M, double* W, double* idx, int32_t* status, void* ws,
                   size_t ws_bytes, void* stream) {
  if (M < 1 || !w || !W || !status || !ws) return DRS_ERR_ARG;
  if (((uintptr_t)w | (uintptr_t)W) & 15) return DRS_ERR_ALIGN;
  const IndexDesc d = make_index_desc(M);
  if (d.levels > 0 && !idx) return DRS_ERR_ARG;
  const int64_t nt = cdiv(M, (int64_t)THREADS * K_TABLE);
  if (nt > ws_tile_capacity(ws_bytes)) return DRS_ERR_WORKSPACE;
  if (nt > (int64_t)CHAIN_MAX_GROUPS * GROUP_TILES) return DRS_ERR_ARG;
  set_attrs();
  const ScanWS s = carve(ws, ws_bytes);
  cudaStream_t st = (cudaStream_t)stream;
  const int smem = THREADS * K_TABLE * 8;
  launch_pdl(k_table_pass1<false>, dim3((unsigned)nt), dim3(THREADS), smem, st, w, M, s, (double*)nullptr);
  launch_chain(s, nt, 0, status, nullptr, st);
  launch_pdl(k_table_pass2<false, false>, dim3((unsigned)nt), dim3(THREADS), smem, st, w, M, nt, s, W, idx, d,
             status, (double*)nullptr);
  if (launch_rc() || write_direct_header(idx, M, st)) return DRS_ERR_LAUNCH;
  return launch_top_guide(M, idx, st);
}

int dr_build_table_deferred(const double* w, int64_t M, double* V, double* idx, int32_t* status, void* ws,
                            size_t ws_bytes, void* stream) {
  return build_deferred(w, false, M, V, idx, status, ws, ws_bytes, (cudaStream_t)stream);
}

int dr_build_table_log_deferred(const double* logw, int64_t M, double* V, double* idx, int32_t* status, void* ws,
                                size_t ws_bytes, void* stream) {
  return build_deferred(logw, true, M, V, idx, status, ws, ws_bytes, (cudaStream_t)stream);
}

int dr_table_materialize(const double* V, const double* idx, int64_t M, double* W, void* stream) {
  if (M < 1 || !V || !W) return DRS_ERR_ARG;
  const IndexDesc d = make_index_desc(M);
  const int64_t blocks = cdiv(M, 256) < 148 * 16 ? cdiv(M, 256) : 148 * 16;
  k_table_materialize<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(V, M, idx ? idx + d.aoff : nullptr, W);
  return launch_rc();
}

int dr_build_table_log(const double* logw, int64_t M, double* W, double* idx, int32_t* status, void* ws,
                       size_t ws_bytes, void* stream) {
  if (M < 1 || !logw || !W || !status || !ws) return DRS_ERR_ARG;
  if (((uintptr_t)logw | (uintptr_t)W) & 15) return DRS_ERR_ALIGN;
  const IndexDesc d = make_index_desc(M);
  if (d.levels > 0 && !idx) return DRS_ERR_ARG;
  const int64_t nt = cdiv(M, (int64_t)THREADS * K_TABLE);
  if (nt > ws_tile_capacity(ws_bytes)) return DRS_ERR_WORKSPACE;
  if (nt > (int64_t)CHAIN_MAX_GROUPS * GROUP_TILES) return DRS_ERR_ARG;
  set_attrs();
  const ScanWS s = carve(ws, ws_bytes);
  cudaStream_t st = (cudaStream_t)stream;
  const int smem = THREADS * K_TABLE * 8;
  const int64_t mb = cdiv(M, 256 * 8);
  const unsigned mgrid = (unsigned)(mb < nt ? (mb < 1 ? 1 : mb) : nt);  // partials fit in agg[nt]
  launch_pdl(k_max_logw, dim3(mgrid < 1184 ? mgrid : 1184), dim3(256), 0, st, logw, M, s);
  launch_pdl(k_table_pass1<true>, dim3((unsigned)nt), dim3(THREADS), smem, st, logw, M, s, W);  // w -> W
  launch_chain(s, nt, 0, status, nullptr, st);
  launch_pdl(k_table_pass2<false, false>, dim3((unsigned)nt), dim3(THREADS), smem, st, (const double*)W, M, nt, s,
             W, idx, d, status, (double*)nullptr);
  if (launch_rc() || write_direct_header(idx, M, st)) return DRS_ERR_LAUNCH;
  return launch_top_guide(M, idx, st);
}

int dr_shard_scan(const double* w_shard, int64_t Mg, double* S, double* Tg, int32_t* status,
                  void* ws, size_t ws_bytes, void* stream) {
  if (Mg < 1 || !w_shard || !S || !Tg || !status || !ws) return DRS_ERR_ARG;
  if (((uintptr_t)w_shard | (uintptr_t)S) & 15) return DRS_ERR_ALIGN;
  const int64_t nt = cdiv(Mg, (int64_t)THREADS * K_TABLE);
  if (nt > ws_tile_capacity(ws_bytes)) return DRS_ERR_WORKSPACE;
  if (nt > (int64_t)CHAIN_MAX_GROUPS * GROUP_TILES) return DRS_ERR_ARG;
  set_attrs();
  const ScanWS s = carve(ws, ws_bytes);
  cudaStream_t st = (cudaStream_t)stream;
  const int smem = THREADS * K_TABLE * 8;
  const IndexDesc d = make_index_desc(Mg);
  launch_pdl(k_table_pass1<false>, dim3((unsigned)nt), dim3(THREADS), smem, st, w_shard, Mg, s, (double*)nullptr);
  launch_chain(s, nt, 0, status, Tg, st);
  launch_pdl(k_table_pass2<true, false>, dim3((unsigned)nt), dim3(THREADS), smem, st, w_shard, Mg, nt, s, S,
             (double*)nullptr, d, status, Tg);
  return launch_rc();
}

int dr_shard_scan_deferred(const double* w_shard, int64_t Mg, double* V, double* idx, double* Tg, int32_t* status,
                           void* ws, size_t ws_bytes, void* stream) {
  if (Mg < 1 || !w_shard || !V || !idx || !Tg || !status || !ws) return DRS_ERR_ARG;
  if (((uintptr_t)w_shard | (uintptr_t)V | (uintptr_t)idx) & 15) return DRS_ERR_ALIGN;
  const IndexDesc d = make_index_desc(Mg);
  const int64_t nt = cdiv(Mg, (int64_t)THREADS * K_TABLE);
  if (nt > ws_tile_capacity(ws_bytes)) return DRS_ERR_WORKSPACE;
  if (nt > (int64_t)CHAIN_MAX_GROUPS * GROUP_TILES) return DRS_ERR_ARG;
  set_attrs();
  const ScanWS s = carve(ws, ws_bytes);
  cudaStream_t st = (cudaStream_t)stream;
  const int smem = THREADS * K_TABLE * 8;
  launch_pdl(k_table_local<false>, dim3((unsigned)nt), dim3(THREADS), smem, st, w_shard, Mg, s, V,
             d.levels > 0 ? idx + d.off[1] : (double*)nullptr, (double*)nullptr);
  launch_chain(s, nt, 0, status, Tg, st);
  launch_pdl(k_table_pairs, dim3((unsigned)std::min<int64_t>(cdiv(nt, 256), 1184)), dim3(256), 0, st, nt, s,
             idx + d.aoff);
  return launch_rc();
}

int dr_uniforms(uint64_t k0, uint64_t k1, uint64_t offset, int64_t k, double* u, void* stream) {
  if (k < 0 || (k > 0 && !u)) return DRS_ERR_ARG;
  if (k == 0) return DRS_OK;
  const int64_t blocks = (int64_t)((offset + (uint64_t)k - 1) >> 2) - (int64_t)(offset >> 2) + 1;
  const int tpb = 256;
  k_uniforms<<<(unsigned)cdiv(blocks, tpb), tpb, 0, (cudaStream_t)stream>>>(k0, k1, offset, k, u);
  return launch_rc();
}

int dr_sorted_uniforms(uint64_t k0, uint64_t k1, uint64_t offset, int64_t n, double* U,
                       int32_t* status, void* ws, size_t ws_bytes, void* stream) {
  if (n < 1 || !U || !status || !ws) return DRS_ERR_ARG;
  return sorted_uniforms_auto(k0, k1, offset, nullptr, nullptr, n, U, status, ws, ws_bytes, (cudaStream_t)stream);
}

int dr_sorted_uniforms_from(const double* raw, int64_t n, double* U, int32_t* status, void* ws,
                            size_t ws_bytes, void* stream) {
  if (n < 1 || !raw || !U || !status || !ws) return DRS_ERR_ARG;
  return sorted_uniforms_auto(0, 0, 0, nullptr, raw, n, U, status, ws, ws_bytes, (cudaStream_t)stream);
}

}  // extern "C"
