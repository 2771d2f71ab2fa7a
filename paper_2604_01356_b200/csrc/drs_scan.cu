// drs_scan.cu -- the two fp64 scans of the resampling path on sm_100a.
//
//   K1 build_table     (cdf.py:59-89)      raw w -> W = S/T, W[M-1] == 1, + search index
//   K2 sorted_uniforms (randkit.py:70-101) Philox draws -> -log -> Z -> U = Z/Z[n], + repair
//
// Both are reduce-then-scan over tiles of THREADS*K elements:
//   pass 1: tile aggregate A_t (chained fold), then a
//           decoupled look-back publishes the chained inclusive prefix
//           incl[t] = incl[t-1] + A_t (left fold from the nearest published
//           inclusive, so the value is the same whichever predecessor was found);
//   pass 2: recompute the tile chain, S = P + (R + (Q + s)), apply the epilogue.
// The table pass reads w twice and writes W once (24 bytes per entry); the
// uniform pass regenerates its draws in pass 2 and writes only U (8 bytes per u).
#include "drs_common.cuh"

namespace drs {

// ------------------------------------------------------ workspace layout ----
static constexpr size_t kHdr = 64;

__host__ inline size_t ws_fixed_bytes() { return kHdr + 8 * (size_t)SITE_CAP + 64; }

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
  s.flags = (uint32_t*)(b + o);
  o += 4 * (size_t)C;
  o = (o + 15) & ~(size_t)15;
  s.agg = (double*)(b + o);
  o += 8 * (size_t)C;
  s.incl = (double*)(b + o);
  o += 8 * (size_t)C;
  s.sites = (long long*)(b + o);
  return s;
}

__global__ void k_ws_init(ScanHdr* h) {
  h->ticket = 0; h->done1 = 0; h->done2 = 0; h->epoch = 1;
  h->status = 0; h->nsites = 0; h->top = 0; h->bar_count = 0; h->bar_gen = 0;
  h->zmin_bits = 0x7FF0000000000000ULL;
}

// --------------------------------------------------------- tile chain ----
// Q: fold of previous lane-chunk totals in the warp; R: fold of previous warp
// totals in the tile; returns A = tile total.  Serial folds, starting at 0.0.
__device__ __forceinline__ double chain_fold(double tau, double* s_g, double& Q, double& R) {
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
  return r;
}

// Decoupled look-back, executed by warp 0.  Returns the exclusive prefix P_t.
// The warp inspects 32 predecessors at a time; a window holding only
// aggregates is stashed in shared memory and the walk continues further back
// (up to LB_MAXW windows), so the inclusive frontier is never a bottleneck.
// The prefix is always the left fold incl[k] + agg[k+1] + ... + agg[t-1]
// from the nearest published inclusive k, which equals the chained value
// incl[t-1] bit for bit whichever k was found.
constexpr int LB_MAXW = 16;

__device__ double lookback(const ScanWS& ws, int64_t t, uint32_t ep, double A, double* s_win) {
  const int lane = threadIdx.x & 31;
  if (t == 0) {
    const double I = __dadd_rn(0.0, A);
    if (lane == 0) {
      st_relaxed_f64(&ws.incl[0], I);
      st_release_u32(&ws.flags[0], (ep << 2) | 2u);
    }
    return 0.0;
  }
  if (lane == 0) {
    st_relaxed_f64(&ws.agg[t], A);
    st_release_u32(&ws.flags[t], (ep << 2) | 1u);
  }
  int64_t base = t - 1;
  int nw = 0;
  double P = 0.0;
  int spins = 0;
  while (true) {
    const int64_t tt = base - lane;
    uint32_t st = 0;
    if (tt >= 0) {
      const uint32_t f = ld_acquire_u32(&ws.flags[tt]);
      st = ((f >> 2) == ep) ? (f & 3u) : 0u;
    }
    const uint32_t incl_mask = __ballot_sync(FULL, st == 2u);
    const uint32_t avail_mask = __ballot_sync(FULL, st != 0u);
    if (incl_mask) {
      const int j = __ffs(incl_mask) - 1;
      const uint32_t need = (j == 0) ? 0u : ((1u << j) - 1u);
      if ((avail_mask & need) == need) {
        double val = 0.0;
        if (lane == j) val = ld_relaxed_f64(&ws.incl[tt]);
        else if (lane < j) val = ld_relaxed_f64(&ws.agg[tt]);
        P = __shfl_sync(FULL, val, j);
        for (int k = j - 1; k >= 0; --k) P = __dadd_rn(P, __shfl_sync(FULL, val, k));
        break;
      }
    } else if (avail_mask == FULL && nw < LB_MAXW) {
      s_win[nw * 32 + lane] = ld_relaxed_f64(&ws.agg[tt]);
      __syncwarp();
      ++nw;
      base -= 32;
      spins = 0;
      continue;
    }
    if (++spins > 4) __nanosleep(32);
  }
  for (int w = nw - 1; w >= 0; --w)
    for (int k = 31; k >= 0; --k) P = __dadd_rn(P, s_win[w * 32 + k]);
  const double I = __dadd_rn(P, A);
  if (lane == 0) {
    st_relaxed_f64(&ws.incl[t], I);
    st_release_u32(&ws.flags[t], (ep << 2) | 2u);
  }
  return P;
}

// pass-1 epilogue common to all sources: completion count, epoch bump
__device__ __forceinline__ void pass1_finish(const ScanWS& ws, uint32_t ep) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ws.hdr->done1, 1u) == gridDim.x - 1) {
      uint32_t ne = (ep + 1) & 0x3FFFFFFFu;
      if (ne == 0) ne = 1;
      ws.hdr->epoch = ne;
      ws.hdr->ticket = 0;
      ws.hdr->done1 = 0;
      __threadfence();
    }
  }
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

__global__ void __launch_bounds__(THREADS) k_table_pass1(const double* __restrict__ w, int64_t n,
                                                         ScanWS ws) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double s_g[WARPS];
  __shared__ int64_t s_tile;
  __shared__ uint32_t s_ep;
  __shared__ double s_win[LB_MAXW * 32];
  if (threadIdx.x == 0) {
    s_tile = (int64_t)atomicAdd(&ws.hdr->ticket, 1u);
    s_ep = *(volatile uint32_t*)&ws.hdr->epoch;
  }
  __syncthreads();
  const int64_t t = s_tile;
  const uint32_t ep = s_ep;
  stage_tile<K_TABLE>(w, n, t, sm, &bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* chunk = sm + (warp * LANES + lane) * K_TABLE;
  double s = chunk[0];
  bool bad = !(s >= 0.0 && s < dinf());
#pragma unroll
  for (int i = 1; i < K_TABLE; ++i) {
    const double x = chunk[i];
    bad |= !(x >= 0.0 && x < dinf());
    s = __dadd_rn(s, x);
  }
  double Q, R;
  const double A = chain_fold(s, s_g, Q, R);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&ws.hdr->status, (uint32_t)DRS_ST_INVALID_WEIGHT);
  if (warp == 0) lookback(ws, t, ep, A, s_win);
  pass1_finish(ws, ep);
}

// RAW = false: W = min(S/T, 1) with W[n-1] = 1 and the index levels (dr_build_table)
// RAW = true:  the unnormalised local prefix S and *total_out = T (dr_shard_scan)
template <bool RAW>
__global__ void __launch_bounds__(THREADS) k_table_pass2(const double* __restrict__ w, int64_t n,
                                                         int64_t nt, ScanWS ws,
                                                         double* __restrict__ W,
                                                         double* __restrict__ idx, IndexDesc d,
                                                         int32_t* status_out, double* total_out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double s_g[WARPS];
  constexpr int64_t TS = (int64_t)THREADS * K_TABLE;
  const int64_t t = blockIdx.x;
  const int64_t len = stage_tile<K_TABLE>(w, n, t, sm, &bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* chunk = sm + (warp * LANES + lane) * K_TABLE;
  double s = chunk[0];
#pragma unroll
  for (int i = 1; i < K_TABLE; ++i) s = __dadd_rn(s, chunk[i]);
  double Q, R;
  chain_fold(s, s_g, Q, R);
  const double P = (t == 0) ? 0.0 : ws.incl[t - 1];
  const double T = ws.incl[nt - 1];
  const int64_t jb = t * TS + (int64_t)(warp * LANES + lane) * K_TABLE;
  double s2 = 0.0;
#pragma unroll
  for (int i = 0; i < K_TABLE; ++i) {
    const double x = chunk[i];
    s2 = (i == 0) ? x : __dadd_rn(s2, x);
    const double S = __dadd_rn(P, __dadd_rn(R, __dadd_rn(Q, s2)));
    const int64_t j = jb + i;
    if (RAW) {
      chunk[i] = S;
      continue;
    }
    double v = fmin(__ddiv_rn(S, T), 1.0);
    if (j == n - 1) v = 1.0;
    chunk[i] = v;
    if (j < n && ((j & (FANOUT - 1)) == FANOUT - 1 || j == n - 1)) {
      int64_t span = FANOUT;
      for (int k = 1; k <= d.levels; ++k, span *= FANOUT) {
        const bool edge = ((j + 1) % span) == 0;
        if (!edge && j != n - 1) break;
        idx[d.off[k] + j / span] = v;
        if (j == n - 1) {
          const int64_t padded = cdiv(d.n[k], FANOUT) * FANOUT;
          for (int64_t p = d.n[k]; p < padded; ++p) idx[d.off[k] + p] = dinf();
        }
      }
    }
  }
  fence_proxy_async_smem();
  __syncthreads();
  const int64_t len_even = len & ~(int64_t)1;
  if (threadIdx.x == 0) {
    if (len_even > 0) {
      bulk_s2g(W + t * TS, sm, (uint32_t)(len_even * 8));
      bulk_commit_wait();
    }
    if (len & 1) W[t * TS + len - 1] = sm[len - 1];
    __threadfence();
    if (atomicAdd(&ws.hdr->done2, 1u) == gridDim.x - 1) {
      uint32_t st = *(volatile uint32_t*)&ws.hdr->status;
      if (T == 0.0) st |= DRS_ST_DEGENERATE;
      if (!(T < dinf())) st |= DRS_ST_ACCUM_OVERFLOW;
      *status_out = (int32_t)st;
      if (RAW) *total_out = T;
      ws.hdr->status = 0;
      ws.hdr->done2 = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------- K2 sorted uniforms ----
// Spacing sources: element e (0 <= e <= n) of the n+1 spacings.
struct PhiloxSpacings {
  uint64_t k0, k1, offset;
  const uint64_t* offset_dev;  // device-resident stream position (graph capture)
  // the K_UNIF = 4 consecutive spacings starting at e0
  __device__ __forceinline__ void chunk4(int64_t e0, int64_t count, double z[4]) const {
    const uint64_t off = offset_dev ? *(volatile const uint64_t*)offset_dev : offset;
    const uint64_t d0 = off + (uint64_t)e0;
    const uint64_t b0 = d0 >> 2, b1 = (d0 + 3) >> 2;
    const U64x4 v0 = philox_block(k0, k1, b0);
    U64x4 v1 = v0;
    if (b1 != b0) v1 = philox_block(k0, k1, b1);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint64_t dd = d0 + (uint64_t)i;
      const uint64_t raw = ((dd >> 2) == b0) ? pick(v0, (int)(dd & 3)) : pick(v1, (int)(dd & 3));
      z[i] = (e0 + i < count) ? neglog(u01(raw)) : 0.0;
    }
  }
};

struct ArraySpacings {
  const double* raw;
  __device__ __forceinline__ void chunk4(int64_t e0, int64_t count, double z[4]) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) z[i] = (e0 + i < count) ? neglog(raw[e0 + i]) : 0.0;
  }
};

__device__ __forceinline__ unsigned long long zmin_key(double z) {
  // positive doubles order like their bit patterns; NaN / <= 0 force the exact check
  if (!(z > 0.0)) return 0ull;
  return (unsigned long long)__double_as_longlong(z);
}

template <class Src>
__global__ void __launch_bounds__(THREADS) k_unif_pass1(Src src, int64_t n, ScanWS ws) {
  __shared__ double s_g[WARPS];
  __shared__ int64_t s_tile;
  __shared__ uint32_t s_ep;
  __shared__ unsigned long long s_min;
  __shared__ double s_win[LB_MAXW * 32];
  if (threadIdx.x == 0) {
    s_tile = (int64_t)atomicAdd(&ws.hdr->ticket, 1u);
    s_ep = *(volatile uint32_t*)&ws.hdr->epoch;
    s_min = 0x7FF0000000000000ULL;
  }
  __syncthreads();
  const int64_t t = s_tile;
  const uint32_t ep = s_ep;
  constexpr int64_t TS = (int64_t)THREADS * K_UNIF;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e0 = t * TS + (int64_t)(warp * LANES + lane) * K_UNIF;
  double z[4];
  src.chunk4(e0, n + 1, z);
  unsigned long long mn = 0x7FF0000000000000ULL;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (e0 + i <= n) mn = min(mn, zmin_key(z[i]));
  double s = z[0];
#pragma unroll
  for (int i = 1; i < 4; ++i) s = __dadd_rn(s, z[i]);
  atomicMin(&s_min, mn);
  double Q, R;
  const double A = chain_fold(s, s_g, Q, R);  // contains __syncthreads
  if (threadIdx.x == 0) atomicMin(&ws.hdr->zmin_bits, s_min);
  if (warp == 0) lookback(ws, t, ep, A, s_win);
  pass1_finish(ws, ep);
}

__device__ void repair_sites(double* U, int64_t n, const ScanWS& ws, uint32_t nsites, bool top) {
  // forward pass of randkit.py:107-111 restricted to the recorded collapse
  // sites (every other position satisfies U[i] > lo and is left alone)
  long long* sites = ws.sites;
  if (nsites > (uint32_t)SITE_CAP) {
    double lo = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double v = ld_relaxed_f64(U + i);
      if (v <= lo) { v = nextafter(lo, 1.0); U[i] = v; }
      lo = v;
    }
  } else {
    for (uint32_t a = 1; a < nsites; ++a) {  // insertion sort, nsites is tiny
      const long long key = sites[a];
      int b = (int)a - 1;
      while (b >= 0 && sites[b] > key) { sites[b + 1] = sites[b]; --b; }
      sites[b + 1] = key;
    }
    int64_t done_to = -1;
    for (uint32_t a = 0; a < nsites; ++a) {
      int64_t i = sites[a];
      if (i <= done_to) continue;
      double lo = (i == 0) ? 0.0 : ld_relaxed_f64(U + i - 1);
      while (i < n) {
        const double v = ld_relaxed_f64(U + i);
        if (!(v <= lo)) break;
        const double nv = nextafter(lo, 1.0);
        U[i] = nv;
        lo = nv;
        ++i;
      }
      done_to = i;
    }
  }
  // backward pass (randkit.py:112-116): stops at the first untouched entry,
  // after which the forward-repaired prefix is strictly increasing below it
  (void)top;
  double hi = 1.0;
  for (int64_t i = n - 1; i >= 0; --i) {
    const double v = ld_relaxed_f64(U + i);
    if (!(v >= hi)) break;
    const double nv = nextafter(hi, 0.0);
    U[i] = nv;
    hi = nv;
  }
}

template <class Src>
__global__ void __launch_bounds__(THREADS) k_unif_pass2(Src src, int64_t n, int64_t nt, ScanWS ws,
                                                        double* __restrict__ U,
                                                        int32_t* status_out) {
  __shared__ double s_g[WARPS];
  __shared__ double s_last[WARPS];
  constexpr int64_t TS = (int64_t)THREADS * K_UNIF;
  const int64_t t = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e0 = t * TS + (int64_t)(warp * LANES + lane) * K_UNIF;
  double z[4];
  src.chunk4(e0, n + 1, z);
  double sc[4];
  sc[0] = z[0];
#pragma unroll
  for (int i = 1; i < 4; ++i) sc[i] = __dadd_rn(sc[i - 1], z[i]);
  double Q, R;
  chain_fold(sc[3], s_g, Q, R);
  const double P = (t == 0) ? 0.0 : ws.incl[t - 1];
  const double total = ws.incl[nt - 1];
  const double zmin = __longlong_as_double((long long)*(volatile unsigned long long*)&ws.hdr->zmin_bits);
  const bool need = !(zmin > __dmul_rn(1e-14, total));
  double u[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double Z = __dadd_rn(P, __dadd_rn(R, __dadd_rn(Q, sc[i])));
    u[i] = __ddiv_rn(Z, total);
    if (e0 + i < n) U[e0 + i] = u[i];
  }
  if (need) {
    // previous U for each element: inside the chunk, from lane-1, from the
    // previous warp, or from the previous tile's last Z (= incl[t-1])
    double prev_lane = __shfl_up_sync(FULL, u[3], 1);
    if (lane == 31) s_last[warp] = u[3];
    __syncthreads();
    if (lane == 0) {
      if (warp > 0) prev_lane = s_last[warp - 1];
      else prev_lane = (t == 0) ? 0.0 : __ddiv_rn(P, total);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
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
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ws.hdr->done2, 1u) == gridDim.x - 1) {
      __threadfence();
      const uint32_t nsites = *(volatile uint32_t*)&ws.hdr->nsites;
      const uint32_t top = *(volatile uint32_t*)&ws.hdr->top;
      int32_t st = 0;
      if (need && (nsites > 0 || top)) {
        repair_sites(U, n, ws, nsites, top != 0);
        st |= DRS_ST_REPAIRED;
      }
      *status_out = st;
      ws.hdr->nsites = 0;
      ws.hdr->top = 0;
      ws.hdr->zmin_bits = 0x7FF0000000000000ULL;
      ws.hdr->done2 = 0;
      __threadfence();
    }
  }
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
  return d;
}

static int launch_rc() {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

static bool g_attr_done = false;
static void set_attrs() {
  if (g_attr_done) return;
  const int smem = THREADS * K_TABLE * 8;
  cudaFuncSetAttribute(k_table_pass1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_table_pass2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_table_pass2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  g_attr_done = true;
}

int64_t index_entries(int64_t M) {
  const IndexDesc d = make_index_desc(M);
  if (d.levels == 0) return 0;
  return d.off[d.levels] + cdiv(d.n[d.levels], FANOUT) * FANOUT;
}

int64_t ws_capacity_tiles(size_t ws_bytes) { return ws_tile_capacity(ws_bytes); }
ScanWS carve_ws(void* ws, size_t ws_bytes) { return carve(ws, ws_bytes); }

template <class Src>
static int sorted_impl(const Src& src, int64_t n, double* U, int32_t* status, void* ws,
                       size_t ws_bytes, cudaStream_t st) {
  const int64_t nt = cdiv(n + 1, (int64_t)THREADS * K_UNIF);
  if (nt > ws_tile_capacity(ws_bytes)) return DRS_ERR_WORKSPACE;
  const ScanWS s = carve(ws, ws_bytes);
  k_unif_pass1<Src><<<(unsigned)nt, THREADS, 0, st>>>(src, n, s);
  k_unif_pass2<Src><<<(unsigned)nt, THREADS, 0, st>>>(src, n, nt, s, U, status);
  return launch_rc();
}

int sorted_uniforms_launch(uint64_t k0, uint64_t k1, uint64_t offset, const uint64_t* offset_dev,
                           int64_t n, double* U, int32_t* status, void* ws, size_t ws_bytes,
                           cudaStream_t st) {
  PhiloxSpacings src{k0, k1, offset, offset_dev};
  const int rc = sorted_impl(src, n, U, status, ws, ws_bytes, st);
  if (rc || !offset_dev) return rc;
  k_advance_offset<<<1, 1, 0, st>>>(const_cast<uint64_t*>(offset_dev), (uint64_t)(n + 1));
  return launch_rc();
}

int sorted_uniforms_from_launch(const double* raw, int64_t n, double* U, int32_t* status, void* ws,
                                size_t ws_bytes, cudaStream_t st) {
  ArraySpacings src{raw};
  return sorted_impl(src, n, U, status, ws, ws_bytes, st);
}

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

void dr_scan_geometry(int32_t g[5]) {
  g[0] = LANES; g[1] = WARPS; g[2] = K_TABLE; g[3] = K_UNIF; g[4] = FANOUT;
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
  set_attrs();
  const ScanWS s = carve(ws, ws_bytes);
  cudaStream_t st = (cudaStream_t)stream;
  const int smem = THREADS * K_TABLE * 8;
  k_table_pass1<<<(unsigned)nt, THREADS, smem, st>>>(w, M, s);
  k_table_pass2<false><<<(unsigned)nt, THREADS, smem, st>>>(w, M, nt, s, W, idx, d, status, nullptr);
  return launch_rc();
}

int dr_shard_scan(const double* w_shard, int64_t Mg, double* S, double* Tg, int32_t* status,
                  void* ws, size_t ws_bytes, void* stream) {
  if (Mg < 1 || !w_shard || !S || !Tg || !status || !ws) return DRS_ERR_ARG;
  if (((uintptr_t)w_shard | (uintptr_t)S) & 15) return DRS_ERR_ALIGN;
  const int64_t nt = cdiv(Mg, (int64_t)THREADS * K_TABLE);
  if (nt > ws_tile_capacity(ws_bytes)) return DRS_ERR_WORKSPACE;
  set_attrs();
  const ScanWS s = carve(ws, ws_bytes);
  cudaStream_t st = (cudaStream_t)stream;
  const int smem = THREADS * K_TABLE * 8;
  const IndexDesc d = make_index_desc(Mg);
  k_table_pass1<<<(unsigned)nt, THREADS, smem, st>>>(w_shard, Mg, s);
  k_table_pass2<true><<<(unsigned)nt, THREADS, smem, st>>>(w_shard, Mg, nt, s, S, nullptr, d, status, Tg);
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
  return sorted_uniforms_launch(k0, k1, offset, nullptr, n, U, status, ws, ws_bytes, (cudaStream_t)stream);
}

int dr_sorted_uniforms_from(const double* raw, int64_t n, double* U, int32_t* status, void* ws,
                            size_t ws_bytes, void* stream) {
  if (n < 1 || !raw || !U || !status || !ws) return DRS_ERR_ARG;
  ArraySpacings src{raw};
  return sorted_impl(src, n, U, status, ws, ws_bytes, (cudaStream_t)stream);
}

}  // extern "C"
