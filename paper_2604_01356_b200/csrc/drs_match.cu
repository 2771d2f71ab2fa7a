// drs_match.cu -- the three inverse-CMF searches and their validators (sm_100a).
//
//   K4 match_binary / sample_binary  (samplers.py:93-97, 238-252)
//        one lane per u, 16-ary descent of the table's index: one 128-byte
//        line (4 x 256-bit loads) per level, W itself only at the last level.
//   K5 match_ccf                     (samplers.py:100-107, 162-188)
//        W streamed once: one CTA per W tile (TMA bulk copy into shared
//        memory), its u-run found by warp 32-ary searches of U, then a
//        bisection per u (short runs) or merge path (long runs).
//   K6 match_dac                     (samplers.py:110-146, 191-210)
//        divide step = the U-range split by W tiles (merge mode) or by index
//        blocks (search mode); AUTO picks merge when M <= tau*N.
// All three return the unique lower bound: first j with W[j] >= u (W[j] < u
// compared strictly, ties to the first of an equal run), clamped to M-1.
#include <cstdlib>

#include "drs_common.cuh"

namespace drs {

IndexDesc make_index_desc(int64_t M);  // drs_scan.cu

constexpr int64_t DAC_TAU = DRS_DAC_TAU;  // drs_common.cuh

static int launch_rc() {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

// ------------------------------------------------------- K4 index search ----
__global__ void __launch_bounds__(256) k_match_index(const double* __restrict__ W,
                                                     const double* __restrict__ idx, IndexDesc d,
                                                     const double* __restrict__ u, int64_t N,
                                                     int64_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  out[i] = index_lower_bound(W, idx, d, load_aux(idx ? idx + d.aoff : nullptr), __ldg(u + i));
}

// fused binary_sampler: the warp's 32 consecutive draws come from <= 9 Philox
// blocks, computed once by lanes 0..8 and distributed by shuffles
__global__ void __launch_bounds__(256) k_sample_binary(const double* __restrict__ W,
                                                       const double* __restrict__ idx, IndexDesc d,
                                                       uint64_t k0, uint64_t k1, uint64_t offset,
                                                       int64_t N, int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) - lane;
  if (base >= N) return;
  const uint64_t d0 = offset + (uint64_t)base;
  const uint64_t b0 = d0 >> 2;
  U64x4 v{0, 0, 0, 0};
  if (lane < 9) v = philox_block(k0, k1, b0 + (uint64_t)lane);
  const uint64_t dd = d0 + (uint64_t)lane;
  const int src = (int)((dd >> 2) - b0);
  const uint64_t w0 = __shfl_sync(FULL, v.w0, src), w1 = __shfl_sync(FULL, v.w1, src);
  const uint64_t w2 = __shfl_sync(FULL, v.w2, src), w3 = __shfl_sync(FULL, v.w3, src);
  const int wi = (int)(dd & 3);
  const uint64_t raw = wi == 0 ? w0 : (wi == 1 ? w1 : (wi == 2 ? w2 : w3));
  const int64_t i = base + lane;
  if (i < N) out[i] = index_lower_bound(W, idx, d, load_aux(idx ? idx + d.aoff : nullptr), u01(raw));
}

// -------------------------------------------------------- K5 merge stream ----
// #(U[i] <= key) for sorted U, by a warp: 32-ary narrowing then one final probe.
__device__ __forceinline__ int64_t warp_count_le(const double* __restrict__ U, int64_t N, double key) {
  const int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = N;  // answer in [lo, hi]
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

// #(a[i] <= key) for sorted a[0..n) in shared memory, by a warp
__device__ __forceinline__ int warp_count_le_smem(const double* a, int n, double key) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = n;
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) / 32;
    const int p = lo + (lane + 1) * step - 1;
    const int cnt = __popc(__ballot_sync(FULL, p < hi && a[p] <= key));
    const int nhi = lo + (cnt + 1) * step - 1;
    lo += cnt * step;
    hi = nhi < hi ? nhi : hi;
  }
  return lo + __popc(__ballot_sync(FULL, lo + lane < hi && a[lo + lane] <= key));
}

// The streaming merge (CCF, and DaC in merge mode).  One CTA per W tile of
// `tw` entries (4096 at M >> N, smaller when the table is small so that every
// SM holds several tiles): the tile arrives by one TMA bulk copy while two
// warps find the tile's u-run [#(u <= W[j0-1]), #(u <= W[j0+len-1])) by
// warp-cooperative 32-ary searches of U.  Several CTAs per SM keep HBM busy
// (a probe of persistent TMA rings measured no better; profiles/r1_s3).
// In the tile: a short u-run (M >> N) gets one shared-memory bisection per u;
// a long one (M ~ N) is staged in shared memory and merged with the tile by
// merge path -- every thread takes an equal diagonal segment, locates its
// start by bisection and merges branch-free, taking W before u only when
// W < u, so each u gets the first j with W[j] >= u.
// first p in [0, n) with a[p] >= x, clamped to n-1 (the reference's bisection)
__device__ __forceinline__ int smem_lower_bound(const double* a, int n, double x) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (a[m] < x) lo = m + 1;
    else hi = m;
  }
  return lo;
}

// a staged W tile sw[0..len) of entries j0.. of a deferred table -> W itself:
// S = C_g + (D_t + L), W = min(S / T, 1) (the division by the shared T as a
// multiply and two FMAs, div_rn), W[M-1] = 1.  The pair is re-read per entry
// from L1 (holding both in registers costs k_merge_tiles its eighth CTA per SM).
__device__ __forceinline__ void stage_to_w(double* sw, int len, int64_t j0, int64_t M, const TabAux& ta) {
  const double2* P = ta.P + j0 / TABLE_TILE;
  const int jb = (int)((j0 / TABLE_TILE + 1) * TABLE_TILE - j0);
  const int il = (M - 1 - j0 < (int64_t)len) ? (int)(M - 1 - j0) : -1;  // the pinned last entry, if in this tile
  const DivBy byT = div_by(ta.T);
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    const double2 cd = __ldg(P + (i < jb ? 0 : 1));
    sw[i] = (i == il && ta.pin) ? 1.0 : fmin(div_rn(tab_sum(ta, cd, sw[i]), byT), 1.0);
  }
}

// W[j] at the end of a 16-entry block (j = 16 m + 15, or M - 1): a direct
// table's value itself (often already in L2: the neighbouring tile's copy);
// for a deferred table level 1 of the index, which holds W there -- or
// (TAB_L1) the in-tile value, turned into W with the tile pair.  The value
// and the header are loaded together; only a deferred table pays the second
// round trip.  A table without an index is direct.
__device__ __forceinline__ double block_end_w(const double* __restrict__ W, const double* __restrict__ idx,
                                              const double* __restrict__ aux, int64_t M, int64_t j) {
  const double v = __ldg(W + j);
  if (!aux) return v;
  const double2 h = __ldg(reinterpret_cast<const double2*>(aux));
  const int mode = (int)h.y;
  if (mode == 0) return v;
  const double l1v = __ldg(idx + j / FANOUT);  // level 1 sits at offset 0 (a deferred table has M > 16 here or idx)
  if (!(mode & TAB_L1)) return (M > FANOUT) ? l1v : tab_w(load_aux(aux), __ldg(reinterpret_cast<const double2*>(aux + TAB_HDR) + j / TABLE_TILE), v, j == M - 1);
  const TabAux ta = load_aux(aux);
  return tab_w(ta, __ldg(ta.P + j / TABLE_TILE), l1v, j == M - 1);
}

constexpr int MT_THREADS = 256;
constexpr int MT_TW = 4096;   // max W entries per tile (32 KB)
constexpr int MT_TW3 = 3072;  // tiles of large tables with few u's each (24 KB: eight CTAs per SM)
constexpr int MT_UC = 1024;   // u's staged per merge-path chunk (8 KB)
constexpr int MT_HEAVY = 4 * MT_UC;  // a tile's u-run longer than this is spread over k_merge_heavy

__global__ void __launch_bounds__(MT_THREADS, 8) k_merge_tiles(const double* __restrict__ W, int64_t M,
                                                            const double* __restrict__ idx,
                                                            const double* __restrict__ aux,
                                                            const double* __restrict__ U, int64_t N,
                                                            int64_t* __restrict__ out, int tw, int paths) {
  extern __shared__ __align__(128) double msm[];
  double* sw = msm;            // [tw]
  double* su = msm + tw;       // [MT_UC]
  int64_t* so = (int64_t*)(su + MT_UC);  // [MT_UC] results, written out coalesced
  __shared__ __align__(8) uint64_t bar;
  __shared__ int64_t s_ib, s_ie;
  __shared__ int s_w0, s_w1;
  __shared__ double2 s_hdr, s_hdr2;  // the table header {T, mode}, {O, pin}, read beside the u-run searches
  __shared__ double2 s_pair[2];  // a deferred table's tile pairs around j0
  __shared__ int s_probe;        // deferred, few u's: W formed at each bisection probe
  const int64_t t = blockIdx.x;
  const int64_t j0 = t * tw;
  const int len = (int)((M - j0) < tw ? (M - j0) : tw);
  const bool last = (j0 + len == M);
  const int len_even = len & ~1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  STAMPK(4, 0);
  pdl_wait();
  STAMPK(4, 1);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, (uint32_t)len_even * 8u);
    if (len_even > 0) bulk_g2s(sw, W + j0, (uint32_t)len_even * 8u, &bar);
  }
  if (threadIdx.x == 64 && (len & 1)) sw[len - 1] = W[j0 + len - 1];
  if (threadIdx.x == 96) {
    // the table header and, for a deferred table, its tile pairs around j0:
    // loaded beside the u-run searches (a direct table loads the header only)
    const double2 h = aux ? __ldg(reinterpret_cast<const double2*>(aux)) : make_double2(1.0, 0.0);
    s_hdr = h;
    s_hdr2 = aux ? __ldg(reinterpret_cast<const double2*>(aux) + 1) : make_double2(0.0, 1.0);
    s_probe = 0;
    if (h.y != 0.0) {
      const double2* P = reinterpret_cast<const double2*>(aux + TAB_HDR);
      const int64_t t0 = j0 / TABLE_TILE, tl = table_tiles(M) - 1;
      s_pair[0] = __ldg(P + t0);
      s_pair[1] = __ldg(P + (t0 + 1 < tl ? t0 + 1 : tl));
    }
  }
  if (warp == 0) {  // tile edges are block ends (tw is a multiple of 16): level 1 holds W there
    const int64_t v = (t == 0) ? 0 : warp_count_le(U, N, block_end_w(W, idx, aux, M, j0 - 1));
    if (lane == 0) s_ib = v;
  } else if (warp == 1) {
    const int64_t v = last ? N : warp_count_le(U, N, block_end_w(W, idx, aux, M, j0 + len - 1));
    if (lane == 0) s_ie = v;
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  const int64_t ib = s_ib, ie = s_ie;
  // a deferred table: a tile holding many u's becomes W once (a multiply and
  // two FMAs per entry); one holding few (M >> N) forms W at each probe
  if (s_hdr.y != 0.0) {
    if (16 * (ie - ib) > (int64_t)len) stage_to_w(sw, len, j0, M, load_aux(aux));
    else if (threadIdx.x == 0) s_probe = 1;
    __syncthreads();
  }
  STAMPK(4, 2);
  // a long run: the whole MT_UC-chunks inside it are left to k_merge_heavy
  // (many CTAs), each marked in out[] by the first slot of the chunk holding
  // -1 - t; this CTA keeps the ragged ends [ib, sk0) and [sk1, ie)
  int64_t sk0 = ie, sk1 = ie;
  if (ie - ib > MT_HEAVY) {
    sk0 = (ib + MT_UC - 1) / MT_UC * MT_UC;
    sk1 = ie / MT_UC * MT_UC;
    for (int64_t k = sk0 / MT_UC + threadIdx.x; k < sk1 / MT_UC; k += MT_THREADS) out[k * MT_UC] = -1 - t;
  }
  // short u-runs (or no room for a u chunk: paths == 0): a bisection per u
  if (!paths || ie - ib <= 2 * MT_THREADS) {
    if (s_probe) {  // a deferred table, few u's: W formed at each probe (CTA-uniform branch)
      const int jb = (int)((j0 / TABLE_TILE + 1) * TABLE_TILE - j0);
      const bool shard = ((int)s_hdr.y & TAB_SHARD) != 0, pin = s_hdr2.y != 0.0;
      for (int seg = 0; seg < 2; ++seg) {
        const int64_t r0 = seg ? sk1 : ib, r1 = seg ? ie : sk0;
        for (int64_t i = r0 + threadIdx.x; i < r1; i += MT_THREADS) {
          const double x = __ldg(U + i);
          int lo = 0, hi = len - 1;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const double2 cd = s_pair[mid < jb ? 0 : 1];
            double S = __dadd_rn(cd.x, __dadd_rn(cd.y, sw[mid]));
            if (shard) S = __dadd_rn(s_hdr2.x, S);  // a shard of a W-sharded table
            const double v = (j0 + mid == M - 1 && pin) ? 1.0 : fmin(__ddiv_rn(S, s_hdr.x), 1.0);
            if (v < x) lo = mid + 1;
            else hi = mid;
          }
          out[i] = j0 + lo;
        }
      }
    } else {
      for (int seg = 0; seg < 2; ++seg) {
        const int64_t r0 = seg ? sk1 : ib, r1 = seg ? ie : sk0;
        for (int64_t i = r0 + threadIdx.x; i < r1; i += MT_THREADS) {
          const double x = __ldg(U + i);
          int lo = 0, hi = len - 1;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sw[mid] < x) lo = mid + 1;
            else hi = mid;
          }
          out[i] = j0 + lo;
        }
      }
    }
    pdl_trigger();
    STAMPK(4, 3);
    return;
  }
  for (int seg = 0; seg < 2; ++seg) {
  const int64_t r0 = seg ? sk1 : ib, r1 = seg ? ie : sk0;
  for (int64_t c0 = r0; c0 < r1; c0 += MT_UC) {
    const int c = (int)((r1 - c0) < MT_UC ? (r1 - c0) : MT_UC);
    for (int i = threadIdx.x; i < c; i += MT_THREADS) su[i] = __ldg(U + c0 + i);  // (a deferred tile is W here)
    __syncthreads();
    // the chunk's u's land in sw[wa0 .. wa1] (wa0 = lower bound of its first
    // u, wa1 of its last): merge only that part of the tile
    if (threadIdx.x < 2) {
      const int v = smem_lower_bound(sw, len, su[threadIdx.x == 0 ? 0 : c - 1]);
      if (threadIdx.x == 0) s_w0 = v;
      else s_w1 = v;
    }
    __syncthreads();
    const int wa0 = s_w0;
    const int wl = s_w1 - wa0 + 1;  // W entries in the merge
    const double* sws = sw + wa0;
    const int total = wl + c;
    const int per = (total + MT_THREADS - 1) / MT_THREADS;
    const int d0 = min(total, (int)threadIdx.x * per), d1 = min(total, d0 + per);
    int lo = max(0, d0 - c), hi = min(d0, wl);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sws[mid] < su[d0 - mid - 1]) lo = mid + 1;
      else hi = mid;
    }
    int ia = lo, ibb = d0 - lo;
    for (int d = d0; d < d1; ++d) {
      const double wa = (ia < wl) ? sws[ia] : dinf();
      const double xb = (ibb < c) ? su[ibb] : dinf();
      if (ibb >= c || (ia < wl && wa < xb)) {
        ++ia;
      } else {
        so[ibb] = j0 + wa0 + (ia < wl ? ia : wl - 1);  // clamp (u > 1 only without check)
        ++ibb;
      }
    }
    __syncthreads();
    // coalesced (the destination may be pinned host memory written over the link)
    for (int i = threadIdx.x; i < c; i += MT_THREADS) out[c0 + i] = so[i];
    __syncthreads();  // su / so reuse
  }
  }
  // late (an early trigger: c2 45.0 us against 43.0): k_merge_heavy's CTAs
  // would take the slots of the last tiles
  pdl_trigger();
  STAMPK(4, 3);
}

// The whole u-chunks of long runs (marked by k_merge_tiles): persistent CTAs
// stride over the chunks, skip unmarked ones (one load), stage the marked
// chunk's W tile by TMA (kept while consecutive chunks share it) and bisect.
__global__ void __launch_bounds__(MT_THREADS) k_merge_heavy(const double* __restrict__ W, int64_t M,
                                                            const double* __restrict__ aux,
                                                            const double* __restrict__ U, int64_t N,
                                                            int64_t* __restrict__ out, int tw) {
  extern __shared__ __align__(128) double hsw[];  // [tw]
  __shared__ __align__(8) uint64_t bar;
  STAMPK(5, 0);
  pdl_wait();
  STAMPK(5, 1);
  pdl_trigger();
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  const TabAux ta = load_aux(aux);
  __shared__ int64_t s_mark[MT_THREADS];
  uint32_t phase = 0;
  int64_t cur = -1;
  int len = 0;
  const int64_t nch = N / MT_UC;
  // the CTA's chunks are blockIdx.x + q * gridDim.x; their markers are read
  // MT_THREADS at a time (one load per thread), then the marked ones processed
  for (int64_t kb = blockIdx.x; kb < nch; kb += (int64_t)gridDim.x * MT_THREADS) {
    const int64_t kk = kb + (int64_t)threadIdx.x * gridDim.x;
    s_mark[threadIdx.x] = (kk < nch) ? out[kk * MT_UC] : 0;
    __syncthreads();
    for (int q = 0; q < MT_THREADS; ++q) {
      const int64_t k = kb + (int64_t)q * gridDim.x;
      if (k >= nch) break;
      const int64_t m = s_mark[q];
      if (m >= 0) continue;
      const int64_t t = -1 - m;
      const int64_t j0 = t * tw;
      if (t != cur) {
        len = (int)((M - j0) < tw ? (M - j0) : tw);
        const int len_even = len & ~1;
        if (threadIdx.x == 0) {
          mbar_expect_tx(&bar, (uint32_t)len_even * 8u);
          if (len_even > 0) bulk_g2s(hsw, W + j0, (uint32_t)len_even * 8u, &bar);
        }
        if (threadIdx.x == 64 && (len & 1)) hsw[len - 1] = W[j0 + len - 1];
        mbar_wait(&bar, phase);
        phase ^= 1u;
        __syncthreads();
        if (ta.def) {  // a heavy tile serves >= 1024 u's: W itself
          stage_to_w(hsw, len, j0, M, ta);
          __syncthreads();
        }
        cur = t;
      }
      for (int64_t i = k * MT_UC + threadIdx.x; i < (k + 1) * MT_UC; i += MT_THREADS) {
        const double x = __ldg(U + i);
        int lo = 0, hi = len - 1;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (hsw[mid] < x) lo = mid + 1;
          else hi = mid;
        }
        out[i] = j0 + lo;
      }
      __syncthreads();  // hsw reuse
    }
    __syncthreads();  // s_mark reuse
  }
  STAMPK(5, 3);
}

// -------------------------------------------------------------- checks ----
__global__ void k_check_sorted_open(const double* __restrict__ U, int64_t N, int32_t* status) {
  int bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
    if (i == 0 && (U[0] <= 0.0 || U[N - 1] > 1.0)) bad |= DRS_ST_OUT_OF_SUPPORT;
    if (i > 0 && !(__dsub_rn(U[i], U[i - 1]) > 0.0)) bad |= DRS_ST_NOT_SORTED;
  }
  bad = __reduce_or_sync(FULL, bad);
  if (bad && (threadIdx.x & 31) == 0) atomicOr(status, bad);
}

__global__ void k_validate_table(const double* __restrict__ W, int64_t M, int32_t* status) {
  int bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += stride) {
    const double v = W[i];
    if (!(v > -dinf() && v < dinf())) bad |= DRS_ST_NONFINITE;
    if (i == 0 && v < 0.0) bad |= DRS_ST_DECREASING;
    if (i > 0 && __dsub_rn(v, W[i - 1]) < 0.0) bad |= DRS_ST_DECREASING;
    if (i == M - 1 && v != 1.0) bad |= DRS_ST_TOP_NOT_ONE;
  }
  bad = __reduce_or_sync(FULL, bad);
  if (bad && (threadIdx.x & 31) == 0) atomicOr(status, bad);
}

__global__ void k_build_index(const double* __restrict__ W, int64_t M, double* __restrict__ idx,
                              IndexDesc d, int64_t total) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  int k = d.levels;
  while (k > 1 && e < d.off[k]) --k;
  const int64_t b = e - d.off[k];
  int64_t span = 1;
  for (int q = 0; q < k; ++q) span *= FANOUT;
  double v = dinf();
  if (b < d.n[k]) {
    int64_t j = (b + 1) * span - 1;
    if (j > M - 1) j = M - 1;
    v = W[j];
  }
  idx[e] = v;
}

// upper_bound_search (cdf.py:92-126): bisection with the reference's probe count
__global__ void k_lower_bound_range(const double* __restrict__ W, int64_t lo, int64_t hi, double x,
                                    int64_t* out) {
  int64_t a = lo, b = hi, probes = 0;
  while (a != b) {
    const int64_t m = (a + b) / 2;
    ++probes;
    if (W[m] < x) a = m + 1;
    else b = m;
  }
  out[0] = a;
  out[1] = probes;
}

int launch_merge(const double* W, const double* idx, int64_t M, const double* U, int64_t N, int64_t* out,
                 cudaStream_t st) {
  const double* aux = idx ? idx + make_index_desc(M).aoff : nullptr;
  static SmemLimit lim;
  lim.raise((const void*)k_merge_tiles, (MT_TW + 2 * MT_UC) * sizeof(double));
  const int sms = drs_sm_count();
  // tiles of up to 4096 entries; smaller for small tables so that every SM
  // gets >= ~6 tiles to overlap
  int tw = MT_TW;  // 8192 / 16384: c3 ccf 105.8 / 118.3 us against 104.8
  // from ~512 u's per 4096-entry tile a CTA's serial work (a u load and a
  // bisection per u, 256 at a time) outweighs its fixed cost (the two u-run
  // searches): half-size tiles (N = M = 2^22: 151 -> 113 us, 2^24: 497 -> 378 us;
  // profiles/r2/merge_paths/tile_width_sweep.txt)
  if ((double)N * MT_TW >= 512.0 * (double)M) tw = MT_TW / 2;
  // few u's per tile (M >> N) and a large table: 24 KB tiles, so that eight CTAs (not seven) fit an SM and
  // more u-run searches are in flight -- c5 ccf 2.09 -> 1.88 ms, M = 2^26 N = 2^20 145 -> 133 us, c3 ccf
  // unchanged; 2560 / 2816 / 3328 / 3584 measured too (tile_width_sweep.txt: not monotone, 3072 the best)
  // (with fewer than ~16 u's per tile the searches are few and the 32 KB tiles stream best: c3, ncu 85 vs 90 us)
  else if ((double)N * MT_TW >= 16.0 * (double)M && cdiv(M, MT_TW3) >= 6 * (int64_t)sms) tw = MT_TW3;
  while (tw > 256 && cdiv(M, tw) < 6 * (int64_t)sms) tw >>= 1;
  if (const char* f = getenv("DRS_MERGE_TW")) tw = atoi(f);  // sweeps only (a power of two in [256, 4096])
  // the CTA is its W tile alone (no u chunk: more tiles in flight per SM) and
  // every u bisects the staged tile;
  // measured (scripts/paths_ab.py, profiles/r2/merge_paths/): the per-u bisection of the staged tile is
  // never slower than the linear merge path, whatever the u's per tile (N = M included: no u chunk to
  // stage, no barriers, more CTAs per SM), so the merge path runs only when DRS_MERGE_PATHS_MIN (average
  // u's per tile from which it is used) asks for it
  const char* pm = getenv("DRS_MERGE_PATHS_MIN");
  const int paths = pm && (double)N * tw >= atof(pm) * (double)M ? 1 : 0;
  const size_t smem = (size_t)(tw + (paths ? 2 * MT_UC : 0)) * sizeof(double);
  launch_pdl(k_merge_tiles, dim3((unsigned)cdiv(M, tw)), dim3(MT_THREADS), smem, st, W, M, idx, aux, U, N, out, tw,
             paths);
  if (N > MT_HEAVY) {  // a run can be long: the helper grid (it exits after one load per chunk otherwise)
    static SmemLimit hl;
    hl.raise((const void*)k_merge_heavy, (size_t)MT_TW * sizeof(double));
    const int64_t nch = N / MT_UC;
    const unsigned g = (unsigned)(nch < 2 * (int64_t)sms ? nch : 2 * (int64_t)sms);
    launch_pdl(k_merge_heavy, dim3(g), dim3(MT_THREADS), (size_t)tw * sizeof(double), st, W, M, aux, U, N, out, tw);
  }
  return launch_rc();
}

// the top guide (drs_common.cuh) from the finished level kt: level kt
// (<= 16384 entries, L2-resident) staged in shared memory by one TMA bulk copy
// per CTA, then one thread per bucket bisects it there (a 14-step chain of
// shared-memory reads instead of L2 round trips); the storage tail past
// bucket B + 1 is zeroed
__global__ void __launch_bounds__(256) k_build_top_guide(double* __restrict__ idx, IndexDesc d) {
  extern __shared__ __align__(128) double sL[];
  __shared__ __align__(8) uint64_t bar;
  STAMPK(6, 0);
  pdl_wait();
  STAMPK(6, 1);
  pdl_trigger();
  const int64_t nk = d.n[d.kt];
  const uint32_t bytes = (uint32_t)(cdiv(nk, FANOUT) * FANOUT * 8);  // the level is padded to whole nodes
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, bytes);
    bulk_g2s(sL, idx + d.off[d.kt], bytes, &bar);
  }
  __syncthreads();
  int32_t* G = reinterpret_cast<int32_t*>(idx + d.toff);
  const int64_t cap = 2 * tg_doubles(d), nb = ((int64_t)1 << d.tshift) + 2;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  mbar_wait(&bar, 0);
  if (b >= cap) return;
  if (b >= nb) {
    G[b] = 0;
    return;
  }
  const double x = (double)b / (double)((int64_t)1 << d.tshift);  // exact
  int lo = 0, hi = (int)nk - 1;
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (sL[m] < x) lo = m + 1;
    else hi = m;
  }
  G[b] = (int32_t)lo;
  STAMPK(6, 3);
}

int launch_top_guide(int64_t M, double* idx, cudaStream_t st) {
  const IndexDesc d = make_index_desc(M);
  if (!d.kt) return DRS_OK;
  static SmemLimit lim;
  const size_t smem = (size_t)cdiv(d.n[d.kt], FANOUT) * FANOUT * 8;
  lim.raise((const void*)k_build_top_guide, (size_t)(DRS_TG_ENTRIES + FANOUT) * 8);
  launch_pdl(k_build_top_guide, dim3((unsigned)cdiv(2 * tg_doubles(d), 256)), dim3(256), smem, st, idx, d);
  return launch_rc();
}

// the header and tile pairs of a direct table, all zero (deferred = 0:
// searches compare W itself)
int write_direct_header(double* idx, int64_t M, cudaStream_t st) {
  if (!idx) return DRS_OK;
  const IndexDesc d = make_index_desc(M);
  const size_t bytes = (size_t)(TAB_HDR + 2 * table_tiles(M)) * sizeof(double);
  return cudaMemsetAsync(idx + d.aoff, 0, bytes, st) == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

int launch_build_index(const double* W, int64_t M, double* idx, cudaStream_t st) {
  const IndexDesc d = make_index_desc(M);
  if (write_direct_header(idx, M, st)) return DRS_ERR_LAUNCH;
  if (d.levels == 0) return DRS_OK;
  if (!idx) return DRS_ERR_ARG;
  const int64_t total = d.off[d.levels] + cdiv(d.n[d.levels], FANOUT) * FANOUT;
  k_build_index<<<(unsigned)cdiv(total, 256), 256, 0, st>>>(W, M, idx, d, total);
  if (launch_rc()) return DRS_ERR_LAUNCH;
  return launch_top_guide(M, idx, st);
}

int launch_index_sm(const double* W, const double* idx, int64_t M, const double* u, int64_t N, int64_t* out,
                    cudaStream_t st, const int64_t* rng = nullptr, int64_t shift = 0);  // drs_fused.cu

int launch_index(const double* W, const double* idx, int64_t M, const double* u, int64_t N,
                        int64_t* out, cudaStream_t st) {
  const IndexDesc d = make_index_desc(M);
  if (d.levels > 0) return launch_index_sm(W, idx, M, u, N, out, st);
  k_match_index<<<(unsigned)cdiv(N, 256), 256, 0, st>>>(W, idx, d, u, N, out);
  return launch_rc();
}

}  // namespace drs

using namespace drs;

extern "C" {

#ifdef DRS_PHASE_TIMING
int dr_debug_phase_times_match(unsigned long long* host, int n) {
  return cudaMemcpyFromSymbol(host, g_phase, sizeof(unsigned long long) * (size_t)n) == cudaSuccess ? 0 : -1;
}
int dr_debug_phase_clear_match(void) {
  void* p = nullptr;
  if (cudaGetSymbolAddress(&p, g_phase) != cudaSuccess) return -1;
  return cudaMemset(p, 0, sizeof(g_phase)) == cudaSuccess ? 0 : -1;
}
#endif

int dr_validate_table(const double* W, int64_t M, int32_t* status, void* stream) {
  if (M < 1 || !W || !status) return DRS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(status, 0, sizeof(int32_t), st) != cudaSuccess) return DRS_ERR_LAUNCH;
  const int64_t blocks = cdiv(M, 256) < 148 * 8 ? cdiv(M, 256) : 148 * 8;
  k_validate_table<<<(unsigned)blocks, 256, 0, st>>>(W, M, status);
  return launch_rc();
}

int dr_build_index(const double* W, int64_t M, double* idx, void* stream) {
  if (M < 1 || !W) return DRS_ERR_ARG;
  return launch_build_index(W, M, idx, (cudaStream_t)stream);
}

int dr_match_binary(const double* W, const double* idx, int64_t M, const double* u, int64_t N,
                    int64_t* out, void* stream) {
  if (M < 1 || N < 0 || !W || (N > 0 && (!u || !out))) return DRS_ERR_ARG;
  if ((uintptr_t)W & 31) return DRS_ERR_ALIGN;
  if (N == 0) return DRS_OK;
  if (make_index_desc(M).levels > 0 && !idx) return DRS_ERR_ARG;
  return launch_index(W, idx, M, u, N, out, (cudaStream_t)stream);
}

int dr_sample_binary(const double* W, const double* idx, int64_t M, uint64_t k0, uint64_t k1,
                     uint64_t offset, int64_t N, int64_t* out, void* stream) {
  if (M < 1 || N < 0 || !W || (N > 0 && !out)) return DRS_ERR_ARG;
  if ((uintptr_t)W & 31) return DRS_ERR_ALIGN;
  if (N == 0) return DRS_OK;
  const IndexDesc d = make_index_desc(M);
  if (d.levels > 0 && !idx) return DRS_ERR_ARG;
  k_sample_binary<<<(unsigned)cdiv(N, 256), 256, 0, (cudaStream_t)stream>>>(W, idx, d, k0, k1,
                                                                           offset, N, out);
  return launch_rc();
}

int dr_match_ccf(const double* W, const double* idx, int64_t M, const double* U, int64_t N, int64_t* out,
                 void* stream) {
  if (M < 1 || N < 0 || !W || (N > 0 && (!U || !out))) return DRS_ERR_ARG;
  if ((uintptr_t)W & 15) return DRS_ERR_ALIGN;
  if (N == 0) return DRS_OK;
  return launch_merge(W, idx, M, U, N, out, (cudaStream_t)stream);
}

int dr_match_dac(const double* W, const double* idx, int64_t M, const double* U, int64_t N,
                 int64_t* out, int32_t mode, void* stream) {
  if (M < 1 || N < 0 || !W || (N > 0 && (!U || !out))) return DRS_ERR_ARG;
  if (mode != DRS_DAC_AUTO && mode != DRS_DAC_MERGE && mode != DRS_DAC_SEARCH) return DRS_ERR_MODE;
  if ((uintptr_t)W & 31) return DRS_ERR_ALIGN;
  if (N == 0) return DRS_OK;
  bool merge = (mode == DRS_DAC_MERGE) || (mode == DRS_DAC_AUTO && M <= DAC_TAU * N);
  if (!merge && make_index_desc(M).levels > 0 && !idx) merge = true;
  cudaStream_t st = (cudaStream_t)stream;
  if (merge) return launch_merge(W, idx, M, U, N, out, st);
  return launch_index(W, idx, M, U, N, out, st);
}

int dr_check_sorted_open(const double* U, int64_t N, int32_t* status, void* stream) {
  if (N < 0 || !status || (N > 0 && !U)) return DRS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(status, 0, sizeof(int32_t), st) != cudaSuccess) return DRS_ERR_LAUNCH;
  if (N == 0) return DRS_OK;
  const int64_t blocks = cdiv(N, 256) < 148 * 8 ? cdiv(N, 256) : 148 * 8;
  k_check_sorted_open<<<(unsigned)blocks, 256, 0, st>>>(U, N, status);
  return launch_rc();
}

int dr_lower_bound_range(const double* W, int64_t lo, int64_t hi, double x, int64_t* out,
                         void* stream) {
  if (!W || !out || lo < 0 || hi < lo) return DRS_ERR_ARG;
  k_lower_bound_range<<<1, 1, 0, (cudaStream_t)stream>>>(W, lo, hi, x, out);
  return launch_rc();
}

}  // extern "C"
