// drs_fused.cu -- dac_sampler / binary_sampler as ONE kernel launch (sm_100a).
//
// dac_sampler (samplers.py:262-266) = sorted_uniforms (randkit.py:70-101)
// followed by dac_match (samplers.py:191-210).  For N+1 <= (co-resident
// CTAs) * 1024 the whole call is one cooperative launch:
//
//   1. thread 0 TMA-prefetches the top levels of the table's search index
//      (a contiguous suffix of idx, <= 64 KB) into shared memory;
//   2. every thread draws its 4 Philox uniforms, z = -log u, and the CTA
//      forms its tile of the chained scan (identical association to
//      dr_sorted_uniforms, so U is bit-identical to the two-pass path);
//   3. one grid barrier; each CTA folds the tile totals before it (the same
//      left fold the look-back computes) and the spacing minimum;
//   4. U = Z / Z[n] in registers; the rare collapse repair runs behind two
//      more grid barriers only when the reference's exactness check fires;
//   5. each thread searches its 4 sorted u's: the top index levels from
//      shared memory, the lower ones as one 128-byte line (4 x 256-bit
//      loads) per level, W last -- O(N log_16 M) lines instead of 8M bytes;
//   6. indices (and optionally U) are written coalesced.
// The stream position may live in device memory (offset_dev) and is then
// advanced on the device, so the launch can be captured in a CUDA graph
// and replayed with fresh draws each time.
#include <algorithm>
#include <cooperative_groups.h>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "drs_common.cuh"

namespace drs {

IndexDesc make_index_desc(int64_t M);
int64_t ws_capacity_tiles(size_t ws_bytes);
ScanWS carve_ws(void* ws, size_t ws_bytes);
int sorted_uniforms_launch(uint64_t k0, uint64_t k1, uint64_t offset, const uint64_t* offset_dev,
                           int64_t n, double* U, int32_t* status, void* ws, size_t ws_bytes,
                           cudaStream_t st);
int launch_merge(const double* W, const double* idx, int64_t M, const double* U, int64_t N, int64_t* out,
                 cudaStream_t st);
int launch_index(const double* W, const double* idx, int64_t M, const double* u, int64_t N,
                 int64_t* out, cudaStream_t st);

constexpr int SIDX_CAP = 24576;
constexpr int FUSED_MAX_TILES = 1024;  // 32 lanes x GROUP_TILES; the launch also needs co-residency
#ifndef DRS_L2_PREFETCH_MB
#define DRS_L2_PREFETCH_MB 4
#endif
// the first global index level below the shared-memory levels (2 MB at
// M = 2^26) is prefetched into L2 while the uniforms are formed; the larger
// levels and W are reached at random and are left to the searches
constexpr int64_t L2_PREFETCH_DOUBLES = (int64_t)DRS_L2_PREFETCH_MB << 17;
constexpr int64_t TS_U = (int64_t)THREADS * K_UNIF;

struct SmemLevels {
  int k_smem;       // levels k >= k_smem are staged in shared memory (k_smem > levels: none)
  int64_t base;     // idx offset of level k_smem
  int64_t count;    // doubles staged
  int tg;           // the top guide is staged too (k_smem == kt): the search enters at level kt
  int64_t hdr;      // offset in the stage of the table header (it follows the guide), -1: not staged
};

SmemLevels plan_smem_levels(const IndexDesc& d, int64_t cap = SIDX_CAP) {
  SmemLevels s{d.levels + 1, 0, 0, 0, -1};
  if (d.levels == 0) return s;
  if (d.kt) {  // level kt, the levels above it, the top guide and the table header: one contiguous range
    const int64_t need = d.toff + tg_doubles(d) - d.off[d.kt];
    if (need + TAB_HDR <= cap) return SmemLevels{d.kt, d.off[d.kt], need + TAB_HDR, 1, d.aoff - d.off[d.kt]};
  }
  const int64_t end = d.off[d.levels] + cdiv(d.n[d.levels], FANOUT) * FANOUT;
  for (int k = d.levels; k >= 1; --k) {
    if (end - d.off[k] > cap) break;
    s.k_smem = k;
    s.base = d.off[k];
    s.count = end - d.off[k];
  }
  return s;
}

__device__ __forceinline__ int count_lt16_smem(const double* p, double x) {
  int c = 0;
#pragma unroll
  for (int i = 0; i < 16; i += 2) {
    const double2 v = *reinterpret_cast<const double2*>(p + i);
    c += (v.x < x) ? 1 : 0;
    c += (v.y < x) ? 1 : 0;
  }
  return c;
}

// K_UNIF independent searches in lock-step: the level loop is outside, so the
// lines of a level are in flight together
template <bool DEF>
__device__ __forceinline__ void search_k_sm_impl(const double* __restrict__ W, const double* __restrict__ idx,
                                            const double* sidx, const IndexDesc& d, const SmemLevels& sl,
                                            const TabAux& ta, const double x[K_UNIF], int64_t r[K_UNIF]) {
  int64_t b[K_UNIF];
#pragma unroll
  for (int q = 0; q < K_UNIF; ++q) b[q] = 0;
  int ktop = d.levels;
  if (sl.tg) {
    // the top guide: the level-kt node from one bucket, [Gt[b], Gt[b+1]]
    // narrowed by a bisection over level kt (in shared memory; mostly empty)
    const int32_t* Gt = reinterpret_cast<const int32_t*>(sidx + (d.toff - sl.base));
    const double* Lk = sidx + (d.off[d.kt] - sl.base);
    const int64_t B = (int64_t)1 << d.tshift;
#pragma unroll
    for (int q = 0; q < K_UNIF; ++q) {
      const double xb = x[q] * (double)B;
      const int64_t bk = (xb >= (double)B) ? B : ((xb > 0.0) ? (int64_t)xb : 0);  // NaN -> 0
      int lo = Gt[bk], hi = Gt[bk + 1];
      while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (Lk[m] < x[q]) lo = m + 1;
        else hi = m;
      }
      b[q] = lo;
    }
    ktop = d.kt - 1;
  }
  // a deferred table's tile pair and band of each u: formed at level 1 when
  // that level holds in-tile values (TAB_L1: its 256-entry node and the W
  // line below lie in one tile), else at the W line
  double2 cd[K_UNIF];
  WKey key[K_UNIF];
  bool have = false;
  for (int k = ktop; k >= 1; --k) {
    int c[K_UNIF];
    if (k >= sl.k_smem) {
      const double* base = sidx + (d.off[k] - sl.base);
#pragma unroll
      for (int q = 0; q < K_UNIF; ++q) c[q] = count_lt16_smem(base + FANOUT * b[q], x[q]);
    } else if (DEF && k == 1 && ta.l1) {
      const double* base = idx + d.off[1];
      double v1[K_UNIF][16];
#pragma unroll
      for (int q = 0; q < K_UNIF; ++q) {
        const double* p = base + FANOUT * b[q];
        ldg256(p + 0, v1[q][0], v1[q][1], v1[q][2], v1[q][3]);
        ldg256(p + 4, v1[q][4], v1[q][5], v1[q][6], v1[q][7]);
        ldg256(p + 8, v1[q][8], v1[q][9], v1[q][10], v1[q][11]);
        ldg256(p + 12, v1[q][12], v1[q][13], v1[q][14], v1[q][15]);
        cd[q] = __ldg(ta.P + b[q] / (TABLE_TILE / (FANOUT * FANOUT)));
      }
#pragma unroll
      for (int q = 0; q < K_UNIF; ++q) {
        key[q] = tab_wkey(ta, x[q]);
        c[q] = count_w16(v1[q], ta, cd[q], x[q], key[q]);
      }
      have = true;
    } else {
      const double* base = idx + d.off[k];
#pragma unroll
      for (int q = 0; q < K_UNIF; ++q) c[q] = count_lt16(base + FANOUT * b[q], x[q]);
    }
#pragma unroll
    for (int q = 0; q < K_UNIF; ++q) {
      const int64_t valid = d.n[k] - FANOUT * b[q];
      if (c[q] >= valid) c[q] = (int)valid - 1;
      b[q] = FANOUT * b[q] + c[q];
    }
  }
  // W level: the lines are loaded together (branch-free addresses; the rare
  // short tail line is re-read scalar), so the DRAM round trips overlap; a
  // deferred table's tile pairs and keys are formed while they are in flight
  double v[K_UNIF][16];
#pragma unroll
  for (int q = 0; q < K_UNIF; ++q) {
    const int64_t j0 = FANOUT * b[q];
    const double* p = (d.n[0] - j0 >= FANOUT) ? W + j0 : W;
    ldg256(p + 0, v[q][0], v[q][1], v[q][2], v[q][3]);
    ldg256(p + 4, v[q][4], v[q][5], v[q][6], v[q][7]);
    ldg256(p + 8, v[q][8], v[q][9], v[q][10], v[q][11]);
    ldg256(p + 12, v[q][12], v[q][13], v[q][14], v[q][15]);
    if (DEF && !have) cd[q] = __ldg(ta.P + j0 / TABLE_TILE);
  }
  if (DEF && !have) {
#pragma unroll
    for (int q = 0; q < K_UNIF; ++q) key[q] = tab_wkey(ta, x[q]);
  }
#pragma unroll
  for (int q = 0; q < K_UNIF; ++q) {
    const int64_t j0 = FANOUT * b[q];
    const int64_t valid = d.n[0] - j0;
    int c = 0;
    if (DEF) {
      c = (valid >= FANOUT) ? count_w16(v[q], ta, cd[q], x[q], key[q])
                            : count_w_tail(W, j0, (int)valid, ta, cd[q], x[q]);
    } else if (valid >= FANOUT) {
#pragma unroll
      for (int i = 0; i < 16; ++i) c += (v[q][i] < x[q]) ? 1 : 0;
    } else {
      for (int i = 0; i < (int)valid; ++i) c += (__ldg(W + j0 + i) < x[q]) ? 1 : 0;
    }
    if (c >= valid) c = (int)valid - 1;
    r[q] = j0 + c;
  }
}

// one search body per kind of table (the header is uniform across the
// grid): a direct table runs exactly the compare-W code, with no
// deferred-table state live in it
__device__ __forceinline__ void search_k_sm(const double* __restrict__ W, const double* __restrict__ idx,
                                            const double* sidx, const IndexDesc& d, const SmemLevels& sl,
                                            const TabAux& ta, const double x[K_UNIF], int64_t r[K_UNIF]) {
  if (ta.def) search_k_sm_impl<true>(W, idx, sidx, d, sl, ta, x, r);
  else search_k_sm_impl<false>(W, idx, sidx, d, sl, ta, x, r);
}

// The throughput variant for many u's (k_match_index_sm): KQ searches per
// thread in lock-step, and every global node is read as 72 bytes instead of
// 128 -- its entry 7 decides the half (entries 0..7 are all < x when entry 7
// is), then the half's 8 entries by two 256-bit loads.  The searches of the
// c5 shape are bound by the L1 data pipe (every lane reads its own line), so
// bytes per node, not dependent round trips, set their time.
__device__ __forceinline__ int count_lt16_half(const double* p, double x) {
  const double p7 = __ldg(p + 7);
  const bool up = p7 < x;
  const double* h = p + (up ? 8 : 0);
  double v[8];
  ldg256(h + 0, v[0], v[1], v[2], v[3]);
  ldg256(h + 4, v[4], v[5], v[6], v[7]);
  int c = up ? 8 : 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) c += (v[i] < x) ? 1 : 0;
  return c;
}

// the same on a W line of a deferred table: its values against the band of
// the line's tile (tab_lband), the exact quotient inside the band
__device__ __forceinline__ int count_w16_half(const double* p, const TabAux& ta, double2 cd, double x, const WKey& k) {
  if (!ta.def) return count_lt16_half(p, x);
  const LBand b = tab_lband(ta, k, cd);
  const bool up = tab_below(ta, cd, __ldg(p + 7), x, b);
  const double* h = p + (up ? 8 : 0);
  double v[8];
  ldg256(h + 0, v[0], v[1], v[2], v[3]);
  ldg256(h + 4, v[4], v[5], v[6], v[7]);
  int c = up ? 8 : 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) c += tab_below(ta, cd, v[i], x, b) ? 1 : 0;
  return c;
}

template <int KQ, bool DEF>
__device__ __forceinline__ void search_half_impl(const double* __restrict__ W, const double* __restrict__ idx,
                                            const double* sidx, const IndexDesc& d, const SmemLevels& sl,
                                            const TabAux& ta, const double x[KQ], int64_t r[KQ]) {
  int64_t b[KQ];
#pragma unroll
  for (int q = 0; q < KQ; ++q) b[q] = 0;
  int ktop = d.levels;
  if (sl.tg) {  // the top guide, as in search_k_sm
    const int32_t* Gt = reinterpret_cast<const int32_t*>(sidx + (d.toff - sl.base));
    const double* Lk = sidx + (d.off[d.kt] - sl.base);
    const int64_t B = (int64_t)1 << d.tshift;
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      const double xb = x[q] * (double)B;
      const int64_t bk = (xb >= (double)B) ? B : ((xb > 0.0) ? (int64_t)xb : 0);  // NaN -> 0
      int lo = Gt[bk], hi = Gt[bk + 1];
      while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (Lk[m] < x[q]) lo = m + 1;
        else hi = m;
      }
      b[q] = lo;
    }
    ktop = d.kt - 1;
  }
  double2 cd[KQ];
  WKey key[KQ];
  bool have = false;
  for (int k = ktop; k >= 1; --k) {
    int c[KQ];
    if (k >= sl.k_smem) {
      const double* base = sidx + (d.off[k] - sl.base);
#pragma unroll
      for (int q = 0; q < KQ; ++q) c[q] = count_lt16_smem(base + FANOUT * b[q], x[q]);
    } else if (DEF && k == 1 && ta.l1) {  // level 1 in-tile (its node and the W line share a tile)
      const double* base = idx + d.off[1];
#pragma unroll
      for (int q = 0; q < KQ; ++q) {
        cd[q] = __ldg(ta.P + b[q] / (TABLE_TILE / (FANOUT * FANOUT)));
        key[q] = tab_wkey(ta, x[q]);
      }
#pragma unroll
      for (int q = 0; q < KQ; ++q) c[q] = count_w16_half(base + FANOUT * b[q], ta, cd[q], x[q], key[q]);
      have = true;
    } else {
      const double* base = idx + d.off[k];  // levels are padded to whole nodes with +inf
#pragma unroll
      for (int q = 0; q < KQ; ++q) c[q] = count_lt16_half(base + FANOUT * b[q], x[q]);
    }
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      const int64_t valid = d.n[k] - FANOUT * b[q];
      if (c[q] >= valid) c[q] = (int)valid - 1;
      b[q] = FANOUT * b[q] + c[q];
    }
  }
  if (DEF && !have) {
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      cd[q] = __ldg(ta.P + FANOUT * b[q] / TABLE_TILE);
      key[q] = tab_wkey(ta, x[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < KQ; ++q) {
    const int64_t j0 = FANOUT * b[q];
    const int64_t valid = d.n[0] - j0;
    int c = 0;
    if (DEF) {
      c = (valid >= FANOUT) ? count_w16_half(W + j0, ta, cd[q], x[q], key[q])
                            : count_w_tail(W, j0, (int)valid, ta, cd[q], x[q]);
    } else if (valid >= FANOUT) {
      c = count_lt16_half(W + j0, x[q]);
    } else {
      for (int i = 0; i < (int)valid; ++i) c += (__ldg(W + j0 + i) < x[q]) ? 1 : 0;
    }
    if (c >= valid) c = (int)valid - 1;
    r[q] = j0 + c;
  }
}

template <int KQ>
__device__ __forceinline__ void search_half(const double* __restrict__ W, const double* __restrict__ idx,
                                            const double* sidx, const IndexDesc& d, const SmemLevels& sl,
                                            const TabAux& ta, const double x[KQ], int64_t r[KQ]) {
  if (ta.def) search_half_impl<KQ, true>(W, idx, sidx, d, sl, ta, x, r);
  else search_half_impl<KQ, false>(W, idx, sidx, d, sl, ta, x, r);
}

// Sense-free grid barrier for a cooperative launch (all CTAs co-resident).
__device__ __forceinline__ void grid_barrier(uint32_t* count, uint32_t* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t g = ld_acquire_u32(gen);
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *count = 0;
      __threadfence();
      st_release_u32(gen, g + 1);
    } else {
      while (ld_acquire_u32(gen) == g) __nanosleep(20);
    }
  }
  __syncthreads();
}

struct FusedArgs {
  const double* W;
  const double* idx;
  IndexDesc d;
  SmemLevels sl;
  uint64_t k0, k1, offset;
  uint64_t* offset_dev;  // optional device-resident stream position
  const double* raw;     // optional supplied uniforms (n+1) instead of Philox draws
  int64_t n;
  double* U;      // optional
  int64_t* out;
  int32_t* status;
  ScanWS ws;
  // optional: the step after resampling, fused with the index
  // writes: gout[i][0..d) = states[out[i] / divisor][0..d), states[K][d] row-major
  const double* states;
  int64_t K, gd, divisor;
  double* gout;  // null: no gather
  bool gd_vec2;  // rows as 16-byte pairs (gd even, both bases aligned)
};

// SEARCH = false: the sorted uniforms alone (a.out == nullptr: no table touched, no
// index stage).  Its own instantiation, because without the search and the gather
// it needs a quarter of the registers: four CTAs per SM are co-resident, so the
// single cooperative launch covers n + 1 <= 4 * 148 * 512 spacings.
template <bool SEARCH>
__global__ void __launch_bounds__(THREADS, SEARCH ? 1 : 4) k_dac_fused(const __grid_constant__ FusedArgs a) {
  extern __shared__ __align__(128) double sidx[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ FoldSmem fs;
  __shared__ double s_last[WARPS];
  __shared__ double s_C, s_P, s_total;
  __shared__ unsigned long long s_min;
  __shared__ uint32_t s_flag;
  __shared__ uint64_t s_words[PhiloxSpacings::SMEM_WORDS];
  __shared__ double s_agg[FUSED_MAX_TILES + FUSED_MAX_TILES / 32 + 256 + 8];  // padded tile totals
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = blockIdx.x;
  const int64_t nt = gridDim.x;
  const int64_t n = a.n;
  if (threadIdx.x == 0) STAMP1(10);  // entry
  uint32_t* bcount = &a.ws.hdr->bar_count;
  uint32_t* bgen = &a.ws.hdr->bar_gen;

  // 1. stage the top index levels in shared memory (TMA bulk copy) and
  // prefetch the next global levels into L2 (one slice per CTA): both overlap
  // steps 2-4, so the search finds them on chip instead of in HBM
  constexpr bool search = SEARCH;
  const uint32_t sbytes = search ? (uint32_t)(a.sl.count * 8) : 0u;
  if (threadIdx.x == 0) {
    s_min = 0x7FF0000000000000ULL;
    s_flag = 0;
  }
  // issued by the last warp: thread 0's release of the tile total below must
  // not queue behind these bulk transfers
  if (threadIdx.x == THREADS - 32) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, sbytes);
    if (sbytes) bulk_g2s(sidx, a.idx + a.sl.base, sbytes, &bar);
    const int64_t lvl = (search && a.sl.k_smem >= 2) ? a.sl.base - a.d.off[a.sl.k_smem - 1] : 0;  // doubles
    const int64_t cap = lvl < L2_PREFETCH_DOUBLES ? lvl : L2_PREFETCH_DOUBLES;
    const int64_t plo = a.sl.base - cap;
    const int64_t per = cdiv(cdiv(a.sl.base - plo, (int64_t)gridDim.x), 2) * 2;  // 16-byte multiples
    const int64_t p0 = plo + t * per, p1 = min(a.sl.base, p0 + per) & ~(int64_t)1;
    for (int64_t p = p0 & ~(int64_t)1; p < p1; p += 8192)  // 64 KB pieces
      prefetch_l2(a.idx + p, (uint32_t)(min((int64_t)8192, p1 - p) * 8));
  }
  const unsigned long long gen = *(volatile unsigned long long*)&a.ws.hdr->fgen;
  const uint64_t offset = a.offset_dev ? *(volatile uint64_t*)a.offset_dev : a.offset;
  __syncthreads();
  STAMP(0);

  // 2. draws, spacings, tile chain
  const int64_t e0 = t * TS_U + (int64_t)(warp * LANES + lane) * K_UNIF;
  double z[K_UNIF];
  if (a.raw) {  // uniforms supplied by a host stream
    const ArraySpacings src{a.raw};
    src.tile(t, n + 1, 0, nullptr, z);
  } else {      // each Philox block generated once, shared through shared memory
    const PhiloxSpacings src{a.k0, a.k1, offset, nullptr};
    src.tile(t, n + 1, offset, s_words, z);
  }
  STAMP(1);
  unsigned long long mn = 0x7FF0000000000000ULL;
#pragma unroll
  for (int i = 0; i < K_UNIF; ++i)
    if (e0 + i <= n) mn = min(mn, (z[i] > 0.0) ? (unsigned long long)__double_as_longlong(z[i]) : 0ull);
  double sc[K_UNIF];
  sc[0] = z[0];
#pragma unroll
  for (int i = 1; i < K_UNIF; ++i) sc[i] = __dadd_rn(sc[i - 1], z[i]);
  block_min_u64(&s_min, mn);
  double Q, R;
  const double A = block_fold(sc[K_UNIF - 1], fs, Q, R);
  STAMP(2);
  STAMP(3);
  // 3. the tile chain: every CTA publishes its total and spacing minimum and
  // bumps the arrival counter of this call's parity (cnt[gen & 1]); thread 0
  // of every CTA polls that one word until all nt tiles arrived, then warp 0
  // loads the nt totals (one coalesced round trip) and folds the chain in
  // tile order itself (D inside groups of GROUP_TILES tiles, C over the
  // groups).  CTA 0 zeroes the other parity's counter for the next call and
  // advances the generation; no grid barrier, no leader hop.
  unsigned long long* cnt = a.ws.tflag + FLAG_CAP - 2;  // two 64-bit counters, by parity
  if (threadIdx.x == 0) {
    st_relaxed_f64(&a.ws.agg[t], A);
    st_relaxed_f64(&a.ws.incl[t], __longlong_as_double((long long)s_min));
    red_release_add_u64(cnt + (gen & 1), 1ull);
    while (ld_acquire_u64(cnt + (gen & 1)) < (unsigned long long)nt) {
    }
  }
  __syncthreads();
  STAMP(9);
  if (search && threadIdx.x == THREADS - 32 && a.sl.hdr >= 0) {
    // a deferred table's tile pairs (a W line, or a level-1 node, needs its
    // tile's pair: 16 bytes per 8448 entries, 127 KB at M = 2^26) into L2, one
    // slice per CTA, while warp 0 folds the chain; the header came with the staged
    // levels (which have landed by now), so a direct table skips this
    mbar_wait(&bar, 0);
    if (sidx[a.sl.hdr + 1] != 0.0) {
      const int64_t pb = a.d.aoff + TAB_HDR, pn = 2 * table_tiles(a.d.n[0]);
      const int64_t pper = cdiv(cdiv(pn, (int64_t)gridDim.x), 2) * 2;
      const int64_t q0 = t * pper, q1 = min(pn, q0 + pper);
      for (int64_t q = q0; q < q1; q += 8192)
        prefetch_l2(a.idx + pb + q, (uint32_t)(min((int64_t)8192, q1 - q) * 8));
    }
  }
  if (warp == 0) {
    // the nt totals and minima arrive by coalesced L2 loads (.cg: no stale
    // L1 copies of the previous call's values) into shared memory, padded
    // one slot per 32 so that lane g then reads group g (tiles 32g .. 32g+31)
    // conflict-free and folds it serially; the group totals are folded in
    // group order below: a 32 + ng step chain instead of nt steps
    static_assert(GROUP_TILES == 32, "one lane per group of 32 tiles");
    unsigned long long gmin = 0x7FF0000000000000ULL;
    for (int64_t k0 = 0; k0 < nt; k0 += 8 * 32) {
      double v[8], m[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t k = k0 + q * 32 + lane;
        v[q] = (k < nt) ? __ldcg(&a.ws.agg[k]) : 0.0;
        m[q] = (k < nt) ? __ldcg(&a.ws.incl[k]) : __longlong_as_double(0x7FF0000000000000LL);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t k = k0 + q * 32 + lane;
        s_agg[k + (k >> 5)] = v[q];  // tiles past nt hold +0.0: the folds are unchanged
        gmin = min(gmin, (unsigned long long)__double_as_longlong(m[q]));
      }
    }
    __syncwarp();
    double D = 0.0, Dt = 0.0;
    const int64_t gb = (int64_t)lane * GROUP_TILES;
    if (gb < nt) {
#pragma unroll
      for (int k = 0; k < GROUP_TILES; ++k) {
        Dt = (gb + k == t) ? D : Dt;
        D = __dadd_rn(D, s_agg[gb + k + lane]);
      }
    }
    if (t == 0 && lane == 0) {
      // every CTA has read the stream position and the generation
      if (a.offset_dev) *a.offset_dev = offset + (uint64_t)(n + 1);
      cnt[(gen + 1) & 1] = 0ull;  // the next call's counter
      a.ws.hdr->fgen = gen + 1;
    }
    const int ng = (int)cdiv(nt, GROUP_TILES);
    double C = 0.0, Ct = 0.0;
    for (int g = 0; g < ng; ++g) {  // C over the group totals, in group order
      const double e = __shfl_sync(FULL, D, g);
      Ct = (g == (int)(t / GROUP_TILES)) ? C : Ct;
      C = __dadd_rn(C, e);
    }
    const double total = C;
    const double dt = __shfl_sync(FULL, Dt, (int)(t / GROUP_TILES));
    if (threadIdx.x == 0) STAMP1(13);
    for (int o = 16; o > 0; o >>= 1) gmin = min(gmin, __shfl_xor_sync(FULL, gmin, o));
    if (lane == 0) {
      s_C = Ct;
      s_P = dt;
      s_total = total;
      s_min = gmin;
    }
  }
  __syncthreads();
  const double Cg = s_C, P = s_P, total = s_total;
  const double zmin = __longlong_as_double((long long)s_min);
  const bool need = !(zmin > __dmul_rn(1e-14, total));
  STAMP(4);

  // 4. U in registers
  double u[K_UNIF];
#pragma unroll
  for (int i = 0; i < K_UNIF; ++i)
    u[i] = __ddiv_rn(__dadd_rn(Cg, __dadd_rn(P, __dadd_rn(R, __dadd_rn(Q, sc[i])))), total);

  if (need) {  // grid-uniform: the reference's exactness check (randkit.py:95-100)
    double prev_lane = __shfl_up_sync(FULL, u[K_UNIF - 1], 1);
    if (lane == 31) s_last[warp] = u[K_UNIF - 1];
    __syncthreads();
    if (lane == 0)
      prev_lane = (warp > 0) ? s_last[warp - 1] : ((t == 0) ? 0.0 : __ddiv_rn(__dadd_rn(Cg, P), total));
#pragma unroll
    for (int i = 0; i < K_UNIF; ++i) {
      const int64_t e = e0 + i;
      if (e < n) {
        const double pv = (i == 0) ? prev_lane : u[i - 1];
        if (u[i] <= pv) {
          const uint32_t slot = atomicAdd(&a.ws.hdr->nsites, 1u);
          if (slot < (uint32_t)SITE_CAP) a.ws.sites[slot] = (long long)e;
        }
        if (e == n - 1 && u[i] >= 1.0) atomicOr(&a.ws.hdr->top, 1u);
      }
      if (e < n) a.U[e] = u[i];  // U must be in memory for the repair
    }
    grid_barrier(bcount, bgen);
    const uint32_t nsites = *(volatile uint32_t*)&a.ws.hdr->nsites;
    const uint32_t top = *(volatile uint32_t*)&a.ws.hdr->top;
    if (nsites || top) {
      if (t == 0 && threadIdx.x == 0) {
        // the forward / backward nextafter passes of randkit.py:104-116,
        // restricted to the recorded collapse sites
        repair_sites(a.U, n, a.ws, nsites, true);
        s_flag = 1;
      }
      grid_barrier(bcount, bgen);
#pragma unroll
      for (int i = 0; i < K_UNIF; ++i)
        if (e0 + i < n) u[i] = ld_relaxed_f64(a.U + e0 + i);
    }
  }

  // 5. search: K_UNIF sorted u's per thread, top index levels in shared memory
  STAMP(5);
  int64_t r[K_UNIF];
#pragma unroll
  for (int i = 0; i < K_UNIF; ++i) r[i] = 0;
  if (search) {  // grid-uniform
    mbar_wait(&bar, 0);
    STAMP(6);
    // the table header arrived with the staged levels (no global round trip here)
    const TabAux ta = (a.sl.hdr >= 0) ? tab_aux_at(sidx + a.sl.hdr, a.idx + a.d.aoff)
                                      : load_aux(a.idx ? a.idx + a.d.aoff : nullptr);
    search_k_sm(a.W, a.idx, sidx, a.d, a.sl, ta, u, r);
    STAMP(7);

    // 6. write back: one 16-byte store per lane when aligned, so a warp's
    // stores cover whole lines (the destination may be pinned host memory)
    if (K_UNIF == 2 && e0 + 2 <= n && (((uintptr_t)(a.out + e0)) & 15) == 0) {
      *reinterpret_cast<longlong2*>(a.out + e0) = make_longlong2((long long)r[0], (long long)r[K_UNIF - 1]);
    } else {
#pragma unroll
      for (int i = 0; i < K_UNIF; ++i)
        if (e0 + i < n) a.out[e0 + i] = r[i];
    }
  }
  if (a.U && !need) {
    if (e0 + K_UNIF <= n && vec_ok(a.U + e0)) {
      store_k(a.U + e0, u);
    } else {
#pragma unroll
      for (int i = 0; i < K_UNIF; ++i)
        if (e0 + i < n) a.U[e0 + i] = u[i];
    }
  }
  if (search && a.gout) {
    // the resampled particle states, straight from the indices in registers
    // (lane l holds rows 2l, 2l+1 of the warp's 64).  The host checked
    // (M - 1) / divisor < K, so every row exists.
    const int64_t ew = t * TS_U + (int64_t)warp * LANES * K_UNIF;  // the warp's first draw
    const int64_t rows = n - ew < LANES * K_UNIF ? n - ew : LANES * K_UNIF;
    if (rows > 0) {
      const int64_t s0 = r[0] / a.divisor, s1 = r[K_UNIF - 1] / a.divisor;
      if (a.gd_vec2) gather_warp_rows<double2>((const double2*)a.states, a.gd / 2, s0, s1, rows,
                                               (double2*)(a.gout + ew * a.gd), lane);
      else gather_warp_rows<double>(a.states, a.gd, s0, s1, rows, a.gout + ew * a.gd, lane);
    }
  }
  __syncthreads();
  STAMP(8);
  if (t == 0 && threadIdx.x == 0) {
    // every CTA read the offset and the shared words before the last barrier
    *a.status = s_flag ? DRS_ST_REPAIRED : 0;
  }
  if (need) {
    grid_barrier(bcount, bgen);  // all reads of nsites/top done before the reset
    if (t == 0 && threadIdx.x == 0) {
      a.ws.hdr->nsites = 0;
      a.ws.hdr->top = 0;
    }
  }
}

// binary_sampler: persistent CTAs stage the top index levels in shared memory
// once (TMA) and loop over chunks of 2 x 256 draws; a warp's 32 consecutive
// draws come from <= 9 Philox blocks computed by lanes 0..8 and shuffled;
// each thread then runs its two 16-ary searches in lock-step
__device__ __forceinline__ uint64_t warp_raw_draw(uint64_t k0, uint64_t k1, uint64_t d0) {
  const int lane = threadIdx.x & 31;  // lane's draw: d0 + lane
  const uint64_t b0 = d0 >> 2;
  U64x4 v{0, 0, 0, 0};
  if (lane < 9) v = philox_block(k0, k1, b0 + (uint64_t)lane);
  const uint64_t dd = d0 + (uint64_t)lane;
  const int src = (int)((dd >> 2) - b0);
  const uint64_t w0 = __shfl_sync(FULL, v.w0, src), w1 = __shfl_sync(FULL, v.w1, src);
  const uint64_t w2 = __shfl_sync(FULL, v.w2, src), w3 = __shfl_sync(FULL, v.w3, src);
  const int wi = (int)(dd & 3);
  return wi == 0 ? w0 : (wi == 1 ? w1 : (wi == 2 ? w2 : w3));
}

__global__ void __launch_bounds__(256) k_sample_binary_sm(const double* __restrict__ W,
                                                          const double* __restrict__ idx, IndexDesc d,
                                                          SmemLevels sl, uint64_t k0, uint64_t k1,
                                                          uint64_t offset, uint64_t* offset_dev,
                                                          int64_t N, int64_t* __restrict__ out) {
  extern __shared__ __align__(128) double sidx[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t sbytes = (uint32_t)(sl.count * 8);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, sbytes);
    if (sbytes) bulk_g2s(sidx, idx + sl.base, sbytes, &bar);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t off = offset_dev ? *(volatile uint64_t*)offset_dev : offset;
  TabAux ta;
  bool staged = false;
  static_assert(K_UNIF == 2, "two draws per thread per chunk");
  for (int64_t base = (int64_t)blockIdx.x * 2 * blockDim.x; base < N; base += (int64_t)gridDim.x * 2 * blockDim.x) {
    double u[K_UNIF];
    int64_t i[K_UNIF];
#pragma unroll
    for (int h = 0; h < K_UNIF; ++h) {
      const int64_t w0 = base + h * blockDim.x + threadIdx.x - lane;  // the warp's first draw
      i[h] = w0 + lane;
      u[h] = u01(warp_raw_draw(k0, k1, off + (uint64_t)w0));
    }
    if (!staged) {
      mbar_wait(&bar, 0);
      staged = true;
      ta = (sl.hdr >= 0) ? tab_aux_at(sidx + sl.hdr, idx + d.aoff) : load_aux(idx ? idx + d.aoff : nullptr);
    }
    int64_t r[K_UNIF];
    search_k_sm(W, idx, sidx, d, sl, ta, u, r);
#pragma unroll
    for (int h = 0; h < K_UNIF; ++h)
      if (i[h] < N) out[i[h]] = r[h];
  }
}

// dr_match_dac (search mode) / dr_match_binary on given u's: persistent CTAs
// stage the top index levels once (capped so that several CTAs share an SM)
// and run two lock-step searches per thread over coalesced chunks of u
#ifndef DRS_MATCH_SMEM_CAP
#define DRS_MATCH_SMEM_CAP 2048
#endif
#ifndef MATCH_KQ
#define MATCH_KQ 4  // u's per thread in lock-step
#endif
#ifndef MATCH_KQ_DEF
#define MATCH_KQ_DEF 2  // the same on a deferred table (its band per u: registers)
#endif
// rng (optional, on the device, the range8 of include/drs.h): search only
// global u's rng[0] .. rng[1] of the windows u (base rng[4]) and out (base
// rng[5]) and add `shift` to the indices (a W shard of a sharded table)
// KIND 0: two full-node searches per thread (search_k_sm), the latency-bound
// case of few u's, either kind of table; KIND 1 / 2: MATCH_KQ searches per
// thread reading half nodes (search_half), for many u's per CTA, on a direct /
// a deferred table only -- the two are launched together and the one that
// does not match the table's header exits at once, so each compiles for its
// own kind (the deferred search's state would otherwise cost the direct one
// half its resident CTAs: 128 registers against 52)
template <int KIND>
__global__ void __launch_bounds__(256) k_match_index_sm(const double* __restrict__ W, const double* __restrict__ idx,
                                                        IndexDesc d, SmemLevels sl, const double* __restrict__ u,
                                                        int64_t N, int64_t* __restrict__ out,
                                                        const int64_t* __restrict__ rng, int64_t shift) {
  constexpr bool THROUGHPUT = KIND != 0;
  extern __shared__ __align__(128) double sidx[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t sbytes = (uint32_t)(sl.count * 8);
  pdl_wait();
  if (THROUGHPUT) {
    const bool def = idx && __ldg(idx + d.aoff + 1) != 0.0;
    if (def != (KIND == 2)) return;
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, sbytes);
    if (sbytes) bulk_g2s(sidx, idx + sl.base, sbytes, &bar);
  }
  __syncthreads();
  pdl_trigger();
  mbar_wait(&bar, 0);
  const TabAux ta = (sl.hdr >= 0) ? tab_aux_at(sidx + sl.hdr, idx + d.aoff) : load_aux(idx ? idx + d.aoff : nullptr);
  const int64_t lo = rng ? rng[0] : 0, hi = rng ? rng[1] : N;
  if (rng) {  // sharded: U and out are windows with global bases rng[4], rng[5]
    u -= rng[4];
    out -= rng[5];
  }
  constexpr int KQ = KIND == 1 ? MATCH_KQ : (KIND == 2 ? MATCH_KQ_DEF : K_UNIF);
  for (int64_t base = lo + (int64_t)blockIdx.x * KQ * blockDim.x; base < hi;
       base += (int64_t)gridDim.x * KQ * blockDim.x) {
    double x[KQ];
    int64_t i[KQ];
#pragma unroll
    for (int h = 0; h < KQ; ++h) {
      i[h] = base + h * blockDim.x + threadIdx.x;
      x[h] = (i[h] < hi) ? __ldg(u + i[h]) : 0.5;
    }
    int64_t r[KQ];
    if constexpr (KIND == 1) search_half_impl<KQ, false>(W, idx, sidx, d, sl, ta, x, r);
    else if constexpr (KIND == 2) search_half_impl<KQ, true>(W, idx, sidx, d, sl, ta, x, r);
    else search_k_sm(W, idx, sidx, d, sl, ta, x, r);
#pragma unroll
    for (int h = 0; h < KQ; ++h)
      if (i[h] < hi) out[i[h]] = shift + r[h];
  }
}

int launch_index_sm(const double* W, const double* idx, int64_t M, const double* u, int64_t N, int64_t* out,
                    cudaStream_t st, const int64_t* rng, int64_t shift) {
  const IndexDesc d = make_index_desc(M);
  const SmemLevels sl = plan_smem_levels(d, DRS_MATCH_SMEM_CAP);
  static SmemLimit lim, lim_1, lim_2;
  static OccupancyCache occ, occ_1, occ_2;
  const size_t smem = (size_t)sl.count * 8;
  lim.raise((const void*)k_match_index_sm<0>, SIDX_CAP * 8);
  lim_1.raise((const void*)k_match_index_sm<1>, SIDX_CAP * 8);
  lim_2.raise((const void*)k_match_index_sm<2>, SIDX_CAP * 8);
  const int64_t cap = (int64_t)drs_sm_count() * occ.get((const void*)k_match_index_sm<0>, 256, smem);
  // many u's per resident CTA: the data pipe bounds the searches (half nodes,
  // MATCH_KQ per thread); few: the dependent round trips do (full nodes, two)
  if (cdiv(N, 256 * K_UNIF) >= 4 * cap) {
    const int64_t chunks = cdiv(N, 256 * MATCH_KQ);
    const int64_t cap_1 = (int64_t)drs_sm_count() * occ_1.get((const void*)k_match_index_sm<1>, 256, smem);
    const int64_t cap_2 = (int64_t)drs_sm_count() * occ_2.get((const void*)k_match_index_sm<2>, 256, smem);
    // one of the two exits at its first instruction (the table header)
    launch_pdl(k_match_index_sm<1>, dim3((unsigned)(chunks < cap_1 ? chunks : cap_1)), dim3(256), smem, st, W, idx,
               d, sl, u, N, out, rng, shift);
    const int64_t chunks_2 = cdiv(N, 256 * MATCH_KQ_DEF);
    launch_pdl(k_match_index_sm<2>, dim3((unsigned)(chunks_2 < cap_2 ? chunks_2 : cap_2)), dim3(256), smem, st, W, idx,
               d, sl, u, N, out, rng, shift);
    return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
  }
  const int64_t chunks = cdiv(N, 256 * K_UNIF);
  const int64_t grid = chunks < cap ? chunks : cap;
  launch_pdl(k_match_index_sm<0>, dim3((unsigned)grid), dim3(256), smem, st, W, idx, d, sl, u, N, out, rng, shift);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

__global__ void k_advance_offset(uint64_t* p, uint64_t by) { *p += by; }

// co-resident CTAs of the cooperative fused kernel on this device
static int coop_capacity() {
  static SmemLimit lim;
  static OccupancyCache occ;
  lim.raise((const void*)k_dac_fused<true>, SIDX_CAP * 8);
  return drs_sm_count() * occ.get((const void*)k_dac_fused<true>, THREADS, SIDX_CAP * 8);
}
static int coop_capacity_uniforms() {  // the uniforms-only instantiation: no dynamic shared memory
  static OccupancyCache occ;
  return drs_sm_count() * occ.get((const void*)k_dac_fused<false>, THREADS, 0);
}

}  // namespace drs

using namespace drs;

namespace drs {
int sorted_uniforms_from_launch(const double* raw, int64_t n, double* U, int32_t* status, void* ws,
                                size_t ws_bytes, cudaStream_t st);

// the optional fused gather: gout[i] = states[out[i] / divisor] (K rows of gd)
struct GatherSpec {
  const double* states;
  int64_t K, gd, divisor;
  double* gout;
};

int launch_gather_rows(const double* states, int64_t K, int64_t d, const int64_t* idx, int64_t N, int64_t divisor,
                       double* out, int32_t* status, cudaStream_t st);

// The fused kernel's launch.  A cooperative launch costs ~7 us of host time
// per call (the co-residency check); the same launch as the one kernel node
// of a graph, instantiated once per (device, stream, grid) with the
// cooperative attribute and re-parameterised per call
// (cudaGraphExecKernelNodeSetParams), costs less host time.  A stream being
// captured (the caller's own CUDA graph) takes the plain cooperative launch.
struct FusedGraph {
  int dev;
  cudaStream_t st;
  unsigned grid;
  cudaGraphExec_t ex;
  cudaGraphNode_t node;
};

static cudaError_t launch_fused(const FusedArgs& a, unsigned grid, cudaStream_t st, bool graph,
                                size_t smem = (size_t)SIDX_CAP * 8) {
  static const bool use_graph = getenv("DRS_NO_GRAPH") == nullptr;
  static std::mutex mu;
  static std::vector<FusedGraph> cache;
  static bool broken = false;
  void* args[] = {(void*)&a};
  if (graph && use_graph && !broken) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    int dev = 0;
    if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone &&
        cudaGetDevice(&dev) == cudaSuccess) {
      cudaKernelNodeParams p = {};
      p.func = (void*)k_dac_fused<true>;
      p.gridDim = dim3(grid);
      p.blockDim = dim3(THREADS);
      p.sharedMemBytes = (unsigned)(SIDX_CAP * 8);
      p.kernelParams = args;
      std::lock_guard<std::mutex> lk(mu);
      FusedGraph* f = nullptr;
      for (auto& c : cache)
        if (c.dev == dev && c.st == st && c.grid == grid) f = &c;
      if (!f) {
        cudaGraph_t g = nullptr;
        FusedGraph n{dev, st, grid, nullptr, nullptr};
        cudaLaunchAttributeValue v = {};
        v.cooperative = 1;
        bool ok = cudaGraphCreate(&g, 0) == cudaSuccess && cudaGraphAddKernelNode(&n.node, g, nullptr, 0, &p) == cudaSuccess &&
                  cudaGraphKernelNodeSetAttribute(n.node, cudaLaunchAttributeCooperative, &v) == cudaSuccess &&
                  cudaGraphInstantiate(&n.ex, g, 0) == cudaSuccess;
        if (!ok) {
          cudaGetLastError();
          broken = true;  // the plain cooperative launch from now on
        } else {
          cache.push_back(n);
          f = &cache.back();
        }
      }
      if (f) {
        if (cudaGraphExecKernelNodeSetParams(f->ex, f->node, &p) == cudaSuccess) return cudaGraphLaunch(f->ex, st);
        cudaGetLastError();
        broken = true;
      }
    }
  }
  return cudaLaunchCooperativeKernel(smem ? (void*)k_dac_fused<true> : (void*)k_dac_fused<false>, dim3(grid),
                                     dim3(THREADS), args, smem, st);
}

// The sorted uniforms alone as ONE cooperative launch (k_dac_fused<false>, no
// table: draws, -log, in-tile chain, counter exchange, every CTA folds the
// tile chain, U = Z / Z[n], the repair behind grid barriers) when the n + 1
// spacings fit a co-resident grid; the pass 1 / chain / pass 2 / finalize
// pipeline otherwise.  U, the status word and the device stream advance are
// bit-identical either way (tests/test_gpu_parity.py).
int sorted_uniforms_auto(uint64_t k0, uint64_t k1, uint64_t offset, uint64_t* offset_dev, const double* raw,
                         int64_t n, double* U, int32_t* status, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int64_t nt = cdiv(n + 1, TS_U);
  const bool fused_ok = getenv("DRS_NO_FUSED_UNIFORMS") == nullptr;  // the pipeline, for A/B and tests
  // up to three tiles per SM: measured (scripts/mid_n_probe.py, M = 2^26 dac search) 19.5 vs 22.5 us at
  // n = 75,776, 21.2 vs 24.2 at 2^17, 29.7 vs 30.7 at 2^18; at the fourth CTA per SM (n ~ 3 10^5) the pipeline wins
  const int64_t fused_cap = std::min<int64_t>(coop_capacity_uniforms(), 3 * (int64_t)drs_sm_count());
  if (fused_ok && n >= 1 && U && nt <= fused_cap && nt <= FUSED_MAX_TILES && nt <= ws_capacity_tiles(ws_bytes)) {
    FusedArgs a = {};
    a.sl.hdr = -1;
    a.k0 = k0; a.k1 = k1; a.offset = offset; a.offset_dev = offset_dev; a.raw = raw;
    a.n = n; a.U = U; a.out = nullptr; a.status = status;
    a.ws = carve_ws(ws, ws_bytes);
    a.divisor = 1;
    return launch_fused(a, (unsigned)nt, st, false, 0) == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
  }
  return raw ? sorted_uniforms_from_launch(raw, n, U, status, ws, ws_bytes, st)
             : sorted_uniforms_launch(k0, k1, offset, offset_dev, n, U, status, ws, ws_bytes, st);
}

static int sample_dac_impl(const double* W, const double* idx, int64_t M, uint64_t k0, uint64_t k1,
                           uint64_t offset, uint64_t* offset_dev, const double* raw, int64_t N,
                           double* U, int64_t* out, int32_t* status, int32_t mode, void* ws,
                           size_t ws_bytes, cudaStream_t st, const GatherSpec* g = nullptr,
                           bool graph = false) {
  if (M < 1 || N < 1 || !W || !out || !status || !ws || !U) return DRS_ERR_ARG;
  if (mode != DRS_DAC_AUTO && mode != DRS_DAC_MERGE && mode != DRS_DAC_SEARCH) return DRS_ERR_MODE;
  if ((uintptr_t)W & 31) return DRS_ERR_ALIGN;
  const IndexDesc d = make_index_desc(M);
  if (d.levels > 0 && !idx) return DRS_ERR_ARG;
  const int64_t nt = cdiv(N + 1, TS_U);
  const bool merge = (mode == DRS_DAC_MERGE) || (mode == DRS_DAC_AUTO && M <= (int64_t)DRS_DAC_TAU * N);
  if (!merge && nt <= coop_capacity() && nt <= FUSED_MAX_TILES && nt <= ws_capacity_tiles(ws_bytes)) {
    FusedArgs a;
    a.W = W; a.idx = idx; a.d = d; a.sl = plan_smem_levels(d);
    a.k0 = k0; a.k1 = k1; a.offset = offset; a.offset_dev = offset_dev; a.raw = raw;
    a.n = N; a.U = U; a.out = out; a.status = status;
    a.ws = carve_ws(ws, ws_bytes);
    a.states = g ? g->states : nullptr; a.gout = g ? g->gout : nullptr;
    a.K = g ? g->K : 0; a.gd = g ? g->gd : 0; a.divisor = g ? g->divisor : 1;
    a.gd_vec2 = g && (g->gd % 2 == 0) && ((((uintptr_t)g->states) | ((uintptr_t)g->gout)) & 15) == 0;
    return launch_fused(a, (unsigned)nt, st, graph) == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
  }
  const int rc = sorted_uniforms_auto(k0, k1, offset, offset_dev, raw, N, U, status, ws, ws_bytes, st);
  if (rc) return rc;
  const int rm = merge ? launch_merge(W, idx, M, U, N, out, st) : launch_index(W, idx, M, U, N, out, st);
  if (rm || !g) return rm;
  // two-pass pipeline: the gather follows the match on the stream
  return launch_gather_rows(g->states, g->K, g->gd, out, N, g->divisor, g->gout, status, st);
}
}  // namespace drs

extern "C" {

#ifdef DRS_PHASE_TIMING
int dr_debug_phase_times(unsigned long long* host, int n) {
  return cudaMemcpyFromSymbol(host, g_phase, sizeof(unsigned long long) * (size_t)n) == cudaSuccess ? 0 : -1;
}
int dr_debug_phase_clear(void) {
  void* p = nullptr;
  if (cudaGetSymbolAddress(&p, g_phase) != cudaSuccess) return -1;
  return cudaMemset(p, 0, sizeof(g_phase)) == cudaSuccess ? 0 : -1;
}
#endif

int dr_sample_dac_from(const double* W, const double* idx, int64_t M, const double* raw, int64_t N,
                       double* U, int64_t* out, int32_t* status, int32_t mode, void* ws,
                       size_t ws_bytes, void* stream) {
  if (!raw) return DRS_ERR_ARG;
  return sample_dac_impl(W, idx, M, 0, 0, 0, nullptr, raw, N, U, out, status, mode, ws, ws_bytes,
                         (cudaStream_t)stream);
}

int dr_sample_dac(const double* W, const double* idx, int64_t M, uint64_t k0, uint64_t k1,
                  uint64_t offset, uint64_t* offset_dev, int64_t N, double* U, int64_t* out,
                  int32_t* status, int32_t mode, void* ws, size_t ws_bytes, void* stream) {
  return sample_dac_impl(W, idx, M, k0, k1, offset, offset_dev, nullptr, N, U, out, status, mode, ws,
                         ws_bytes, (cudaStream_t)stream);
}

int dr_sample_dac_sync(const double* W, const double* idx, int64_t M, uint64_t k0, uint64_t k1,
                       uint64_t offset, uint64_t* offset_dev, int64_t N, double* U, int64_t* out,
                       int32_t* status, int32_t mode, void* ws, size_t ws_bytes, void* stream) {
  const int rc = sample_dac_impl(W, idx, M, k0, k1, offset, offset_dev, nullptr, N, U, out, status, mode, ws,
                                 ws_bytes, (cudaStream_t)stream, nullptr, true);
  if (rc) return rc;
  return cudaStreamSynchronize((cudaStream_t)stream) == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

int dr_sample_dac_gather(const double* W, const double* idx, int64_t M, uint64_t k0, uint64_t k1,
                         uint64_t offset, uint64_t* offset_dev, int64_t N, double* U, int64_t* out,
                         const double* states, int64_t K, int64_t d, int64_t divisor, double* gout,
                         int32_t* status, int32_t mode, void* ws, size_t ws_bytes, void* stream) {
  if (K < 1 || d < 1 || divisor < 1 || !states || !gout) return DRS_ERR_ARG;
  // every index the sampler can return maps to a row: (M - 1) / divisor < K
  if (M >= 1 && (M - 1) / divisor >= K) return DRS_ERR_ARG;
  const GatherSpec g{states, K, d, divisor, gout};
  return sample_dac_impl(W, idx, M, k0, k1, offset, offset_dev, nullptr, N, U, out, status, mode, ws,
                         ws_bytes, (cudaStream_t)stream, &g);
}

int dr_sample_ccf(const double* W, const double* idx, int64_t M, uint64_t k0, uint64_t k1, uint64_t offset,
                  uint64_t* offset_dev, int64_t N, double* U, int64_t* out, int32_t* status, void* ws,
                  size_t ws_bytes, void* stream) {
  if (M < 1 || N < 1 || !W || !U || !out || !status || !ws) return DRS_ERR_ARG;
  if ((uintptr_t)W & 15) return DRS_ERR_ALIGN;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = sorted_uniforms_auto(k0, k1, offset, offset_dev, nullptr, N, U, status, ws, ws_bytes, st);
  if (rc) return rc;
  return launch_merge(W, idx, M, U, N, out, st);
}

int dr_sample_binary_dev(const double* W, const double* idx, int64_t M, uint64_t k0, uint64_t k1,
                      uint64_t offset, uint64_t* offset_dev, int64_t N, int64_t* out, void* stream) {
  if (M < 1 || N < 0 || !W || (N > 0 && !out)) return DRS_ERR_ARG;
  if ((uintptr_t)W & 31) return DRS_ERR_ALIGN;
  if (N == 0) return DRS_OK;
  const IndexDesc d = make_index_desc(M);
  if (d.levels > 0 && !idx) return DRS_ERR_ARG;
  const SmemLevels sl = plan_smem_levels(d);
  // persistent grid: as many CTAs as fit with this shared-memory size
  static SmemLimit lim;
  static OccupancyCache occ;
  const size_t smem = (size_t)sl.count * 8;
  lim.raise((const void*)k_sample_binary_sm, SIDX_CAP * 8);
  const int64_t cap = (int64_t)drs_sm_count() * occ.get((const void*)k_sample_binary_sm, 256, smem);
  const int64_t chunks = cdiv(N, 512);
  const int64_t grid = chunks < cap ? chunks : cap;
  k_sample_binary_sm<<<(unsigned)grid, 256, smem, (cudaStream_t)stream>>>(W, idx, d, sl, k0, k1, offset,
                                                                          offset_dev, N, out);
  if (cudaGetLastError() != cudaSuccess) return DRS_ERR_LAUNCH;
  if (offset_dev) k_advance_offset<<<1, 1, 0, (cudaStream_t)stream>>>(offset_dev, (uint64_t)N);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

}  // extern "C"
