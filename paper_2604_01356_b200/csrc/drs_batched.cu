// drs_batched.cu -- many independent filters in one launch (config 4).
//
// The reference resamples a bank of filters with a Python loop of
// build_weight_table (cdf.py:59-89) + dac_sampler (samplers.py:262-266) per
// filter.  Here two launches serve the whole bank:
//
//   k_batched_uniforms_warp (N_f + 1 <= 512; k_batched_uniforms beyond) one
//     warp per filter draws the N_f + 1 Philox spacings (each Philox block
//     once), folds them with the association of dr_sorted_uniforms,
//     normalises, repairs collapses and writes U[f]; 24+ warps per SM keep
//     this compute-bound step wide;
//   k_resample_batched  one thread-block CLUSTER per filter, one CTA per table
//     tile of the chained scan (THREADS x K_TABLE = 8448 weights; M_f = 16384
//     is a 2-CTA cluster):
//   * CTA r stages its tile of w_f in shared memory with one TMA bulk copy
//     (~66 KB, so three CTAs share an SM and one CTA's copy overlaps the
//     others' compute) and U[f] with a second one;
//   * ONE sweep over the tile: each lane folds its K_TABLE-element chunk
//     serially (validating from the high words in the integer pipe), writes
//     the chunk-local prefix s2 in place, and the CTA folds lane and warp
//     totals (Q, R) -- the chained association of dr_build_table, so W is
//     bit-identical to the single-filter path;
//   * the tile totals A_r are exchanged through distributed shared memory
//     (st.async into every peer, completing the peer's transaction barrier;
//     no cluster-wide barrier after the start); every CTA then folds the
//     tile prefixes P_r and the filter total T in tile order;
//   * CTA r answers exactly the draws u with W_end(r-1) < u <= W_end(r),
//     W_end(r) = min(P_{r+1} / T, 1) being W at the tile's last entry, i.e.
//     P_r < s*(u) <= P_{r+1}: every thread forms s*(u) for its draws and keeps
//     those of its tile, then a bisection over its lane-chunk ends and inside
//     the chunk, whose
//     probes form W_j = min((P_r + (R + (Q + s2_j))) / T, 1) on the fly
//     (a few divisions per draw instead of one per weight; all of W only on
//     request).
// Global traffic per filter: w_f once, U twice (written, read), the indices
// (+ W on request).
// The (k0, k1, offset) stream keys are read on the device and, with
// `advance`, moved forward by N_f + 1 there (graph-replayable).  Filters
// shard across GPUs with no collective.
#include "drs_common.cuh"

namespace drs {

constexpr int64_t TS_TABLE = (int64_t)THREADS * K_TABLE;
constexpr int64_t TS_UNIF = (int64_t)THREADS * K_UNIF;
constexpr int MAX_TT = 8;  // table tiles per filter = cluster size (portable limit)
constexpr int MAX_UT = 8;  // uniform tiles per filter

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// store v into the shared-memory word `local` of CTA `rank` of this cluster
// and complete 8 bytes of that CTA's transaction barrier `bar` (st.async: no
// cluster barrier, no fence; the receiver waits on its own barrier)
__device__ __forceinline__ void st_async_cluster_f64(double* local, uint64_t* bar, uint32_t rank, double v) {
  uint32_t rdst, rbar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(smem_u32(local)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(rdst),
               "l"((unsigned long long)__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
// wait for phase `phase` of a barrier completed by peers of the cluster
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

// s*(x) = s_star (drs_common.cuh): the least double s with fl(s / T) >= x,
// so that fl(S / T) < x <=> S < s*(x).

// the exactness check and repair of randkit.py:95-116 on a filter's U (in
// shared memory), by thread 0 and serially: rare, and N_f is small
__device__ __forceinline__ void uniform_repair(double* su, int64_t Nf, unsigned long long smin, double total,
                                               int r, int32_t* status) {
  const double zmin = __longlong_as_double((long long)smin);
  if (threadIdx.x != 0 || zmin > __dmul_rn(1e-14, total)) return;
  bool b2 = (su[0] <= 0.0) || (su[Nf - 1] >= 1.0);
  for (int64_t i = 1; !b2 && i < Nf; ++i) b2 = !(__dsub_rn(su[i], su[i - 1]) > 0.0);
  if (!b2) return;
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
  if (r == 0) atomicOr(status, DRS_ST_REPAIRED);
}

struct BatchedArgs {
  const double* w;
  int64_t B, Mf, Nf;
  uint64_t* keys;  // [B][3] = k0, k1, draw offset
  int advance;     // move keys[f][2] forward by Nf + 1 on the device
  double* Wout;    // optional [B][Mf]
  double* Uout;    // optional [B][Nf]
  const double* Uin;  // [B][Nf] from k_batched_uniforms
  int64_t* out;    // [B][Nf]
  int32_t* status;
  int ntt, ntu;
};

// Sorted uniforms of every filter: one CTA per filter draws its N_f + 1
// spacings (each Philox block once when they fit one tile), folds them with
// the association of dr_sorted_uniforms, normalises, repairs collapses and
// writes U[f] -- all filters in one wide launch of small CTAs (8 or more per
// SM), so the cluster kernel below only reads 8 N_f bytes per filter.
__global__ void __launch_bounds__(THREADS) k_batched_uniforms(const __grid_constant__ BatchedArgs a,
                                                              double* __restrict__ U) {
  asm volatile("griddepcontrol.launch_dependents;");  // the cluster kernel may start its weight copies
  extern __shared__ __align__(128) double su[];  // [ne + 8]: Philox words, inner sums, then U
  __shared__ FoldSmem fs;
  __shared__ double s_Au[MAX_UT];
  __shared__ unsigned long long s_min;
  const int64_t Nf = a.Nf, ne = Nf + 1;
  const int64_t f = blockIdx.x;
  const int r = 0;
  const uint64_t k0 = a.keys[3 * f], k1 = a.keys[3 * f + 1], off = a.keys[3 * f + 2];
  if (threadIdx.x == 0) s_min = 0x7FF0000000000000ULL;
  __syncthreads();
  if (Nf > 0) {
    unsigned long long mn = 0x7FF0000000000000ULL;
    for (int t = 0; t < a.ntu; ++t) {
      const int64_t e0 = t * TS_UNIF + (int64_t)threadIdx.x * K_UNIF;
      double z[K_UNIF];
#pragma unroll
      for (int i = 0; i < K_UNIF; ++i) z[i] = 0.0;
      if (a.ntu == 1) {
        // one tile: each Philox block is computed once, by one thread, into
        // su (sized for it; su is written only after these words are read)
        uint64_t* words = reinterpret_cast<uint64_t*>(su);
        const uint64_t b0 = off >> 2;
        const int nblk = (int)(((off + (uint64_t)ne - 1) >> 2) - b0 + 1);
        for (int blk = threadIdx.x; blk < nblk; blk += THREADS) {
          const U64x4 v = philox_block(k0, k1, b0 + (uint64_t)blk);
          words[4 * blk + 0] = v.w0; words[4 * blk + 1] = v.w1;
          words[4 * blk + 2] = v.w2; words[4 * blk + 3] = v.w3;
        }
        __syncthreads();
        const int a0 = (int)(off & 3);
#pragma unroll
        for (int i = 0; i < K_UNIF; ++i) {
          if (e0 + i < ne) {
            z[i] = neglog(u01(words[a0 + e0 + i]));
            mn = min(mn, (z[i] > 0.0) ? (unsigned long long)__double_as_longlong(z[i]) : 0ull);
          }
        }
        __syncthreads();  // words read before su is written
      } else if (e0 < ne) {
        const uint64_t d0 = off + (uint64_t)e0;
        const uint64_t b0 = d0 >> 2, b1 = (d0 + K_UNIF - 1) >> 2;
        const U64x4 v0 = philox_block(k0, k1, b0);
        U64x4 v1 = v0;
        if (b1 != b0) v1 = philox_block(k0, k1, b1);
#pragma unroll
        for (int i = 0; i < K_UNIF; ++i) {
          const uint64_t dd = d0 + (uint64_t)i;
          const uint64_t raw = ((dd >> 2) == b0) ? pick(v0, (int)(dd & 3)) : pick(v1, (int)(dd & 3));
          if (e0 + i < ne) {
            z[i] = neglog(u01(raw));
            mn = min(mn, (z[i] > 0.0) ? (unsigned long long)__double_as_longlong(z[i]) : 0ull);
          }
        }
      }
      double sc[K_UNIF];
      sc[0] = z[0];
#pragma unroll
      for (int i = 1; i < K_UNIF; ++i) sc[i] = __dadd_rn(sc[i - 1], z[i]);
      double Q, R;
      const double A = block_fold(sc[K_UNIF - 1], fs, Q, R);
      if (threadIdx.x == 0) s_Au[t] = A;
#pragma unroll
      for (int i = 0; i < K_UNIF; ++i)
        if (e0 + i < ne) su[e0 + i] = __dadd_rn(R, __dadd_rn(Q, sc[i]));
      __syncthreads();  // fs reuse
    }
    block_min_u64(&s_min, mn);
    double Pu[MAX_UT];
    double total = 0.0;
#pragma unroll
    for (int t = 0; t < MAX_UT; ++t) {
      Pu[t] = total;
      if (t < a.ntu) total = __dadd_rn(total, s_Au[t]);
    }
    for (int64_t i = threadIdx.x; i < Nf; i += THREADS) {
      const int t = (int)(i / TS_UNIF);
      double p = Pu[0];
#pragma unroll
      for (int q = 1; q < MAX_UT; ++q) p = (q == t) ? Pu[q] : p;
      su[i] = __ddiv_rn(__dadd_rn(p, su[i]), total);
    }
    __syncthreads();
    uniform_repair(su, Nf, s_min, total, r, a.status);
  }

  __syncthreads();
  for (int64_t i = threadIdx.x; i < Nf; i += THREADS) U[f * Nf + i] = su[i];
  if (threadIdx.x == 0 && a.advance) a.keys[3 * f + 2] = off + (uint64_t)ne;  // every thread has read it
}

// N_f + 1 <= 512 (one uniform tile): ONE WARP per filter, eight filters per
// CTA, no CTA barrier.  Lane l holds the two spacings 64 w + 2 l, + 1 of every
// spacing row w < nw = ceil((N_f + 1) / 64) -- the lane chunks of
// dr_sorted_uniforms' tile (rows past nw hold zeros, so folding only nw rows
// gives the tile fold's bits: x + 0.0 == x).  The filter's Philox blocks are
// computed once each (lane b takes blocks b, b + 32, ...) into the warp's
// shared buffer; lane w folds row w's 32 chunk totals serially in place
// (the row bases Q), every lane folds the row totals (R, A); U is divided in
// registers and stored 16 bytes per lane.  The exactness check / repair of
// randkit.py:95-116 runs on lane 0 when the spacing minimum asks for it.
constexpr int UW_FILTERS = 4;                 // warps (filters) per CTA
constexpr int UW_BUF = TS_UNIF + 8;           // doubles per warp: Philox words, then row totals, then U
#ifdef DRS_PHASE_TIMING
#define WSTAMP(ph)                                                                          \
  do {                                                                                      \
    if (lane == 0) {                                                                        \
      unsigned long long tt_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt_));                              \
      g_phase[150000 + ((int64_t)blockIdx.x * UW_FILTERS + warp) * 8 + (ph)] = tt_;        \
    }                                                                                       \
  } while (0)
#else
#define WSTAMP(ph) do {} while (0)
#endif
template <int NW>  // spacing rows = ceil((N_f + 1) / 64), unrolled without guards
__global__ void __launch_bounds__(UW_FILTERS * LANES, 7) k_batched_uniforms_warp(const __grid_constant__ BatchedArgs a,
                                                                                double* __restrict__ U) {
  asm volatile("griddepcontrol.launch_dependents;");  // the cluster kernel may start its weight copies
  __shared__ __align__(16) double sbuf[UW_FILTERS][UW_BUF];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t f = (int64_t)blockIdx.x * UW_FILTERS + warp;
  if (f >= a.B) return;
  WSTAMP(0);
  const int64_t Nf = a.Nf, ne = Nf + 1;
  constexpr int nw = NW;
  double* buf = sbuf[warp];
  uint64_t* words = reinterpret_cast<uint64_t*>(buf);
  const uint64_t k0 = a.keys[3 * f], k1 = a.keys[3 * f + 1], off = a.keys[3 * f + 2];
  const uint64_t b0 = off >> 2;
  const int nblk = (int)(((off + (uint64_t)Nf) >> 2) - b0 + 1);
  WSTAMP(1);
  for (int blk = lane; blk < nblk; blk += 2 * LANES) {  // two blocks per lane in flight
    const int blk2 = blk + LANES;
    const U64x4 v = philox_block(k0, k1, b0 + (uint64_t)blk);
    words[4 * blk + 0] = v.w0; words[4 * blk + 1] = v.w1;
    words[4 * blk + 2] = v.w2; words[4 * blk + 3] = v.w3;
    if (blk2 < nblk) {  // a warp whose lanes all lie past the last block skips the second block
      const U64x4 v2 = philox_block(k0, k1, b0 + (uint64_t)blk2);
      words[4 * blk2 + 0] = v2.w0; words[4 * blk2 + 1] = v2.w1;
      words[4 * blk2 + 2] = v2.w2; words[4 * blk2 + 3] = v2.w3;
    }
  }
  __syncwarp();
  WSTAMP(2);
  const int a0 = (int)(off & 3);
  double sc0[NW], sc1[NW];
  unsigned long long mn = 0x7FF0000000000000ULL;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int e0 = 64 * w + 2 * lane;
    const bool v0 = e0 < ne, v1 = e0 + 1 < ne;
    // rows before the last are full (64 (NW - 1) < ne); in the last one a log
    // no lane needs is not issued at all (N_f = 256: one spacing in that row)
    const double l0 = (w < NW - 1 || v0) ? neglog(u01(words[a0 + (v0 ? e0 : 0)])) : 0.0;
    const double l1 = (w < NW - 1 || v1) ? neglog(u01(words[a0 + (v1 ? e0 + 1 : 0)])) : 0.0;
    const double z0 = v0 ? l0 : 0.0, z1 = v1 ? l1 : 0.0;
    const unsigned long long m0 = (v0 && !(z0 > 0.0)) ? 0ull
                                  : (v0 ? (unsigned long long)__double_as_longlong(z0) : 0x7FF0000000000000ULL);
    const unsigned long long m1 = (v1 && !(z1 > 0.0)) ? 0ull
                                  : (v1 ? (unsigned long long)__double_as_longlong(z1) : 0x7FF0000000000000ULL);
    mn = min(mn, min(m0, m1));
    sc0[w] = z0;
    sc1[w] = __dadd_rn(z0, z1);
  }
  // rounded down to the high word (see block_min_u64): only the exactness trigger uses it
  mn = (unsigned long long)__reduce_min_sync(FULL, (unsigned)(mn >> 32)) << 32;
  WSTAMP(3);
  __syncwarp();  // the words are consumed: the buffer holds the row totals now
  double* rows = buf;  // [w][33]: chunk totals of row w, then their bases Q (in place)
#pragma unroll
  for (int w = 0; w < NW; ++w) rows[w * (LANES + 1) + lane] = sc1[w];
  __syncwarp();
  double* G = buf + WARPS * (LANES + 1);  // row totals
  if (lane < nw) {
    double* row = rows + lane * (LANES + 1);
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < LANES; ++j) {
      const double v = row[j];
      row[j] = acc;
      acc = __dadd_rn(acc, v);
    }
    G[lane] = acc;
  }
  __syncwarp();
  WSTAMP(4);
  double A = 0.0, R[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    R[w] = A;
    A = __dadd_rn(A, G[w]);
  }
  double* Uf = U + f * Nf;
  const double zmin = __longlong_as_double((long long)mn);
  const bool rep = !(zmin > __dmul_rn(1e-14, A));  // the exactness check of randkit.py:95
  const bool vec = (((uintptr_t)Uf) & 15) == 0;
  // all 2 NW divisions first (independent, so they overlap), then the stores
  double u0[NW], u1[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const double Q = rows[w * (LANES + 1) + lane];
    if (w < NW - 1 || 64 * w < Nf) {  // the last row may hold only the (n+1)-th spacing, never stored
      u0[w] = __ddiv_rn(__dadd_rn(R[w], __dadd_rn(Q, sc0[w])), A);
      u1[w] = __ddiv_rn(__dadd_rn(R[w], __dadd_rn(Q, sc1[w])), A);
    } else {
      u0[w] = u1[w] = 2.0;
    }
  }
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int e0 = 64 * w + 2 * lane;
    if (vec && e0 + 1 < Nf) {
      *reinterpret_cast<double2*>(Uf + e0) = make_double2(u0[w], u1[w]);
    } else {
      if (e0 < Nf) Uf[e0] = u0[w];
      if (e0 + 1 < Nf) Uf[e0 + 1] = u1[w];
    }
  }
  if (rep) {  // warp-uniform, rare: lane 0 checks and repairs the stored U serially
    __syncwarp();
    double* su = Uf;
    if (lane == 0 && Nf > 0) {
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
        atomicOr(a.status, DRS_ST_REPAIRED);
      }
    }
  }
  if (lane == 0 && a.advance) a.keys[3 * f + 2] = off + (uint64_t)ne;  // every lane has read it
  WSTAMP(5);
}

__global__ void __launch_bounds__(THREADS) k_resample_batched(const __grid_constant__ BatchedArgs a) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar, baru, barx;
  __shared__ FoldSmem fs;         // fold of the table tile
  __shared__ double s_R[WARPS];   // warp bases R of the table tile
  __shared__ double s_A[MAX_TT];  // tile totals, written by every CTA of the cluster
  __shared__ int s_bad;
  __shared__ double s_cend[THREADS];  // S at each lane chunk's last entry
  const int64_t Mf = a.Mf, Nf = a.Nf;
  const int r = (int)cluster_rank();
  const int64_t f = blockIdx.x / a.ntt;
  const int64_t j0 = (int64_t)r * TS_TABLE;  // first weight of this tile
  const int len = (int)((Mf - j0) < TS_TABLE ? (Mf - j0) : TS_TABLE);
  double* sw = sm;             // [TS_TABLE] raw w, then chunk-local prefixes s2
  double* sQ = sw + TS_TABLE;  // [THREADS] lane-chunk bases Q
  double* su = sQ + THREADS;   // [ne] inner sums, then U
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* wt = a.w + f * Mf + j0;
  const bool tma = ((((uintptr_t)wt) | ((uintptr_t)len * 8)) & 15) == 0;

  const double* ut = a.Uin + f * Nf;
  const bool tmau = Nf > 0 && ((((uintptr_t)ut) | ((uintptr_t)Nf * 8)) & 15) == 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&barx, 1);  // the peers' tile totals (st.async, 8 bytes each)
    mbar_init(&baru, 1);  // U[f]
    if (tma) {
      mbar_expect_tx(&bar, (uint32_t)len * 8u);
      bulk_g2s(sw, wt, (uint32_t)len * 8u, &bar);
    }
    s_bad = 0;
  }
  if (!tma)
    for (int i = threadIdx.x; i < len; i += THREADS) sw[i] = wt[i];
  for (int i = len + threadIdx.x; i < TS_TABLE; i += THREADS) sw[i] = 0.0;  // tile padding
  __syncthreads();
  // U[f] by TMA as early as possible: griddepcontrol.wait blocks only the
  // waiting thread (and returns at once unless this CTA started before the
  // uniforms grid finished, in which case the CTA waits at its first barrier)
  if (threadIdx.x == 0 && Nf > 0 && tmau) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    mbar_expect_tx(&baru, (uint32_t)Nf * 8u);
    bulk_g2s(su, ut, (uint32_t)Nf * 8u, &baru);
  }
  STAMP(0);
  // first half of a split cluster barrier: peers may store into this CTA's
  // shared memory only once every CTA of the cluster is running
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");

  // ---- 1. the table sweep over this CTA's tile.  The launch may overlap the
  // uniforms kernel (programmatic dependent launch): the weights were written
  // before it, so the sweep and the in-tile fold run before waiting on U.
  STAMP(1);
  if (tma) mbar_wait(&bar, 0);
  STAMP(2);
  // valid weight <=> 0 <= x < inf (-0.0 included, NaN excluded): one OR of
  // the high words per weight catches any sign bit, and an infinite or NaN
  // weight makes the chunk sum non-finite; either sends the chunk to an exact
  // re-check of the raw weights (a finite overflow of the sum is not invalid)
  uint32_t any_sign = 0;
  const int c0 = threadIdx.x * K_TABLE;
  double* chunk = sw + c0;
  double s = 0.0;
  if (c0 + K_TABLE <= len) {
#pragma unroll
    for (int i = 0; i < K_TABLE; ++i) {
      const double x = chunk[i];
      any_sign |= (uint32_t)__double2hiint(x);
      s = (i == 0) ? x : __dadd_rn(s, x);
      chunk[i] = s;
    }
  } else {
#pragma unroll
    for (int i = 0; i < K_TABLE; ++i) {
      const double x = chunk[i];
      any_sign |= (uint32_t)__double2hiint(x);
      s = (i == 0) ? x : __dadd_rn(s, x);
      if (c0 + i < len) chunk[i] = s;
    }
  }
  bool bad = false;
  if ((any_sign & 0x80000000u) || !(s < dinf()))
    for (int i = 0; i < K_TABLE && c0 + i < len; ++i) {
      const double x = wt[c0 + i];
      bad |= !(x >= 0.0) || x == dinf();
    }
  double Q, R;
  const double A = block_fold(s, fs, Q, R);
  sQ[threadIdx.x] = Q;
  if (lane == 0) s_R[warp] = R;
  if (bad) s_bad = 1;

  // ---- 2. this filter's sorted uniforms when they could not be copied by TMA
  // (thread 0 issued the copy at the start otherwise)
  if (Nf > 0 && !tmau) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int64_t i = threadIdx.x; i < Nf; i += THREADS) su[i] = a.Uin[f * Nf + i];
  }

  STAMP(3);
  // ---- 3. exchange the tile totals through distributed shared memory: each
  // CTA stores its total into every peer with st.async, completing 8 bytes of
  // the peer's transaction barrier, and waits on its own
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  if (threadIdx.x == 0) {
    s_A[r] = A;
    mbar_expect_tx(&barx, 8u * (uint32_t)(a.ntt - 1));
    for (int q = 0; q < a.ntt; ++q)
      if (q != r) st_async_cluster_f64(&s_A[r], &barx, (uint32_t)q, A);
  }
  mbar_wait_cluster(&barx, 0);
  if (Nf > 0 && tmau) mbar_wait(&baru, 0);
  __syncthreads();  // sQ / s_R / s_bad / su / s_A
  double Pr = 0.0, T = 0.0;
  for (int q = 0; q < a.ntt; ++q) {
    if (q == r) Pr = T;
    T = __dadd_rn(T, s_A[q]);
  }
  const double Pnext = __dadd_rn(Pr, s_A[r]);  // == S at the tile's last entry
  // S at the end of every lane chunk (the search's first level)
  {
    const int lastc = (c0 + K_TABLE <= len) ? K_TABLE - 1 : len - 1 - c0;
    s_cend[threadIdx.x] = (lastc >= 0) ? __dadd_rn(Pr, __dadd_rn(s_R[warp], __dadd_rn(Q, chunk[lastc]))) : dinf();
  }
  __syncthreads();
  STAMP(4);
  if (threadIdx.x == 0) {
    int st = s_bad ? DRS_ST_INVALID_WEIGHT : 0;
    if (r == 0) {
      if (T == 0.0) st |= DRS_ST_DEGENERATE;
      if (!(T < dinf())) st |= DRS_ST_ACCUM_OVERFLOW;
    }
    if (st) atomicOr(a.status, st);
  }

  // ---- 4. the draws that land in this tile, by bisection on the unnormalised
  // prefix: W_j < u  <=>  fl(S_j / T) < u  <=>  S_j < s*(u), where s*(u) is
  // the least double s with fl(s / T) >= u (division is monotone in s), so the
  // probes need no division and no clamp (the pinned last weight, W = 1 >= u,
  // is never a probe of a lower-bound bisection: m < hi always).
  if (Nf > 0 && T > 0.0 && T < dinf()) {
    // every thread takes draws i = tid, tid + 256, ... of the filter: u lands in
    // this tile iff P_r < s*(u) <= P_{r+1} (u in (W_end(r-1), W_end(r)]); the
    // first tile takes everything below, the last everything above
    const int nch = (len + K_TABLE - 1) / K_TABLE;
    for (int i = threadIdx.x; i < (int)Nf; i += THREADS) {
      const double sx = s_star(su[i], T);
      if (!((r == 0 || Pr < sx) && (r == a.ntt - 1 || sx <= Pnext))) continue;
      // the chunk: first chunk whose last S is >= s*(x) (the tile's last
      // chunk otherwise), then the entry inside it
      int clo = 0, chi = nch - 1;
      while (clo < chi) {
        const int m = (clo + chi) >> 1;
        if (s_cend[m] < sx) clo = m + 1;
        else chi = m;
      }
      const double Rc = s_R[clo >> 5], Qc = sQ[clo];
      const int cb = clo * K_TABLE;
      int lo = cb, hi = min(cb + K_TABLE, len) - 1;
      while (lo < hi) {
        const int m = (lo + hi) >> 1;
        const double S = __dadd_rn(Pr, __dadd_rn(Rc, __dadd_rn(Qc, sw[m])));
        if (S < sx) lo = m + 1;
        else hi = m;
      }
      a.out[f * Nf + i] = j0 + lo;
    }
  }
  STAMP(5);
  if (a.Wout) {
    for (int j = threadIdx.x; j < len; j += THREADS) {
      const int c = j / K_TABLE;
      const double S = __dadd_rn(Pr, __dadd_rn(s_R[c >> 5], __dadd_rn(sQ[c], sw[j])));
      a.Wout[f * Mf + j0 + j] = (j0 + j == Mf - 1) ? 1.0 : fmin(__ddiv_rn(S, T), 1.0);
    }
  }
}

}  // namespace drs

using namespace drs;

#ifdef DRS_PHASE_TIMING
extern "C" int dr_debug_phase_times_batched(unsigned long long* host, int n) {
  return cudaMemcpyFromSymbol(host, g_phase, sizeof(unsigned long long) * (size_t)n) == cudaSuccess ? 0 : -1;
}
#endif

extern "C" int dr_resample_batched(const double* w, int64_t B, int64_t Mf, int64_t Nf,
                                   uint64_t* keys, int32_t advance, double* W, double* U,
                                   int64_t* out, int32_t* status, void* stream) {
  if (B < 0 || Mf < 1 || Nf < 0 || !status) return DRS_ERR_ARG;
  if (B > 0 && (!w || !keys || (Nf > 0 && !out))) return DRS_ERR_ARG;
  if ((uintptr_t)w & 7) return DRS_ERR_ALIGN;
  const int ntt = (int)cdiv(Mf, TS_TABLE);
  const int ntu = (int)cdiv(Nf + 1, TS_UNIF);
  // su holds N_f + 1 doubles and, first, the Philox words of a one-tile draw
  const size_t smem = (size_t)(TS_TABLE + THREADS + ((Nf + 1 + 8 + 15) & ~(int64_t)15)) * 8;
  if (ntt > MAX_TT || ntu > MAX_UT || smem > (size_t)(227 * 1024 - 1024)) return DRS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(status, 0, sizeof(int32_t), st) != cudaSuccess) return DRS_ERR_LAUNCH;
  if (B == 0) return DRS_OK;
  static SmemLimit lim;  // raised once per size and device (only launches under graph capture)
  lim.raise((const void*)k_resample_batched, smem);
  // U: the caller's buffer, else stream-ordered scratch (graph-capturable)
  double* Ub = U;
  if (!Ub && Nf > 0 && cudaMallocAsync((void**)&Ub, sizeof(double) * (size_t)(B * Nf), st) != cudaSuccess)
    return DRS_ERR_LAUNCH;
  BatchedArgs a{w, B, Mf, Nf, keys, advance, W, Ub, Ub, out, status, ntt, ntu};
  if (Nf > 0) {
    const size_t usmem = (size_t)((Nf + 1 + 8 + 15) & ~(int64_t)15) * 8;
    static SmemLimit ulim;
    ulim.raise((const void*)k_batched_uniforms, usmem);
    if (ntu == 1) {
      const unsigned g = (unsigned)cdiv(B, UW_FILTERS), t = UW_FILTERS * LANES;
      switch ((int)cdiv(Nf + 1, 2 * LANES)) {
        case 1: k_batched_uniforms_warp<1><<<g, t, 0, st>>>(a, Ub); break;
        case 2: k_batched_uniforms_warp<2><<<g, t, 0, st>>>(a, Ub); break;
        case 3: k_batched_uniforms_warp<3><<<g, t, 0, st>>>(a, Ub); break;
        case 4: k_batched_uniforms_warp<4><<<g, t, 0, st>>>(a, Ub); break;
        case 5: k_batched_uniforms_warp<5><<<g, t, 0, st>>>(a, Ub); break;
        case 6: k_batched_uniforms_warp<6><<<g, t, 0, st>>>(a, Ub); break;
        case 7: k_batched_uniforms_warp<7><<<g, t, 0, st>>>(a, Ub); break;
        default: k_batched_uniforms_warp<8><<<g, t, 0, st>>>(a, Ub); break;
      }
    } else {
      k_batched_uniforms<<<(unsigned)B, THREADS, usmem, st>>>(a, Ub);
    }
    if (cudaGetLastError() != cudaSuccess) return DRS_ERR_LAUNCH;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(B * ntt));
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)ntt;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap the uniforms' tail
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = Nf > 0 ? 2 : 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_resample_batched, a);
  if (!U && Nf > 0 && cudaFreeAsync(Ub, st) != cudaSuccess) return DRS_ERR_LAUNCH;
  return e == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}
