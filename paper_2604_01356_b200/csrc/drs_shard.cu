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
int launch_table_levels_from_aux(int64_t M, double* idx, cudaStream_t st);  // drs_scan.cu
int launch_index_sm(const double* W, const double* idx, int64_t M, const double* u, int64_t N, int64_t* out,
                    cudaStream_t st, const int64_t* rng, int64_t shift);
void launch_chain(const ScanWS& s, int64_t nt, int mode, int32_t* status, double* total, cudaStream_t st);
int64_t ws_capacity_tiles(size_t ws_bytes);
ScanWS carve_ws(void* ws, size_t ws_bytes);

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

// the header of a deferred shard {T, mode 1|2 (+4), O_g, pin}: S = O_g + (C + (D + L)),
// W = min(S / T, 1), only the last shard's last entry pinned to 1
__global__ void k_shard_header(const double* __restrict__ totals, int G, int g, double* __restrict__ aux, int l1) {
  double Og, Og1, T;
  fold_offsets(totals, G, g, Og, Og1, T);
  aux[0] = T;
  aux[1] = (double)(TAB_DEFERRED | TAB_SHARD | (l1 ? TAB_L1 : 0));
  aux[2] = Og;
  aux[3] = (g == G - 1) ? 1.0 : 0.0;
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
  if (threadIdx.x >= 2 && threadIdx.x < 8) range[threadIdx.x] = 0;  // full-length U and out
}

__global__ void __launch_bounds__(256) k_shard_match(const double* __restrict__ W,
                                                     const double* __restrict__ idx, IndexDesc d,
                                                     int64_t shard_start, const double* __restrict__ U,
                                                     const int64_t* __restrict__ range,
                                                     int64_t* __restrict__ out) {
  const int64_t a = range[0], b = range[1];
  const double* Ug = U - range[4];  // window -> global index
  int64_t* og = out - range[5];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const TabAux ta = load_aux(idx ? idx + d.aoff : nullptr);
  for (int64_t i = a + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += stride)
    og[i] = shard_start + index_lower_bound(W, idx, d, ta, __ldg(Ug + i));
}

// ---------------------------------------------- sharded sorted uniforms ----
// Sampling over a W-sharded table without replicating U:
//   1. rank g generates spacing tiles [t0, t1) (its 1/G of them): tile totals
//      and spacing minima only (k_unif_tile_totals);
//   2. the caller all-gathers them (one collective per call);
//   3. every rank folds the identical tile chain, finds the tiles holding the
//      u's of its W range (fl(O_g/T), fl(O_{g+1}/T)], regenerates just those
//      tiles into U, repairs collapses there, and counts its slice
//      (dr_shard_unif_local).  Values are bit-identical to dr_sorted_uniforms.
constexpr int64_t TSU = (int64_t)THREADS * K_UNIF;

__global__ void __launch_bounds__(THREADS) k_unif_tile_totals(PhiloxSpacings src, int64_t n, int64_t t0,
                                                             double* __restrict__ agg, double* __restrict__ zmin) {
  __shared__ FoldSmem fs;
  __shared__ unsigned long long s_min;
  __shared__ uint64_t s_words[PhiloxSpacings::SMEM_WORDS];
  if (threadIdx.x == 0) s_min = 0x7FF0000000000000ULL;
  const int64_t t = t0 + blockIdx.x;
  const int64_t e0 = t * TSU + (int64_t)threadIdx.x * K_UNIF;
  double z[K_UNIF];
  src.tile(t, n + 1, src.position(), s_words, z);
  unsigned long long mn = 0x7FF0000000000000ULL;
#pragma unroll
  for (int i = 0; i < K_UNIF; ++i)
    if (e0 + i <= n) mn = min(mn, (z[i] > 0.0) ? (unsigned long long)__double_as_longlong(z[i]) : 0ull);
  double sc = z[0];
#pragma unroll
  for (int i = 1; i < K_UNIF; ++i) sc = __dadd_rn(sc, z[i]);
  block_min_u64(&s_min, mn);
  double Q, R;
  const double A = block_fold(sc, fs, Q, R);
  if (threadIdx.x == 0) {
    agg[blockIdx.x] = A;
    zmin[blockIdx.x] = __longlong_as_double((long long)s_min);
  }
}

__global__ void k_stage_chain(const double* __restrict__ agg_all, const double* __restrict__ zmin, int64_t nz,
                              int64_t nt, ScanWS ws) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += stride) {
    ws.agg[t] = agg_all[t];
    ws.incl[t] = (t < nz) ? zmin[t] : __longlong_as_double(0x7FF0000000000000LL);
  }
}

// u at the last element of tile t: S = C + (D + A) (the tile's inclusive prefix)
__device__ __forceinline__ double tile_end_u(const ScanWS& ws, int64_t t, double total) {
  return __ddiv_rn(__dadd_rn(ws.grp[t / GROUP_TILES], __dadd_rn(ws.incl[t], ws.agg[t])), total);
}

// The rank's window of spacing tiles: a = first tile ending above fl(O_g/T)
// (the slice starts there), c = first tile ending at or above fl(O_{g+1}/T)
// (the slice ends there); the window starts one tile before a, so that a
// collapse chain of the repair (randkit.py:107-111) entering tile a is
// regenerated and repaired from its true start (k_unif_local_finish checks
// that it does not start before the window).  U_win[0] holds the u just
// before the window, then tiles ta .. tb.  full: every tile.
__global__ void k_unif_tile_range(ScanWS ws, int64_t nt, int64_t n, const double* __restrict__ totals, int G,
                                  int g, int64_t* rng, double* U_win, int64_t ucap, int full) {
  double Og, Og1, T;
  fold_offsets(totals, G, g, Og, Og1, T);
  const double lo = fmin(__ddiv_rn(Og, T), 1.0), hi = fmin(__ddiv_rn(Og1, T), 1.0);
  const double total = ws.hdr->total;
  // tiles 0 .. nt-2 end on a u (the last tile holds the final spacing)
  int64_t a = 0, b = nt - 1;  // first t in [0, nt-1) with u_end(t) > lo, else nt-1
  if (g > 0 && !full)
    while (a < b) {
      const int64_t m = (a + b) / 2;
      if (tile_end_u(ws, m, total) > lo) b = m;
      else a = m + 1;
    }
  int64_t c = (g < G - 1 && !full) ? 0 : nt - 1, d = nt - 1;  // first t in [0, nt-1) with u_end(t) >= hi, else nt-1
  if (g < G - 1 && !full)
    while (c < d) {
      const int64_t m = (c + d) / 2;
      if (tile_end_u(ws, m, total) >= hi) d = m;
      else c = m + 1;
    }
  const int64_t ta = a > 0 ? a - 1 : 0;
  const int64_t tb = c > a ? c : a;
  const int64_t ubase = ta * TSU - 1;
  const int64_t end = min((tb + 1) * TSU, n);
  int64_t flags = 0;
  if (end - ubase > ucap) flags |= 1;  // the window does not fit: no tile is regenerated
  rng[2] = ta;
  rng[3] = flags ? ta - 1 : tb;
  rng[4] = ubase;
  rng[6] = flags;
  // the u just before the window (the previous tile's inclusive prefix): the
  // repair's forward pass reads it when the window's first u collapses
  if (ta > 0 && !flags) U_win[0] = tile_end_u(ws, ta - 1, total);
}

__global__ void __launch_bounds__(THREADS) k_unif_pass_range(PhiloxSpacings src, int64_t n, ScanWS ws,
                                                            const int64_t* __restrict__ rng,
                                                            double* __restrict__ U_win) {
  double* U = U_win - rng[4];  // global index -> window
  __shared__ FoldSmem fs;
  __shared__ double s_last[WARPS];
  __shared__ uint64_t s_words[PhiloxSpacings::SMEM_WORDS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double total = ws.hdr->total;
  const bool need = ws.hdr->need != 0u;
  // grid-stride over this rank's tiles [rng[2], rng[3]] (read on the device:
  // no host round trip, no idle CTAs for the other ranks' tiles)
  for (int64_t t = rng[2] + blockIdx.x; t <= rng[3]; t += gridDim.x) {
    const int64_t e0 = t * TSU + (int64_t)threadIdx.x * K_UNIF;
    double z[K_UNIF];
    src.tile(t, n + 1, src.position(), s_words, z);
    double sc[K_UNIF];
    sc[0] = z[0];
#pragma unroll
    for (int i = 1; i < K_UNIF; ++i) sc[i] = __dadd_rn(sc[i - 1], z[i]);
    double Q, R;
    block_fold(sc[K_UNIF - 1], fs, Q, R);
    const double C = ws.grp[t / GROUP_TILES], D = ws.incl[t];
    double u[K_UNIF];
#pragma unroll
    for (int i = 0; i < K_UNIF; ++i) {
      u[i] = __ddiv_rn(__dadd_rn(C, __dadd_rn(D, __dadd_rn(R, __dadd_rn(Q, sc[i])))), total);
      if (e0 + i < n) U[e0 + i] = u[i];
    }
    if (need) {  // collapse sites, exactly as k_unif_pass2
      double prev_lane = __shfl_up_sync(FULL, u[K_UNIF - 1], 1);
      if (lane == 31) s_last[warp] = u[K_UNIF - 1];
      __syncthreads();
      if (lane == 0)
        prev_lane = (warp > 0) ? s_last[warp - 1] : ((t == 0) ? 0.0 : __ddiv_rn(__dadd_rn(C, D), total));
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
    __syncthreads();  // fs / s_last reuse by the next tile
  }
}

// repair inside the window (the backward pass only on the rank holding the
// last tile), the slice counts, the index window, status, counters back to zero
__global__ void k_unif_local_finish(ScanWS ws, int64_t n, int64_t nt, double* U_win, const double* __restrict__ totals,
                                    int G, int g, int64_t* rng, int64_t ocap, int32_t* status) {
  __shared__ int64_t s_flags;
  const int64_t ta = rng[2], tb = rng[3];
  double* U = U_win - rng[4];  // global index -> window
  const int64_t base = ta * TSU, end = min((tb + 1) * TSU, n);
  if (threadIdx.x == 0) {
    int64_t flags = rng[6];
    const uint32_t nsites = ws.hdr->nsites;
    const uint32_t top = ws.hdr->top;
    int32_t st = 0;
    if (!flags && ws.hdr->need && (nsites > 0 || top)) {
      // a chain collapsing at the window's first u may have started in an
      // earlier tile, whose repaired values this rank does not have
      if (ta > 0 && !(U[base] > U[base - 1])) flags |= 4;
      int64_t stop = end;
      repair_sites(U, end, ws, nsites, tb == nt - 1, base, &stop);
      if (ta > 0 && stop == base) flags |= 4;  // the backward pass ran through the window
      st |= DRS_ST_REPAIRED;
    }
    ws.hdr->nsites = 0;
    ws.hdr->top = 0;
    s_flags = flags;
    if (flags & 1) st |= DRS_ST_SHARD_CAPACITY;
    if (flags & 4) st |= DRS_ST_SHARD_WINDOW;
    *status = st;
  }
  __syncthreads();
  const int64_t flags = s_flags;
  double Og, Og1, T;
  fold_offsets(totals, G, g, Og, Og1, T);
  const int warp = threadIdx.x >> 5;
  __shared__ int64_t s_r[2];
  if (flags) {
    if (threadIdx.x < 2) s_r[threadIdx.x] = 0;
  } else if (warp == 0) {
    const int64_t v = (g == 0) ? 0 : base + warp_count_le_s(U + base, end - base, fmin(__ddiv_rn(Og, T), 1.0));
    if ((threadIdx.x & 31) == 0) s_r[0] = v;
  } else if (warp == 1) {
    const int64_t v = (g == G - 1) ? n : base + warp_count_le_s(U + base, end - base, fmin(__ddiv_rn(Og1, T), 1.0));
    if ((threadIdx.x & 31) == 0) s_r[1] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t i0 = s_r[0], i1 = s_r[1];
    int64_t f = flags;
    if (!f && i1 - i0 > ocap) {  // the index window does not fit
      f |= 2;
      *status |= DRS_ST_SHARD_CAPACITY;
    }
    if (f) i1 = i0;  // empty slice: nothing is matched
    rng[0] = i0;
    rng[1] = i1;
    rng[5] = i0;
    rng[6] = f;
  }
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

int dr_shard_finalize_deferred(int64_t Mg, const double* totals, int32_t G, int32_t g, double* idx,
                               void* stream) {
  if (Mg < 1 || !totals || !idx || G < 1 || g < 0 || g >= G) return DRS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const IndexDesc d = make_index_desc(Mg);
  k_shard_header<<<1, 1, 0, st>>>(totals, G, g, idx + d.aoff, d.kt >= 2 ? 1 : 0);
  if (cudaGetLastError() != cudaSuccess) return DRS_ERR_LAUNCH;
  return launch_table_levels_from_aux(Mg, idx, st);
}

int dr_shard_range(const double* U, int64_t N, const double* totals, int32_t G, int32_t g,
                   int64_t* range8, void* stream) {
  int64_t* range = range8;
  if (N < 0 || !totals || !range || G < 1 || g < 0 || g >= G || (N > 0 && !U)) return DRS_ERR_ARG;
  k_shard_range<<<1, 64, 0, (cudaStream_t)stream>>>(U, N, totals, G, g, range);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

int dr_shard_match(const double* W, const double* idx, int64_t Mg, int64_t shard_start,
                   const double* U, int64_t N, const int64_t* range, int64_t* out, void* stream) {
  if (Mg < 1 || !W || !range || (N > 0 && (!U || !out))) return DRS_ERR_ARG;
  // U / out are windows: range[4] / range[5] give their global base (device)
  if ((uintptr_t)W & 31) return DRS_ERR_ALIGN;
  if (N == 0) return DRS_OK;
  const IndexDesc d = make_index_desc(Mg);
  if (d.levels > 0 && !idx) return DRS_ERR_ARG;
  if (d.levels > 0) return launch_index_sm(W, idx, Mg, U, N, out, (cudaStream_t)stream, range, shard_start);
  const int64_t blocks = cdiv(N, 256) < 148 * 16 ? cdiv(N, 256) : 148 * 16;
  k_shard_match<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(W, idx, d, shard_start, U, range, out);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

int dr_shard_unif_totals(uint64_t k0, uint64_t k1, uint64_t offset, int64_t n, int64_t t0, int64_t t1,
                         double* agg, double* zmin, void* stream) {
  if (n < 1 || t0 < 0 || t1 < t0 || !agg || !zmin) return DRS_ERR_ARG;
  if (t1 > cdiv(n + 1, TSU)) return DRS_ERR_ARG;
  if (t1 == t0) return DRS_OK;
  PhiloxSpacings src{k0, k1, offset, nullptr};
  k_unif_tile_totals<<<(unsigned)(t1 - t0), THREADS, 0, (cudaStream_t)stream>>>(src, n, t0, agg, zmin);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

int dr_shard_unif_local(uint64_t k0, uint64_t k1, uint64_t offset, int64_t n, const double* agg_all,
                        const double* zmin, int64_t nz, const double* totals, int32_t G, int32_t g, double* U_win,
                        int64_t ucap, int64_t ocap, int32_t full, int64_t* range8, int32_t* status, void* ws,
                        size_t ws_bytes, void* stream) {
  if (n < 1 || !agg_all || !zmin || nz < 1 || !totals || G < 1 || g < 0 || g >= G || !U_win || ucap < 1 ||
      ocap < 0 || !range8 || !status || !ws)
    return DRS_ERR_ARG;
  const int64_t nt = cdiv(n + 1, TSU);
  if (nt > ws_capacity_tiles(ws_bytes)) return DRS_ERR_WORKSPACE;
  if (nt > (int64_t)8192 * GROUP_TILES) return DRS_ERR_ARG;
  if (full && (ucap < n + 1 || ocap < n)) return DRS_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const ScanWS s = carve_ws(ws, ws_bytes);
  PhiloxSpacings src{k0, k1, offset, nullptr};
  k_stage_chain<<<(unsigned)(cdiv(nt, 256) < 1184 ? cdiv(nt, 256) : 1184), 256, 0, st>>>(agg_all, zmin, nz, nt, s);
  launch_chain(s, nt, 1, nullptr, nullptr, st);
  k_unif_tile_range<<<1, 1, 0, st>>>(s, nt, n, totals, G, g, range8, U_win, ucap, full);
  k_unif_pass_range<<<(unsigned)(nt < 148 * 4 ? nt : 148 * 4), THREADS, 0, st>>>(src, n, s, range8, U_win);
  k_unif_local_finish<<<1, 64, 0, st>>>(s, n, nt, U_win, totals, G, g, range8, ocap, status);
  return cudaGetLastError() == cudaSuccess ? DRS_OK : DRS_ERR_LAUNCH;
}

}  // extern "C"
