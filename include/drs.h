/*
 * drs.h -- C ABI of libdrs.so, the B200 (sm_100a) multinomial-resampling
 * library behind the paper_2604_01356_b200 package.
 *
 * Every entry point is extern "C", takes plain device pointers, sizes and a
 * cudaStream_t passed as void*, never allocates, never synchronises, and is
 * stream-ordered on the caller's stream.  Scratch comes from a caller-owned
 * workspace sized by dr_workspace_bytes() and initialised once with
 * dr_workspace_init().  A workspace serves one stream at a time.
 *
 * Return value: 0 on success, a negative DRS_ERR_* on bad arguments or a
 * launch failure (dr_strerror).  Data-dependent conditions -- the ones the
 * reference reports as ValueError -- are OR-ed into a device int32 status
 * word (DRS_ST_* bits) that the caller reads only where the reference would
 * raise.
 *
 * Each function names the reference interface it replaces
 * (/root/reference/pkg/src/dacresample/<file>:<line>).
 */
#ifndef DRS_H
#define DRS_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --- geometry of the device scan association --- */
#define DRS_SCAN_LANES 32
#define DRS_SCAN_WARPS 8
#define DRS_SCAN_K_TABLE 33 /* elements per lane chunk, table scans   */
#define DRS_SCAN_K_UNIF 2   /* elements per lane chunk, spacing scans */
#define DRS_SCAN_GROUP 32   /* tiles per group of the tile chain          */
#define DRS_INDEX_FANOUT 16
#define DRS_INDEX_MAX_LEVELS 12

/* --- return codes --- */
#define DRS_OK 0
#define DRS_ERR_ARG (-1)       /* invalid size / null pointer               */
#define DRS_ERR_WORKSPACE (-2) /* workspace too small                       */
#define DRS_ERR_LAUNCH (-3)    /* CUDA launch error (cudaGetLastError)      */
#define DRS_ERR_ALIGN (-4)     /* pointer not aligned as documented         */
#define DRS_ERR_MODE (-5)      /* unknown mode                              */

/* --- status bits (device int32) --- */
#define DRS_ST_INVALID_WEIGHT 0x1   /* cdf.py:74-75  "invalid weight"            */
#define DRS_ST_DEGENERATE 0x2       /* cdf.py:77-78  "degenerate distribution"   */
#define DRS_ST_ACCUM_OVERFLOW 0x4   /* cdf.py:83-84  "accumulation overflow"     */
#define DRS_ST_NOT_SORTED 0x8       /* samplers.py:74-75 "input not sorted"      */
#define DRS_ST_OUT_OF_SUPPORT 0x10  /* samplers.py:72-73 "uniforms must lie in (0, 1]" */
#define DRS_ST_REPAIRED 0x20        /* randkit.py:95-100 repair pass taken       */
#define DRS_ST_NONFINITE 0x40       /* cdf.py:35-36 (WeightTable) "invalid weight" */
#define DRS_ST_DECREASING 0x80      /* cdf.py:37-38 "non-decreasing from >= 0"   */
#define DRS_ST_TOP_NOT_ONE 0x100    /* cdf.py:39-40 "must end at exactly 1"      */
#define DRS_ST_SHARD_CAPACITY 0x200 /* sharded sampling: a rank's U / index window was too small (re-run full) */
#define DRS_ST_SHARD_WINDOW 0x400   /* sharded sampling: a repair chain may start before the regenerated tiles (re-run full) */

/* --- workspace ops for dr_workspace_bytes --- */
#define DRS_OP_TABLE 1
#define DRS_OP_SORTED 2

/* --- dac modes --- */
#define DRS_DAC_AUTO 0   /* merge when M <= tau*N, else index search          */
#define DRS_DAC_MERGE 1  /* W-tiled merge (reads all of W; north-star recast) */
#define DRS_DAC_SEARCH 2 /* per-u 16-ary index search                         */

const char *dr_version(void);
const char *dr_strerror(int code);
/* 1 when the device can dereference `p` at the same address (device memory,
 * or pinned host memory under unified addressing, which the search kernels
 * then write directly); 0 otherwise. */
int dr_device_accessible(const void *p);
/* cudaStreamSynchronize(stream): the host waits for a result written to
 * pinned host memory (0 or DRS_ERR_LAUNCH) */
int dr_stream_synchronize(void *stream);
/* writes LANES, WARPS, K_TABLE, K_UNIF, FANOUT, GROUP into g[0..5] */
void dr_scan_geometry(int32_t g[6]);

size_t dr_workspace_bytes(int op, int64_t M, int64_t N, int64_t B);
int dr_workspace_init(void *ws, size_t ws_bytes, void *stream);

/* doubles of the index buffer `idx` of an M-entry table: the 16-ary search
 * levels (none if M <= 16), the top guide, then the table header -- four
 * doubles {T, deferred, 0, 0} -- and one {C_g, D_t} pair per table tile of
 * DRS_SCAN_LANES * DRS_SCAN_WARPS * DRS_SCAN_K_TABLE entries.
 *
 * A table is a value array V[M] (the `W` argument of every search) plus idx.
 * "Direct" tables (dr_build_table, dr_build_index) hold the cumulative
 * weights in V.  "Deferred" tables (dr_build_table_deferred) hold the
 * in-tile chained sums L of the single-pass build in V; their cumulative
 * weights are W_j = fl((C_g + (D_t + L_j)) / T), bit-identical to
 * dr_build_table's W, and every search compares C_g + (D_t + L_j) with the
 * least s for which fl(s / T) >= u.  The searches read
 * the header, so both kinds go through the same entry points; idx may be
 * NULL only for a direct table with M <= 16. */
int64_t dr_index_entries(int64_t M);

/* build_weight_table (cdf.py:59-89): w[M] raw weights -> W[M] cumulative
 * weights with W[M-1] == 1 exactly, idx[dr_index_entries(M)] search index.
 * status gets INVALID_WEIGHT / DEGENERATE / ACCUM_OVERFLOW.  W and w must be
 * 16-byte aligned. */
int dr_build_table(const double *w, int64_t M, double *W, double *idx, int32_t *status,
                   void *ws, size_t ws_bytes, void *stream);

/* build_weight_table (cdf.py:59-89) in ONE pass over w (16 bytes per entry
 * instead of 24): a deferred table (see dr_index_entries) with the same
 * cumulative weights as dr_build_table; V[M] gets the in-tile sums, idx the
 * index (levels hold W), the header and the tile pairs.  Status as
 * dr_build_table.  w, V and idx must be 16-byte aligned. */
int dr_build_table_deferred(const double *w, int64_t M, double *V, double *idx, int32_t *status,
                            void *ws, size_t ws_bytes, void *stream);

/* dr_build_table_log (below) as a deferred table: log-weights read once,
 * the table written once, w never stored. */
int dr_build_table_log_deferred(const double *logw, int64_t M, double *V, double *idx, int32_t *status,
                                void *ws, size_t ws_bytes, void *stream);

/* WeightTable.cum (cdf.py:20-30) of any table: W[j] = the cumulative weight
 * (a copy of V for a direct table, formed for a deferred one). */
int dr_table_materialize(const double *V, const double *idx, int64_t M, double *W, void *stream);

/* The fused weight producer: the table of
 * w = exp(logw - max(logw)) -- weightgen.py:152-153 (engmf_weights' shift and
 * exp) followed by build_weight_table (cdf.py:59-89) -- without writing w:
 * a max reduction, then both table passes form w in shared memory with the
 * device exp (oracle/drs_ref_exp twin).  A NaN log-weight gives INVALID_WEIGHT. */
int dr_build_table_log(const double *logw, int64_t M, double *W, double *idx, int32_t *status,
                       void *ws, size_t ws_bytes, void *stream);

/* WeightTable.__init__ validation (cdf.py:31-42) of a caller-supplied
 * cumulative array: NONFINITE / DECREASING / TOP_NOT_ONE. */
int dr_validate_table(const double *W, int64_t M, int32_t *status, void *stream);

/* search index of an existing table (what dr_build_table writes as a side product) */
int dr_build_index(const double *W, int64_t M, double *idx, void *stream);

/* RngStream.uniforms (randkit.py:47-55): k draws of the numpy-Philox4x64-10
 * stream (key k0,k1) starting at raw draw `offset`, as doubles in (0,1). */
int dr_uniforms(uint64_t k0, uint64_t k1, uint64_t offset, int64_t k, double *u, void *stream);

/* sorted_uniforms (randkit.py:70-101): n+1 draws from `offset` -> spacings
 * -log u -> chained scan -> U[i] = Z[i]/Z[n], with the exact collapse
 * repair (randkit.py:104-116).  status gets REPAIRED when it ran. */
int dr_sorted_uniforms(uint64_t k0, uint64_t k1, uint64_t offset, int64_t n, double *U,
                       int32_t *status, void *ws, size_t ws_bytes, void *stream);

/* same, with the n+1 underlying uniforms supplied (duck-typed host streams,
 * e.g. the reference tests' ReplayStream) */
int dr_sorted_uniforms_from(const double *raw, int64_t n, double *U, int32_t *status,
                            void *ws, size_t ws_bytes, void *stream);

/* _binary_kernel (samplers.py:93-97): out[i] = first j with W[j] >= u[i]
 * (clamped to M-1), any order of u.  idx from dr_build_table/dr_build_index;
 * W must be 32-byte aligned. */
int dr_match_binary(const double *W, const double *idx, int64_t M, const double *u,
                    int64_t N, int64_t *out, void *stream);

/* binary_sampler (samplers.py:238-252) fused: draws N uniforms from the
 * stream at `offset` and searches them, output in draw order. */
int dr_sample_binary(const double *W, const double *idx, int64_t M, uint64_t k0, uint64_t k1,
                     uint64_t offset, int64_t N, int64_t *out, void *stream);

/* dac_sampler (samplers.py:262-266) in one call: sorted uniforms from the
 * stream (k0,k1) at `offset` -- or at *offset_dev when offset_dev is non-NULL,
 * which is then advanced by N+1 on the device (CUDA-graph replayable) --
 * then the divide-and-conquer search.  For N+1 <= 1024 x (co-resident CTAs)
 * and mode SEARCH/AUTO-sparse this is ONE cooperative kernel; otherwise the
 * two-pass sorted uniforms followed by dr_match_dac.  U[N] receives the
 * sorted uniforms, out[N] the indices, status REPAIRED when the repair ran. */
int dr_sample_dac(const double *W, const double *idx, int64_t M, uint64_t k0, uint64_t k1,
                  uint64_t offset, uint64_t *offset_dev, int64_t N, double *U, int64_t *out,
                  int32_t *status, int32_t mode, void *ws, size_t ws_bytes, void *stream);

/* dr_sample_dac for a caller that waits for the result at once (a host
 * result: out in pinned host memory, numpy returned), then
 * cudaStreamSynchronize(stream).  The single-kernel launch goes through a
 * one-node CUDA graph cached per (device, stream, grid) and re-parameterised
 * per call: ~2 us less host time than the cooperative launch, ~1.6 us more
 * between events on the device, so the asynchronous dr_sample_dac keeps the
 * direct launch.  Same results and status as dr_sample_dac. */
int dr_sample_dac_sync(const double *W, const double *idx, int64_t M, uint64_t k0, uint64_t k1,
                       uint64_t offset, uint64_t *offset_dev, int64_t N, double *U, int64_t *out,
                       int32_t *status, int32_t mode, void *ws, size_t ws_bytes, void *stream);

/* dr_sample_dac followed by the step after resampling (the
 * reference leaves it to the caller as states[idx]): gout[i][0..d) =
 * states[out[i] / divisor][0..d), states row-major K x d fp64.  In the
 * single-kernel regime the rows are copied from the indices still in
 * registers (no re-read of out[]); otherwise a gather kernel follows the
 * match on the stream.  DRS_ERR_ARG unless (M - 1) / divisor < K. */
int dr_sample_dac_gather(const double *W, const double *idx, int64_t M, uint64_t k0, uint64_t k1,
                         uint64_t offset, uint64_t *offset_dev, int64_t N, double *U, int64_t *out,
                         const double *states, int64_t K, int64_t d, int64_t divisor, double *gout,
                         int32_t *status, int32_t mode, void *ws, size_t ws_bytes, void *stream);

/* dr_sample_dac with the N+1 underlying uniforms supplied (raw[N+1], a
 * duck-typed host stream such as the reference tests' ReplayStream). */
int dr_sample_dac_from(const double *W, const double *idx, int64_t M, const double *raw, int64_t N,
                       double *U, int64_t *out, int32_t *status, int32_t mode, void *ws,
                       size_t ws_bytes, void *stream);

/* ccf_sampler (samplers.py:255-259): sorted uniforms then the streaming merge. */
int dr_sample_ccf(const double *W, const double *idx, int64_t M, uint64_t k0, uint64_t k1, uint64_t offset,
                  uint64_t *offset_dev, int64_t N, double *U, int64_t *out, int32_t *status,
                  void *ws, size_t ws_bytes, void *stream);

/* binary_sampler with a device-resident stream position (*offset_dev, advanced
 * by N) and the top index levels staged in shared memory. */
int dr_sample_binary_dev(const double *W, const double *idx, int64_t M, uint64_t k0, uint64_t k1,
                         uint64_t offset, uint64_t *offset_dev, int64_t N, int64_t *out,
                         void *stream);

/* _ccf_kernel (samplers.py:100-107) for sorted U: W streamed once through
 * shared memory by TMA bulk copies, each tile merged with its U range. */
int dr_match_ccf(const double *W, const double *idx, int64_t M, const double *U, int64_t N, int64_t *out,
                 void *stream);

/* _dac_kernel (samplers.py:110-146) for sorted U; mode DRS_DAC_*. */
int dr_match_dac(const double *W, const double *idx, int64_t M, const double *U, int64_t N,
                 int64_t *out, int32_t mode, void *stream);

/* _check_sorted_open (samplers.py:69-75): OUT_OF_SUPPORT / NOT_SORTED */
int dr_check_sorted_open(const double *U, int64_t N, int32_t *status, void *stream);

/* upper_bound_search / _upper_bound_nb (cdf.py:92-126, samplers.py:81-90):
 * bisection on [lo,hi] with the reference's clamp-to-hi semantics;
 * out[0] = index, out[1] = number of probes (OpStats.probes). */
int dr_lower_bound_range(const double *W, int64_t lo, int64_t hi, double x, int64_t out[2],
                         void *stream);

/* Batched independent filters (config 4; the reference's per-filter loop
 * over build_weight_table + dac_sampler): w[B][Mf] raw weights, keys[B][3]
 * (k0, k1, draw offset per filter) -> out[B][Nf]; U[B][Nf] and W[B][Mf]
 * are written when non-NULL (U is stream-ordered scratch otherwise).  With
 * advance != 0 each filter's draw offset is moved forward by Nf + 1 on the
 * device (graph-replayable).  Two launches: the uniforms of every filter,
 * then one thread-block cluster per filter (one CTA per 8448-weight tile,
 * tile staged in shared memory by TMA, tile totals exchanged through
 * distributed shared memory).  status gets the OR over filters.  Needs
 * Mf <= 8 x 8448 and Nf + 1 <= 8 x 512. */
int dr_resample_batched(const double *w, int64_t B, int64_t Mf, int64_t Nf, uint64_t *keys,
                        int32_t advance, double *W, double *U, int64_t *out, int32_t *status,
                        void *stream);

/* W-sharded table (config 5).
 * Step 1 on every rank: local chained scan of the rank's shard.
 *   S[Mg] local prefix sums, *Tg (device) = local total.  */
int dr_shard_scan(const double *w_shard, int64_t Mg, double *S, double *Tg, int32_t *status,
                  void *ws, size_t ws_bytes, void *stream);
/* Step 2 after an all-gather of the G totals (device array totals[G]):
 * W[j] = min((O_g + S[j]) / T, 1) in place, O_g and T folded in rank order;
 * the last rank pins its last entry to 1.  Also builds idx of the shard. */
int dr_shard_finalize(double *S_to_W, int64_t Mg, const double *totals, int32_t G, int32_t g,
                      double *idx, void *stream);
/* Step 3: the slice of the (replicated, identical on every rank) sorted U
 * that lands in shard g, as a range8 (layout below) over the full U:
 * range8[0] = #(U <= fl(O_g/T)) (0 for g = 0), range8[1] = #(U <= fl(O_{g+1}/T))
 * (N for the last rank), range8[4] = range8[5] = 0 (U and out are full-length). */
/* The single-pass shard build (16 bytes per entry): dr_shard_scan_deferred
 * writes the shard's in-tile sums to V[Mg], its level-1 index entries and
 * tile pairs to idx[dr_index_entries(Mg)] and its total to *Tg; after the
 * caller's all-gather of the G totals, dr_shard_finalize_deferred writes the
 * header {T, 2, O_g, g == G-1} and the index levels of W -- no pass over the
 * shard's values.  The shard's W (dr_table_materialize) is bit-identical to
 * dr_shard_finalize's. */
int dr_shard_scan_deferred(const double *w_shard, int64_t Mg, double *V, double *idx, double *Tg,
                           int32_t *status, void *ws, size_t ws_bytes, void *stream);
int dr_shard_finalize_deferred(int64_t Mg, const double *totals, int32_t G, int32_t g, double *idx,
                               void *stream);

int dr_shard_range(const double *U, int64_t N, const double *totals, int32_t G, int32_t g,
                   int64_t *range8, void *stream);
/* Step 4: indices of the rank's slice.  range8 (device int64[8]):
 *   [0] i0, [1] i1   the slice [i0, i1) of the N sorted u's routed to shard g
 *   [2] ta, [3] tb   first / last regenerated spacing tile (dr_shard_unif_local)
 *   [4] ubase        global index of U_win[0]
 *   [5] obase        global index of out_win[0]
 *   [6] flags        window overflow / unsafe repair window (device)
 * out_win[i - obase] = shard_start + lower bound of U_win[i - ubase] in the
 * shard's W, for i0 <= i < i1. */
int dr_shard_match(const double *W, const double *idx, int64_t Mg, int64_t shard_start,
                   const double *U_win, int64_t N, const int64_t *range8, int64_t *out_win,
                   void *stream);

/* Sharded sampling without replicating U.
 * Step A on every rank: spacing tiles [t0, t1) of the n+1 spacings of the
 * stream (k0, k1) at `offset` (rank g: t0 = nt g / G, t1 = nt (g+1) / G,
 * nt = ceil((n+1) / (LANES*WARPS*K_UNIF))): agg[t1-t0] tile totals and
 * zmin[t1-t0] spacing minima.  The caller all-gathers them (or every rank
 * computes all nt tiles itself: the zero-communication mode). */
int dr_shard_unif_totals(uint64_t k0, uint64_t k1, uint64_t offset, int64_t n, int64_t t0, int64_t t1,
                         double *agg, double *zmin, void *stream);
/* Step B: from all nt tile totals (agg_all) and nz spacing minima, fold the
 * tile chain, find the tiles holding this rank's u's (those in
 * (fl(O_g/T), fl(O_{g+1}/T)] of the table totals), regenerate them plus the
 * tile before (a repair chain entering the slice starts there), repair
 * collapses and write them into the window U_win[ucap] (U_win[0] = the u just
 * before the window); range8 as above, with obase = i0 and the index window
 * of the caller's capacity ocap.  A window too small for the slice, or a
 * repair chain that may start before the regenerated tiles, sets
 * SHARD_CAPACITY / SHARD_WINDOW in status and an empty slice: re-run with
 * full != 0 (every tile regenerated, ucap >= n + 1, ocap >= n).
 * U values are bit-identical to dr_sorted_uniforms on the slice. */
int dr_shard_unif_local(uint64_t k0, uint64_t k1, uint64_t offset, int64_t n, const double *agg_all,
                        const double *zmin, int64_t nz, const double *totals, int32_t G, int32_t g,
                        double *U_win, int64_t ucap, int64_t ocap, int32_t full, int64_t *range8,
                        int32_t *status, void *ws, size_t ws_bytes, void *stream);

/* --- either side of the path --- */

/* The step after resampling: out[i][0..d) =
 * states[idx[i] / divisor][0..d) for a row-major states[K][d] (divisor = N_Y
 * maps an EnGMF component index (particle, center) to its particle).
 * status gets OUT_OF_SUPPORT for an index outside [0, K*divisor). */
int dr_gather_rows(const double *states, int64_t K, int64_t d, const int64_t *idx, int64_t N,
                   int64_t divisor, double *out, int32_t *status, void *stream);

/* np.bincount(idx, minlength=M) (bench.py:241): counts[M] (zeroed here);
 * status gets OUT_OF_SUPPORT for an index outside [0, M). */
int dr_histogram(const int64_t *idx, int64_t N, int64_t M, uint64_t *counts, int32_t *status,
                 void *stream);

/* chi_square_statistic(counts, n * table.weights()) (bench.py:221-225,
 * cdf.py:51-53) with a fixed reduction order; *out on the device. */
size_t dr_chi_square_workspace(int64_t M);
int dr_chi_square(const uint64_t *counts, const double *W, int64_t M, int64_t n, double *out, void *ws,
                  size_t ws_bytes, void *stream);

/* OpStats of the reference's instrumented twins (samplers.py:40-46,
 * 178-188, 213-232, 249-252), computed exactly from a finished match:
 * kind 0 dac, 1 ccf, 2 binary; u[N] the matched uniforms (sorted for dac /
 * ccf, draw order for binary) and out[N] their lower bounds in W[M].
 * counts[3] (device, zeroed here) = {comparisons, probes, max_depth}. */
int dr_op_counts(int32_t kind, const double *W, int64_t M, const double *u, int64_t N, const int64_t *out,
                 uint64_t *counts, void *stream);

#ifdef __cplusplus
}
#endif
#endif
