/*
 * drs_oracle.h -- CPU oracle for the multinomial-resampling hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it, and only as the checker or as the
 * timed CPU baseline.  The product path (paper_2604_01356_b200) never
 * links, imports or calls this code and fails loudly without its CUDA
 * library.
 *
 * Two families of functions live here:
 *
 *  drs_port_*  -- plain-C restatement of the reference algorithm
 *                 (/root/reference/pkg/src/dacresample, cited per function)
 *                 with the reference's own association: numpy's sequential
 *                 cumsum, the numba bisection / cursor / explicit-stack
 *                 divide-and-conquer kernels.  Pinned against golden vectors
 *                 produced by the reference itself (tests/golden/).
 *                 Used as the CPU baseline ("kind": "port").
 *
 *  drs_ref_*   -- the same algorithms with the DEVICE's association for the
 *                 two fp64 scans (the chained three-level scan described in
 *                 DESIGN.md section 4), so that every value the GPU computes
 *                 has a bit-exact CPU twin.  Only the scan association
 *                 differs from drs_port_*; the search semantics are shared.
 */
#ifndef DRS_ORACLE_H
#define DRS_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* scan geometry of the device association (must equal dr_scan_geometry()) */
#define DRS_REF_LANES 32
#define DRS_REF_WARPS 8
#define DRS_REF_K_TABLE 33
#define DRS_REF_K_UNIF 2
#define DRS_REF_FANOUT 16
#define DRS_REF_GROUP 32 /* tiles per group of the tile chain */
#define DRS_REF_TABLE_TILE ((int64_t)DRS_REF_WARPS * DRS_REF_LANES * DRS_REF_K_TABLE)

/* status bits (same values as include/drs.h) */
#define DRS_REF_ST_INVALID_WEIGHT 0x1
#define DRS_REF_ST_DEGENERATE 0x2
#define DRS_REF_ST_ACCUM_OVERFLOW 0x4
#define DRS_REF_ST_REPAIRED 0x20

/* ---- random numbers (numpy Philox4x64-10 convention) ---- */
void drs_ref_philox4x64_10(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]);
uint64_t drs_ref_raw_draw(uint64_t k0, uint64_t k1, uint64_t d);
double drs_ref_u01(uint64_t raw);
void drs_ref_uniforms(uint64_t k0, uint64_t k1, uint64_t offset, int64_t k, double *u);
double drs_ref_log(double x);
void drs_ref_neglog_array(const double *u, int64_t n, double *z);

/* ---- device-association scans ---- */
void drs_ref_chain_scan(const double *x, int64_t n, int K, double *S, double *total);
double drs_ref_exp(double x);
void drs_ref_exp_array(const double *x, int64_t n, double *y);
int drs_ref_build_table_log(const double *lw, int64_t M, double *W);
int drs_ref_build_table(const double *w, int64_t M, double *W);
int drs_ref_sorted_from_z(const double *z, int64_t n, double *U);
int drs_ref_sorted_uniforms(uint64_t k0, uint64_t k1, uint64_t offset, int64_t n, double *U);
int drs_ref_sorted_uniforms_from(const double *raw, int64_t n, double *U);
int64_t drs_ref_index_entries(int64_t M);
int64_t drs_ref_search_entries(int64_t M);
int drs_ref_build_table_deferred(const double *w, int64_t M, double *V, double *idx, double *Wout);
int drs_ref_index_l1_local(const double *V, int64_t M, double *idx);
void drs_ref_build_index(const double *W, int64_t M, double *idx);
int drs_ref_build_table_sharded(const double *w, int64_t M, int G, double *W,
                                double *shard_totals);
int drs_ref_resample_batched(const double *w, int64_t B, int64_t Mf, int64_t Nf,
                             const uint64_t *keys, double *W, double *U, int64_t *out);

/* ---- reference semantics (numba kernels, samplers.py) ---- */
double drs_port_total(const double *w, int64_t M);
int drs_port_build_table(const double *w, int64_t M, double *W);
int64_t drs_port_upper_bound(const double *cum, int64_t lo, int64_t hi, double x);
void drs_port_match_binary(const double *W, int64_t M, const double *u, int64_t N, int64_t *out);
void drs_port_match_ccf(const double *W, int64_t M, const double *U, int64_t N, int64_t *out);
int drs_port_match_dac(const double *W, int64_t M, const double *U, int64_t N, int64_t *out);
void drs_port_repair_open_strict(double *u, int64_t n);
int drs_port_sorted_from_z(double *z, int64_t n, double *U);
int drs_port_sorted_uniforms(uint64_t k0, uint64_t k1, uint64_t offset, int64_t n, double *U);
int drs_port_sampler(int which, const double *W, int64_t M, uint64_t k0, uint64_t k1,
                     uint64_t offset, int64_t N, double *scratch, int64_t *out);
double drs_port_throughput(int which, const double *W, int64_t M, int64_t N, int threads,
                           int calls_per_thread, uint64_t k0, uint64_t k1);
double drs_port_batched_throughput(const double *w, int64_t B, int64_t Mf, int64_t Nf, int threads,
                                   int reps, uint64_t k0, uint64_t k1);

#ifdef __cplusplus
}
#endif
#endif
