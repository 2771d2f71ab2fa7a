/*
 * drs_oracle.c -- CPU oracle for the multinomial-resampling hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see drs_oracle.h).  Compiled with
 * -ffp-contract=off so every + and * is a single IEEE operation; fused
 * multiply-adds appear only where written as fma(), mirroring the device.
 *
 * Reference citations are relative to /root/reference/pkg/src/dacresample.
 */
#include "drs_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------ */
/* Philox4x64-10 in numpy's convention (numpy/random/src/philox):           */
/* key = SeedSequence.generate_state(2, uint64), 256-bit counter starting   */
/* at 0 and pre-incremented, so raw draw d comes from block d/4 evaluated   */
/* at counter d/4 + 1, word d%4.  RngStream (randkit.py:16-62) uses PCG64;  */
/* DESIGN.md section 5 explains the generator change.                      */
/* ------------------------------------------------------------------------ */
#define PH_M0 0xD2E7470EE14C6C93ULL
#define PH_M1 0xCA5A826395121157ULL
#define PH_W0 0x9E3779B97F4A7C15ULL
#define PH_W1 0xBB67AE8584CAA73BULL

void drs_ref_philox4x64_10(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]) {
  uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint64_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += PH_W0;
      k1 += PH_W1;
    }
    unsigned __int128 p0 = (unsigned __int128)PH_M0 * c0;
    unsigned __int128 p1 = (unsigned __int128)PH_M1 * c2;
    uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

uint64_t drs_ref_raw_draw(uint64_t k0, uint64_t k1, uint64_t d) {
  uint64_t ctr[4] = {(d >> 2) + 1, 0, 0, 0}, key[2] = {k0, k1}, out[4];
  if (ctr[0] == 0) ctr[1] = 1; /* carry; unreachable for d < 2^66 */
  drs_ref_philox4x64_10(ctr, key, out);
  return out[d & 3];
}

/* numpy next_double: (raw >> 11) * 2^-53.  The reference redraws an exact
 * 0 (randkit.py:52-54); the device maps it to 2^-54 instead (probability
 * 2^-53 per draw), and so does this oracle. */
double drs_ref_u01(uint64_t raw) {
  uint64_t m = raw >> 11;
  return m ? (double)m * 0x1.0p-53 : 0x1.0p-54;
}

void drs_ref_uniforms(uint64_t k0, uint64_t k1, uint64_t offset, int64_t k, double *u) {
  for (int64_t i = 0; i < k; ++i) u[i] = drs_ref_u01(drs_ref_raw_draw(k0, k1, offset + (uint64_t)i));
}

/* ------------------------------------------------------------------------ */
/* Natural log, restated (argument reduction to m in [sqrt2/2, sqrt2],      */
/* s = f/(2+f), log(1+f) = f - hfsq + s*(hfsq + R(s^2)) with R the atanh    */
/* series 2/3 z + 2/5 z^2 + ... truncated at 11 terms (|z| < 0.0295, so the */
/* tail is below 2^-60 relative).  The device evaluates the identical       */
/* operation sequence with __fma_rn/__dmul_rn/__dadd_rn, so the two agree    */
/* bit for bit; against np.log it agrees to <= 1 ulp (tests pin this).      */
/* ------------------------------------------------------------------------ */
static inline uint64_t dbits(double x) { uint64_t b; memcpy(&b, &x, 8); return b; }
static inline double bitsd(uint64_t b) { double x; memcpy(&x, &b, 8); return x; }

double drs_ref_log(double x) {
  if (!(x > 0.0)) return (x == 0.0) ? -INFINITY : NAN;
  if (x == INFINITY) return INFINITY;
  int k = 0;
  uint64_t b = dbits(x);
  if ((b >> 52) == 0) { /* subnormal */
    x = x * 0x1.0p54;
    b = dbits(x);
    k = -54;
  }
  k += (int)(b >> 52) - 1023;
  double m = bitsd((b & 0x000FFFFFFFFFFFFFULL) | 0x3FF0000000000000ULL);
  if (m > 0x1.6a09e667f3bcdp+0) {
    m = m * 0.5;
    k += 1;
  }
  const double f = m - 1.0;
  const double s = f / (2.0 + f);
  const double z = s * s;
  double R = 2.0 / 23.0;
  R = fma(R, z, 2.0 / 21.0);
  R = fma(R, z, 2.0 / 19.0);
  R = fma(R, z, 2.0 / 17.0);
  R = fma(R, z, 2.0 / 15.0);
  R = fma(R, z, 2.0 / 13.0);
  R = fma(R, z, 2.0 / 11.0);
  R = fma(R, z, 2.0 / 9.0);
  R = fma(R, z, 2.0 / 7.0);
  R = fma(R, z, 2.0 / 5.0);
  R = fma(R, z, 2.0 / 3.0);
  R = R * z;
  /* log x = k ln2 + f - f^2/2 + s (f^2/2 + R); the three large terms are
   * summed exactly with TwoSum and only the small ones are rounded. */
  const double hf = 0.5 * f;                     /* exact */
  const double hfsq = hf * f;
  const double e1 = fma(hf, f, -hfsq);           /* hf*f = hfsq + e1 exactly */
  const double t = s * (hfsq + R);
  const double dk = (double)k;
  const double a = dk * 0x1.62e42feep-1;         /* ln2 high part: exact product */
  const double c = dk * 0x1.a39ef35793c76p-33;   /* ln2 low part */
  double s1 = a + f, bb = s1 - a;                /* TwoSum(a, f) */
  const double r1 = (a - (s1 - bb)) + (f - bb);
  const double mh = -hfsq;
  double s2 = s1 + mh;                           /* TwoSum(s1, -hfsq) */
  bb = s2 - s1;
  const double r2 = (s1 - (s2 - bb)) + (mh - bb);
  const double small = (((t - e1) + c) + r1) + r2;
  return s2 + small;
}

/* exp with the device's operation sequence (drs_common.cuh:dexp) */
double drs_ref_exp(double x) {
  if (x != x) return x;
  if (x > 709.782712893384) return INFINITY;
  if (x < -745.1332191019412) return 0.0;
  const double kd = rint(x * 0x1.71547652b82fep+0);
  double r = fma(-kd, 0x1.62e42fefa39efp-1, x);
  r = fma(-kd, 0x1.abc9e3b39803fp-56, r);
  double p = 1.0 / 6227020800.0; /* e^r: degree-13 Taylor polynomial, Horner with FMAs */
  p = fma(p, r, 1.0 / 479001600.0);
  p = fma(p, r, 1.0 / 39916800.0);
  p = fma(p, r, 1.0 / 3628800.0);
  p = fma(p, r, 1.0 / 362880.0);
  p = fma(p, r, 1.0 / 40320.0);
  p = fma(p, r, 1.0 / 5040.0);
  p = fma(p, r, 1.0 / 720.0);
  p = fma(p, r, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int k = (int)kd;
  if (k > 1023) return (p * 2.0) * bitsd((uint64_t)(1023 + 1023) << 52);
  if (k >= -1022) return p * bitsd((uint64_t)(k + 1023) << 52);
  return (p * bitsd((uint64_t)(k + 54 + 1023) << 52)) * 0x1.0p-54;
}

void drs_ref_exp_array(const double *x, int64_t n, double *y) {
  for (int64_t i = 0; i < n; ++i) y[i] = drs_ref_exp(x[i]);
}

/* build_weight_table(np.exp(logw - logw.max())) (weightgen.py:152-153 +
 * cdf.py:59-89) with the device exp and association; a NaN log-weight makes
 * the max NaN and every weight NaN ("invalid weight"). */
int drs_ref_build_table_log(const double *lw, int64_t M, double *W) {
  double mx = -INFINITY;
  int nan = 0;
  for (int64_t i = 0; i < M; ++i) {
    if (lw[i] != lw[i]) nan = 1;
    else if (lw[i] > mx) mx = lw[i];
  }
  if (nan) mx = NAN;
  double *w = (double *)malloc(sizeof(double) * (size_t)M);
  for (int64_t i = 0; i < M; ++i) w[i] = drs_ref_exp(lw[i] - mx);
  const int st = drs_ref_build_table(w, M, W);
  free(w);
  return st;
}

void drs_ref_neglog_array(const double *u, int64_t n, double *z) {
  for (int64_t i = 0; i < n; ++i) z[i] = -drs_ref_log(u[i]);
}

/* ------------------------------------------------------------------------ */
/* The device's chained scan.                        */
/*   tile t = WARPS*LANES lane chunks of K consecutive elements              */
/*   s      = serial inclusive sum inside the chunk (s = x0; s = s + xi)     */
/*   Q      = serial fold of previous chunk totals inside the warp (from 0)  */
/*   R      = serial fold of previous warp totals inside the tile (from 0)   */
/*   D      = serial fold of previous tile totals inside the group of        */
/*            GROUP tiles (from 0)                                          */
/*   C      = serial fold of previous group totals (from 0)                  */
/*   S      = C + (D + (R + (Q + s)))                                        */
/* Every group boundary value is the next group's base, so S is monotone    */
/* for non-negative inputs and padding zeros are transparent.               */
/* ------------------------------------------------------------------------ */
void drs_ref_chain_scan(const double *x, int64_t n, int K, double *S, double *total) {
  const int64_t TS = (int64_t)DRS_REF_WARPS * DRS_REF_LANES * K;
  const int64_t nt = (n + TS - 1) / TS;
  double C = 0.0, D = 0.0;
  for (int64_t t = 0; t < nt; ++t) {
    if (t > 0 && t % DRS_REF_GROUP == 0) {
      C = C + D;
      D = 0.0;
    }
    double R = 0.0;
    for (int w = 0; w < DRS_REF_WARPS; ++w) {
      double Q = 0.0;
      for (int l = 0; l < DRS_REF_LANES; ++l) {
        const int64_t base = t * TS + (int64_t)(w * DRS_REF_LANES + l) * K;
        double s = 0.0;
        for (int i = 0; i < K; ++i) {
          const int64_t j = base + i;
          const double xi = (j < n) ? x[j] : 0.0;
          s = (i == 0) ? xi : s + xi;
          if (S && j < n) S[j] = C + (D + (R + (Q + s)));
        }
        Q = Q + s;
      }
      R = R + Q;
    }
    D = D + R;
  }
  if (total) *total = C + D;
}

/* build_weight_table (cdf.py:59-89) with the device association: validate,
 * chained scan, divide by T = S[M-1] (so W[M-1] == 1 exactly), clip, pin. */
int drs_ref_build_table(const double *w, int64_t M, double *W) {
  int st = 0;
  for (int64_t j = 0; j < M; ++j)
    if (!(w[j] >= 0.0 && w[j] < INFINITY)) st |= DRS_REF_ST_INVALID_WEIGHT;
  double T;
  drs_ref_chain_scan(w, M, DRS_REF_K_TABLE, W, &T);
  if (T == 0.0) st |= DRS_REF_ST_DEGENERATE;
  if (!(T < INFINITY)) st |= DRS_REF_ST_ACCUM_OVERFLOW;
  for (int64_t j = 0; j < M; ++j) W[j] = fmin(W[j] / T, 1.0);
  W[M - 1] = 1.0;
  return st;
}

/* A deferred table whose top guide sits above level 1 (kt >= 2) keeps its
 * level-1 index entries as in-tile values: level 1 (offset 0) gets V at the
 * 16-entry block ends.  Returns 1 when it did (the header's mode bit 4). */
static void ref_top_guide(int64_t M, int *kt, int64_t *nkt, int *tshift, int64_t *tdoubles);
int drs_ref_index_l1_local(const double *V, int64_t M, double *idx) {
  int kt, tshift;
  int64_t nkt, td;
  ref_top_guide(M, &kt, &nkt, &tshift, &td);
  if (kt < 2) return 0;
  const int64_t n1 = (M + DRS_REF_FANOUT - 1) / DRS_REF_FANOUT;
  for (int64_t m = 0; m < n1; ++m) {
    int64_t p = m * DRS_REF_FANOUT + DRS_REF_FANOUT - 1;
    if (p > M - 1) p = M - 1;
    idx[m] = V[p];
  }
  return 1;
}

/* dr_build_table_deferred (the single-pass table): the same association as
 * drs_ref_chain_scan, split at the tile prefix: V[j] = R + (Q + s) (the
 * in-tile sums), per tile the pair {C_g, D_t}, so that S = C_g + (D_t + V[j]);
 * idx = the index of W = min(S / T, 1), W[M-1] = 1 (drs_ref_build_table's W),
 * then the header {T, 1, 0, 1} and the pairs.  W may be NULL. */
int drs_ref_build_table_deferred(const double *w, int64_t M, double *V, double *idx, double *Wout) {
  const int K = DRS_REF_K_TABLE;
  const int64_t TS = DRS_REF_TABLE_TILE;
  const int64_t nt = (M + TS - 1) / TS;
  int st = 0;
  for (int64_t j = 0; j < M; ++j)
    if (!(w[j] >= 0.0 && w[j] < INFINITY)) st |= DRS_REF_ST_INVALID_WEIGHT;
  double *P = (double *)malloc(sizeof(double) * 2 * (size_t)nt);
  double *W = (double *)malloc(sizeof(double) * (size_t)M);
  double C = 0.0, D = 0.0;
  for (int64_t t = 0; t < nt; ++t) {
    if (t > 0 && t % DRS_REF_GROUP == 0) {
      C = C + D;
      D = 0.0;
    }
    P[2 * t] = C;
    P[2 * t + 1] = D;
    double R = 0.0;
    for (int wp = 0; wp < DRS_REF_WARPS; ++wp) {
      double Q = 0.0;
      for (int l = 0; l < DRS_REF_LANES; ++l) {
        const int64_t base = t * TS + (int64_t)(wp * DRS_REF_LANES + l) * K;
        double s = 0.0;
        for (int i = 0; i < K; ++i) {
          const int64_t j = base + i;
          const double xi = (j < M) ? w[j] : 0.0;
          s = (i == 0) ? xi : s + xi;
          if (j < M) V[j] = R + (Q + s);
        }
        Q = Q + s;
      }
      R = R + Q;
    }
    D = D + R;
  }
  const double T = C + D;
  if (T == 0.0) st |= DRS_REF_ST_DEGENERATE;
  if (!(T < INFINITY)) st |= DRS_REF_ST_ACCUM_OVERFLOW;
  for (int64_t j = 0; j < M; ++j) {
    const int64_t t = j / TS;
    W[j] = fmin((P[2 * t] + (P[2 * t + 1] + V[j])) / T, 1.0);
  }
  W[M - 1] = 1.0;
  drs_ref_build_index(W, M, idx);
  const int l1 = drs_ref_index_l1_local(V, M, idx);
  double *aux = idx + drs_ref_search_entries(M);
  aux[0] = T;
  aux[1] = l1 ? 5.0 : 1.0; /* mode 1: S = C + (D + V); + 4: level 1 holds V */
  aux[2] = 0.0; /* O (shards only) */
  aux[3] = 1.0; /* the last entry pinned to 1 */
  memcpy(aux + 4, P, sizeof(double) * 2 * (size_t)nt);
  if (Wout) memcpy(Wout, W, sizeof(double) * (size_t)M);
  free(P);
  free(W);
  return st;
}

/* repair (randkit.py:104-116): forward nextafter chain, then backward. */
void drs_port_repair_open_strict(double *u, int64_t n) {
  double lo = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (u[i] <= lo) u[i] = nextafter(lo, 1.0);
    lo = u[i];
  }
  double hi = 1.0;
  for (int64_t i = n - 1; i >= 0; --i) {
    if (u[i] >= hi) u[i] = nextafter(hi, 0.0);
    hi = u[i];
  }
}

/* check + repair exactly as randkit.py:95-100 */
static int check_and_repair(double *U, int64_t n, double zmin, double total) {
  if (zmin > 1e-14 * total) return 0;
  int bad = (U[0] <= 0.0) || (U[n - 1] >= 1.0);
  if (!bad && n > 1)
    for (int64_t i = 1; i < n; ++i)
      if (!(U[i] - U[i - 1] > 0.0)) { bad = 1; break; }
  if (bad) {
    drs_port_repair_open_strict(U, n);
    return DRS_REF_ST_REPAIRED;
  }
  return 0;
}

/* sorted_uniforms (randkit.py:70-101) on given spacings z[0..n], device association */
int drs_ref_sorted_from_z(const double *z, int64_t n, double *U) {
  if (n <= 0) return 0;
  double *Z = (double *)malloc(sizeof(double) * (size_t)(n + 1));
  double total, zmin = INFINITY;
  for (int64_t i = 0; i <= n; ++i) zmin = fmin(zmin, z[i]);
  drs_ref_chain_scan(z, n + 1, DRS_REF_K_UNIF, Z, &total);
  for (int64_t i = 0; i < n; ++i) U[i] = Z[i] / total;
  free(Z);
  return check_and_repair(U, n, zmin, total);
}

int drs_ref_sorted_uniforms(uint64_t k0, uint64_t k1, uint64_t offset, int64_t n, double *U) {
  if (n <= 0) return 0;
  double *z = (double *)malloc(sizeof(double) * (size_t)(n + 1));
  drs_ref_uniforms(k0, k1, offset, n + 1, z);
  for (int64_t i = 0; i <= n; ++i) z[i] = -drs_ref_log(z[i]);
  int st = drs_ref_sorted_from_z(z, n, U);
  free(z);
  return st;
}

int drs_ref_sorted_uniforms_from(const double *raw, int64_t n, double *U) {
  if (n <= 0) return 0;
  double *z = (double *)malloc(sizeof(double) * (size_t)(n + 1));
  for (int64_t i = 0; i <= n; ++i) z[i] = -drs_ref_log(raw[i]);
  int st = drs_ref_sorted_from_z(z, n, U);
  free(z);
  return st;
}

/* ------------------------------------------------------------------------ */
/* The search index of a table: level k (k >= 1) holds the last entry of    */
/* every FANOUT^k-block of W, each level padded with +inf to a multiple of  */
/* FANOUT; levels stop once a level has <= FANOUT entries.                  */
/* ------------------------------------------------------------------------ */
/* After the levels comes the top guide (Chen & Asau's guide table over one */
/* level): kt = the lowest level with <= 16384 entries, B = 2^tshift the    */
/* least power of two >= n_kt / 2 (and >= 16), Gt[b] = lower bound of b / B */
/* among level kt's entries (clamped to n_kt - 1) for b = 0 .. B+1, int32   */
/* packed two per double, zero-padded to a multiple of FANOUT doubles.      */
/* Mirrors make_index_desc / k_build_top_guide.                             */
static void ref_top_guide(int64_t M, int *kt, int64_t *nkt, int *tshift, int64_t *tdoubles) {
  int64_t n = M;
  int L = 0;
  *kt = 0;
  *nkt = 0;
  while (n > DRS_REF_FANOUT) {
    n = (n + DRS_REF_FANOUT - 1) / DRS_REF_FANOUT;
    ++L;
    if (!*kt && n <= 16384) {
      *kt = L;
      *nkt = n;
    }
  }
  *tshift = 0;
  *tdoubles = 0;
  if (!*kt) return;
  int sh = 0;
  while (((int64_t)2 << sh) < *nkt) ++sh;
  *tshift = sh < 4 ? 4 : sh;
  const int64_t n32 = ((int64_t)1 << *tshift) + 2;
  *tdoubles = ((n32 + 1) / 2 + DRS_REF_FANOUT - 1) / DRS_REF_FANOUT * DRS_REF_FANOUT;
}

/* levels + top guide: the part of the index the searches descend */
int64_t drs_ref_search_entries(int64_t M) {
  int64_t total = 0, n = M;
  while (n > DRS_REF_FANOUT) {
    n = (n + DRS_REF_FANOUT - 1) / DRS_REF_FANOUT;
    total += (n + DRS_REF_FANOUT - 1) / DRS_REF_FANOUT * DRS_REF_FANOUT;
  }
  int kt, tshift;
  int64_t nkt, td;
  ref_top_guide(M, &kt, &nkt, &tshift, &td);
  return total + td;
}

/* then the table header {T, deferred, 0, 0} and one {C_g, D_t} pair per
 * table tile (mirrors include/drs.h dr_index_entries) */
int64_t drs_ref_index_entries(int64_t M) {
  return drs_ref_search_entries(M) + 4 + 2 * ((M + DRS_REF_TABLE_TILE - 1) / DRS_REF_TABLE_TILE);
}

void drs_ref_build_index(const double *W, int64_t M, double *idx) {
  /* a direct table: header and tile pairs zero */
  for (int64_t e = drs_ref_search_entries(M); e < drs_ref_index_entries(M); ++e) idx[e] = 0.0;
  int64_t n = M, off = 0;
  int64_t span = 1;
  while (n > DRS_REF_FANOUT) {
    n = (n + DRS_REF_FANOUT - 1) / DRS_REF_FANOUT;
    span *= DRS_REF_FANOUT;
    const int64_t padded = (n + DRS_REF_FANOUT - 1) / DRS_REF_FANOUT * DRS_REF_FANOUT;
    for (int64_t b = 0; b < padded; ++b) {
      if (b < n) {
        int64_t j = (b + 1) * span - 1;
        if (j > M - 1) j = M - 1;
        idx[off + b] = W[j];
      } else {
        idx[off + b] = INFINITY;
      }
    }
    off += padded;
  }
  int kt, tshift;
  int64_t nkt, td;
  ref_top_guide(M, &kt, &nkt, &tshift, &td);
  if (!kt) return;
  /* level kt starts where the levels below it end */
  int64_t koff = 0, m = M;
  for (int k = 1; k < kt; ++k) {
    m = (m + DRS_REF_FANOUT - 1) / DRS_REF_FANOUT;
    koff += (m + DRS_REF_FANOUT - 1) / DRS_REF_FANOUT * DRS_REF_FANOUT;
  }
  const double *Lk = idx + koff;
  int32_t *G = (int32_t *)(idx + off);
  const int64_t B = (int64_t)1 << tshift;
  for (int64_t b = 0; b < 2 * td; ++b) {
    if (b > B + 1) {
      G[b] = 0;
      continue;
    }
    const double x = (double)b / (double)B;
    int64_t lo = 0, hi = nkt - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (Lk[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    G[b] = (int32_t)lo;
  }
}

/* W-sharded table (multi-GPU mode): shard g owns
 * [g*M/G, (g+1)*M/G); local chained scans; O_{g+1} = O_g + T_g folded in
 * rank order; W = min((O_g + S)/T, 1) with T = O_G; W[M-1] = 1. */
int drs_ref_build_table_sharded(const double *w, int64_t M, int G, double *W,
                                double *shard_totals) {
  int st = 0;
  for (int64_t j = 0; j < M; ++j)
    if (!(w[j] >= 0.0 && w[j] < INFINITY)) st |= DRS_REF_ST_INVALID_WEIGHT;
  double *Tg = (double *)malloc(sizeof(double) * (size_t)G);
  for (int g = 0; g < G; ++g) {
    const int64_t a = M * g / G, b = M * (g + 1) / G;
    drs_ref_chain_scan(w + a, b - a, DRS_REF_K_TABLE, W + a, &Tg[g]);
    if (shard_totals) shard_totals[g] = Tg[g];
  }
  double O = 0.0;
  for (int g = 0; g < G; ++g) O = O + Tg[g];
  const double T = O;
  if (T == 0.0) st |= DRS_REF_ST_DEGENERATE;
  if (!(T < INFINITY)) st |= DRS_REF_ST_ACCUM_OVERFLOW;
  O = 0.0;
  for (int g = 0; g < G; ++g) {
    const int64_t a = M * g / G, b = M * (g + 1) / G;
    for (int64_t j = a; j < b; ++j) W[j] = fmin((O + W[j]) / T, 1.0);
    O = O + Tg[g];
  }
  W[M - 1] = 1.0;
  free(Tg);
  return st;
}

/* ------------------------------------------------------------------------ */
/* Search kernels, restated from the numba code.                            */
/* ------------------------------------------------------------------------ */
/* numpy's pairwise summation (ndarray.sum of a contiguous float64 array,
 * used by build_weight_table cdf.py:77): blocks below 8 summed serially,
 * blocks up to 128 with 8 interleaved accumulators, larger ones split in
 * halves rounded down to a multiple of 8. */
static double np_pairwise_sum(const double *a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
  }
}

double drs_port_total(const double *w, int64_t M) { return np_pairwise_sum(w, M); }

/* build_weight_table (cdf.py:59-89) with the reference's own association:
 * pairwise total, sequential cumsum, divide, drift check, clip, pin. */
int drs_port_build_table(const double *w, int64_t M, double *W) {
  int st = 0;
  for (int64_t j = 0; j < M; ++j)
    if (!(w[j] >= 0.0 && w[j] < INFINITY)) return DRS_REF_ST_INVALID_WEIGHT;
  const double total = np_pairwise_sum(w, M);
  if (total == 0.0) return DRS_REF_ST_DEGENERATE;
  double c = 0.0;
  for (int64_t j = 0; j < M; ++j) {
    c = (j == 0) ? w[0] : c + w[j];
    W[j] = c;
  }
  for (int64_t j = 0; j < M; ++j) W[j] = W[j] / total;
  if (!(fabs(W[M - 1] - 1.0) <= 1e-9)) return DRS_REF_ST_ACCUM_OVERFLOW;
  for (int64_t j = 0; j < M; ++j) W[j] = fmin(W[j], 1.0);
  W[M - 1] = 1.0;
  return st;
}

/* _upper_bound_nb (samplers.py:81-90): smallest j in [lo,hi] with cum[j]>=x, else hi */
int64_t drs_port_upper_bound(const double *cum, int64_t lo, int64_t hi, double x) {
  int64_t a = lo, b = hi;
  while (a != b) {
    const int64_t m = (a + b) / 2;
    if (cum[m] < x) a = m + 1;
    else b = m;
  }
  return a;
}

/* _binary_kernel (samplers.py:93-97) */
void drs_port_match_binary(const double *W, int64_t M, const double *u, int64_t N, int64_t *out) {
  for (int64_t i = 0; i < N; ++i) out[i] = drs_port_upper_bound(W, 0, M - 1, u[i]);
}

/* _ccf_kernel (samplers.py:100-107); the j < M-1 guard only matters for
 * u > 1, where the reference reads past the table */
void drs_port_match_ccf(const double *W, int64_t M, const double *U, int64_t N, int64_t *out) {
  int64_t j = 0;
  for (int64_t i = 0; i < N; ++i) {
    const double x = U[i];
    while (j < M - 1 && W[j] < x) ++j;
    out[i] = j;
  }
}

/* _dac_kernel (samplers.py:110-146): explicit LIFO of (a_u, b_u, a_w, b_w) */
int drs_port_match_dac(const double *W, int64_t M, const double *U, int64_t N, int64_t *out) {
  if (N <= 0) return 0;
  int64_t stack[128][4];
  int top = 0;
  stack[0][0] = 0; stack[0][1] = N - 1; stack[0][2] = 0; stack[0][3] = M - 1;
  top = 1;
  while (top > 0) {
    --top;
    const int64_t a_u = stack[top][0], b_u = stack[top][1];
    const int64_t a_w = stack[top][2], b_w = stack[top][3];
    if (a_u == b_u) {
      out[a_u] = drs_port_upper_bound(W, a_w, b_w, U[a_u]);
    } else if (a_w == b_w) {
      for (int64_t i = a_u; i <= b_u; ++i) out[i] = a_w;
    } else {
      const int64_t m_u = (a_u + b_u) / 2;
      const int64_t m_w = drs_port_upper_bound(W, a_w, b_w, U[m_u]);
      out[m_u] = m_w;
      if (m_u < b_u) {
        if (top >= 128) return -1;
        stack[top][0] = m_u + 1; stack[top][1] = b_u; stack[top][2] = m_w; stack[top][3] = b_w;
        ++top;
      }
      if (m_u > a_u) {
        if (top >= 128) return -1;
        stack[top][0] = a_u; stack[top][1] = m_u - 1; stack[top][2] = a_w; stack[top][3] = m_w;
        ++top;
      }
    }
  }
  return 0;
}

/* sorted_uniforms (randkit.py:84-101) with numpy's association: sequential
 * cumsum in place, z_min taken before the cumsum, U = Z[:-1]/Z[-1]. */
int drs_port_sorted_from_z(double *z, int64_t n, double *U) {
  if (n <= 0) return 0;
  double zmin = z[0];
  for (int64_t i = 1; i <= n; ++i) zmin = fmin(zmin, z[i]);
  for (int64_t i = 1; i <= n; ++i) z[i] = z[i - 1] + z[i];
  const double total = z[n];
  for (int64_t i = 0; i < n; ++i) U[i] = z[i] / total;
  return check_and_repair(U, n, zmin, total);
}

int drs_port_sorted_uniforms(uint64_t k0, uint64_t k1, uint64_t offset, int64_t n, double *U) {
  if (n <= 0) return 0;
  double *z = (double *)malloc(sizeof(double) * (size_t)(n + 1));
  drs_ref_uniforms(k0, k1, offset, n + 1, z);
  for (int64_t i = 0; i <= n; ++i) z[i] = -drs_ref_log(z[i]);
  int st = drs_port_sorted_from_z(z, n, U);
  free(z);
  return st;
}

/* one sampler call as the reference makes it (samplers.py:238-266):
 * which = 0 dac, 1 ccf, 2 binary.  scratch holds n+1 doubles. */
int drs_port_sampler(int which, const double *W, int64_t M, uint64_t k0, uint64_t k1,
                     uint64_t offset, int64_t N, double *scratch, int64_t *out) {
  if (N <= 0) return 0;
  if (which == 2) {
    drs_ref_uniforms(k0, k1, offset, N, scratch);
    drs_port_match_binary(W, M, scratch, N, out);
    return 0;
  }
  double *U = scratch + N + 1;
  drs_ref_uniforms(k0, k1, offset, N + 1, scratch);
  for (int64_t i = 0; i <= N; ++i) scratch[i] = -drs_ref_log(scratch[i]);
  drs_port_sorted_from_z(scratch, N, U);
  if (which == 1) drs_port_match_ccf(W, M, U, N, out);
  else drs_port_match_dac(W, M, U, N, out);
  return 0;
}

typedef struct {
  int which, calls;
  const double *W;
  int64_t M, N;
  uint64_t k0, k1, offset;
} port_job;

static void *port_worker(void *arg) {
  port_job *j = (port_job *)arg;
  double *scratch = (double *)malloc(sizeof(double) * (size_t)(2 * j->N + 2));
  int64_t *out = (int64_t *)malloc(sizeof(int64_t) * (size_t)j->N);
  for (int c = 0; c < j->calls; ++c)
    drs_port_sampler(j->which, j->W, j->M, j->k0, j->k1,
                     j->offset + (uint64_t)c * (uint64_t)(j->N + 1), j->N, scratch, out);
  free(scratch);
  free(out);
  return NULL;
}

/* wall seconds for `threads` host threads each making `calls_per_thread`
 * independent sampler calls on the shared table (the reference is
 * single-threaded; threads > 1 runs independent replicas) */
double drs_port_throughput(int which, const double *W, int64_t M, int64_t N, int threads,
                           int calls_per_thread, uint64_t k0, uint64_t k1) {
  if (threads < 1) threads = 1;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
  port_job *jobs = (port_job *)malloc(sizeof(port_job) * (size_t)threads);
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int t = 0; t < threads; ++t) {
    jobs[t].which = which; jobs[t].calls = calls_per_thread; jobs[t].W = W;
    jobs[t].M = M; jobs[t].N = N; jobs[t].k0 = k0 + (uint64_t)t; jobs[t].k1 = k1;
    jobs[t].offset = 0;
    pthread_create(&th[t], NULL, port_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  free(th);
  free(jobs);
  return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

typedef struct {
  const double *w;
  int64_t f0, f1, Mf, Nf;
  int reps;
  uint64_t k0, k1;
} batch_job;

static void *batch_worker(void *arg) {
  batch_job *j = (batch_job *)arg;
  double *W = (double *)malloc(sizeof(double) * (size_t)j->Mf);
  double *scratch = (double *)malloc(sizeof(double) * (size_t)(2 * j->Nf + 2));
  int64_t *out = (int64_t *)malloc(sizeof(int64_t) * (size_t)(j->Nf > 0 ? j->Nf : 1));
  for (int r = 0; r < j->reps; ++r)
    for (int64_t f = j->f0; f < j->f1; ++f) {
      drs_port_build_table(j->w + f * j->Mf, j->Mf, W);
      drs_port_sampler(0, W, j->Mf, j->k0 + (uint64_t)f, j->k1, (uint64_t)r * (uint64_t)(j->Nf + 1), j->Nf,
                       scratch, out);
    }
  free(W);
  free(scratch);
  free(out);
  return NULL;
}

/* wall seconds for the reference's per-filter loop (build_weight_table +
 * dac_sampler per filter, cdf.py:59-89 + samplers.py:262-266) over filters
 * [0, B), `reps` times, the filters split into `threads` contiguous ranges */
double drs_port_batched_throughput(const double *w, int64_t B, int64_t Mf, int64_t Nf, int threads,
                                   int reps, uint64_t k0, uint64_t k1) {
  if (threads < 1) threads = 1;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
  batch_job *jobs = (batch_job *)malloc(sizeof(batch_job) * (size_t)threads);
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int t = 0; t < threads; ++t) {
    jobs[t].w = w; jobs[t].Mf = Mf; jobs[t].Nf = Nf; jobs[t].reps = reps;
    jobs[t].f0 = B * t / threads; jobs[t].f1 = B * (t + 1) / threads;
    jobs[t].k0 = k0; jobs[t].k1 = k1;
    pthread_create(&th[t], NULL, batch_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  free(th);
  free(jobs);
  return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

/* batched filters (config 4): per filter, build_table + sorted_uniforms
 * (keys[3f], keys[3f+1], draw offset keys[3f+2]) + lower-bound match, all with
 * the device association.  W and U may be NULL. */
int drs_ref_resample_batched(const double *w, int64_t B, int64_t Mf, int64_t Nf,
                             const uint64_t *keys, double *W, double *U, int64_t *out) {
  int st = 0;
  double *Wf = (double *)malloc(sizeof(double) * (size_t)Mf);
  double *Uf = (double *)malloc(sizeof(double) * (size_t)(Nf > 0 ? Nf : 1));
  for (int64_t f = 0; f < B; ++f) {
    st |= drs_ref_build_table(w + f * Mf, Mf, Wf);
    st |= drs_ref_sorted_uniforms(keys[3 * f], keys[3 * f + 1], keys[3 * f + 2], Nf, Uf);
    for (int64_t i = 0; i < Nf; ++i) out[f * Nf + i] = drs_port_upper_bound(Wf, 0, Mf - 1, Uf[i]);
    if (W) memcpy(W + f * Mf, Wf, sizeof(double) * (size_t)Mf);
    if (U && Nf > 0) memcpy(U + f * Nf, Uf, sizeof(double) * (size_t)Nf);
  }
  free(Wf);
  free(Uf);
  return st;
}
