/*
 * FP64 C port of the reference nbnxn path -- TEST INFRASTRUCTURE / CPU BASELINE ONLY.
 *
 * Restates, operation for operation, the reference package clustermd:
 *   orc_force        kernels.py:124-221  (_kernel_blocks, canonical layout m x m:
 *                                         rows in CSR order, a outer, b inner)
 *   orc_search_n2    pairlist.py:177-189 (O(n_c^2) AABB-gap search, j >= i)
 *   orc_search_cols  same criterion, O(N) candidate columns (for sizes where the
 *                    reference's O(n_c^2) loop is impractical, e.g. 1.5M atoms)
 *   orc_row_min_d2   pairlist.py:220-239 (einsum order (dx^2 + dz^2) + dy^2)
 *   orc_count_within pairlist.py:303-320
 * geometry from model.py:159-172, gap from gridder.py:165-185.
 *
 * Compiled with -ffp-contract=off (no FMA contraction) so every FP64 decision
 * matches numpy/numba bit for bit.  OpenMP threads split i-clusters into
 * contiguous chunks with private force buffers reduced in fixed order, which
 * is the reference's own worker scheme (engine.py:462-521) and keeps results
 * bit-identical across reruns at a fixed thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

typedef int64_t i64;
typedef uint64_t u64;

enum { ELEC_CUTOFF = 0, ELEC_RF = 1, ELEC_EWALD = 2 };

static inline double min_image_1(double dr, double L) {
  /* model.py:167-171 */
  double out = dr - floor(dr / L + 0.5) * L;
  double half = 0.5 * L;
  if (out >= half) out = out - L;
  if (out < -half) out = out + L;
  return out;
}

static inline double kernel_min_image(double d, double L) {
  /* kernels.py:168-182: same expression, folds as if/elif */
  d -= floor(d / L + 0.5) * L;
  if (d >= 0.5 * L) d -= L;
  else if (d < -0.5 * L) d += L;
  return d;
}

static inline double gap_1d(double lo_i, double hi_i, double lo_j, double hi_j, double span) {
  /* gridder.py:177-183 */
  double a = lo_j - hi_i;
  double b = lo_i - hi_j;
  double t;
  t = a > b ? a : b;            /* np.maximum(a, b) for non-NaN */
  double g0 = 0.0 >= t ? 0.0 : t;
  double am = a - span, bp = b + span;
  t = am > bp ? am : bp;
  double gm = 0.0 >= t ? 0.0 : t;
  double ap = a + span, bm = b - span;
  t = ap > bm ? ap : bm;
  double gp = 0.0 >= t ? 0.0 : t;
  double g = gm <= gp ? gm : gp;
  g = g0 <= g ? g0 : g;
  return g;
}

static inline double gap_sq(const double* bi, const double* bj, const double* L) {
  /* bboxes laid out [lo x,y,z, hi x,y,z]; sum ((0 + gx^2) + gy^2) + gz^2 */
  double s = 0.0;
  for (int d = 0; d < 3; ++d) {
    double g = gap_1d(bi[d], bi[3 + d], bj[d], bj[3 + d], L[d]);
    s = s + g * g;
  }
  return s;
}

/* ---------------------------------------------------------------- search */

i64 orc_search_n2(i64 nc, const double* bboxes, const double* L, double r_list,
                  i64* counts, i64* j_out, const i64* offsets, int nthreads) {
  /* Pass with j_out == NULL: counts[ci]; otherwise write rows at offsets[ci]. */
  const double r2 = r_list * r_list;
  i64 total = 0;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads) reduction(+ : total)
  for (i64 ci = 0; ci < nc; ++ci) {
    const double* bi = bboxes + 6 * ci;
    i64 k = 0;
    i64 base = j_out ? offsets[ci] : 0;
    for (i64 cj = ci; cj < nc; ++cj) {
      if (gap_sq(bi, bboxes + 6 * cj, L) <= r2) {
        if (j_out) j_out[base + k] = cj;
        ++k;
      }
    }
    if (!j_out) counts[ci] = k;
    total += k;
  }
  return total;
}

static int cmp_i64(const void* a, const void* b) {
  i64 x = *(const i64*)a, y = *(const i64*)b;
  return (x > y) - (x < y);
}

i64 orc_search_cols(i64 nc, const double* bboxes, const i64* cell_of_cluster,
                    const i64* col_first /* cells*cells + 1 cluster offsets */,
                    i64 cells, const double* L, double r_list,
                    i64* counts, i64* j_out, const i64* offsets, int nthreads) {
  const double r2 = r_list * r_list;
  const double wx = L[0] / (double)cells, wy = L[1] / (double)cells;
  const i64 rx = (i64)floor(r_list / wx) + 2, ry = (i64)floor(r_list / wy) + 2;
  i64 total = 0;
#pragma omp parallel num_threads(nthreads) reduction(+ : total)
  {
    i64* xs = (i64*)malloc(sizeof(i64) * (size_t)(cells + 4 * rx + 8));
    i64* ys = (i64*)malloc(sizeof(i64) * (size_t)(cells + 4 * ry + 8));
    i64 cap = 1024;
    i64* buf = (i64*)malloc(sizeof(i64) * (size_t)cap);
#pragma omp for schedule(dynamic, 64)
    for (i64 ci = 0; ci < nc; ++ci) {
      const double* bi = bboxes + 6 * ci;
      i64 x0 = (i64)floor(bi[0] / wx) - rx, x1 = (i64)floor(bi[3] / wx) + rx;
      i64 y0 = (i64)floor(bi[1] / wy) - ry, y1 = (i64)floor(bi[4] / wy) + ry;
      i64 nx = 0, ny = 0;
      if (x1 - x0 + 1 >= cells) { for (i64 v = 0; v < cells; ++v) xs[nx++] = v; }
      else { for (i64 v = x0; v <= x1; ++v) xs[nx++] = ((v % cells) + cells) % cells; qsort(xs, nx, sizeof(i64), cmp_i64); }
      if (y1 - y0 + 1 >= cells) { for (i64 v = 0; v < cells; ++v) ys[ny++] = v; }
      else { for (i64 v = y0; v <= y1; ++v) ys[ny++] = ((v % cells) + cells) % cells; qsort(ys, ny, sizeof(i64), cmp_i64); }
      i64 k = 0;
      for (i64 a = 0; a < nx; ++a) {
        for (i64 b = 0; b < ny; ++b) {
          i64 col = xs[a] * cells + ys[b];
          for (i64 cj = col_first[col]; cj < col_first[col + 1]; ++cj) {
            if (cj < ci) continue;
            if (gap_sq(bi, bboxes + 6 * cj, L) <= r2) {
              if (k == cap) { cap *= 2; buf = (i64*)realloc(buf, sizeof(i64) * (size_t)cap); }
              buf[k++] = cj;
            }
          }
        }
      }
      /* columns ascend in cell id and clusters ascend with cell id, so buf is
         ascending already; sort anyway to make the invariant explicit */
      qsort(buf, (size_t)k, sizeof(i64), cmp_i64);
      if (j_out) memcpy(j_out + offsets[ci], buf, sizeof(i64) * (size_t)k);
      else counts[ci] = k;
      total += k;
    }
    free(xs); free(ys); free(buf);
  }
  (void)cell_of_cluster;
  return total;
}

/* ---------------------------------------------------------------- prune / stats */

void orc_row_min_d2(i64 n_clusters, int m, const i64* offsets, const i64* j_idx, const u64* masks,
                    const double* pos, const double* L, double* out, int nthreads) {
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads)
  for (i64 ci = 0; ci < n_clusters; ++ci) {
    for (i64 p = offsets[ci]; p < offsets[ci + 1]; ++p) {
      double best = INFINITY;
      const i64 cj = j_idx[p];
      for (int a = 0; a < m; ++a) {
        const double* pi = pos + 3 * (ci * m + a);
        for (int b = 0; b < m; ++b) {
          if (!((masks[p] >> (a * m + b)) & 1ull)) continue;
          const double* pj = pos + 3 * (cj * m + b);
          double dx = min_image_1(pi[0] - pj[0], L[0]);
          double dy = min_image_1(pi[1] - pj[1], L[1]);
          double dz = min_image_1(pi[2] - pj[2], L[2]);
          double d2 = (dx * dx + dz * dz) + dy * dy; /* numpy einsum order */
          if (d2 < best) best = d2;
        }
      }
      out[p] = best;
    }
  }
}

i64 orc_count_within(i64 n_clusters, int m, const i64* offsets, const i64* j_idx, const u64* masks,
                     const double* pos, const double* L, double r_cut, int nthreads) {
  const double rc2 = r_cut * r_cut;
  i64 total = 0;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads) reduction(+ : total)
  for (i64 ci = 0; ci < n_clusters; ++ci) {
    for (i64 p = offsets[ci]; p < offsets[ci + 1]; ++p) {
      const i64 cj = j_idx[p];
      for (int a = 0; a < m; ++a) {
        const double* pi = pos + 3 * (ci * m + a);
        for (int b = 0; b < m; ++b) {
          if (!((masks[p] >> (a * m + b)) & 1ull)) continue;
          const double* pj = pos + 3 * (cj * m + b);
          double dx = min_image_1(pi[0] - pj[0], L[0]);
          double dy = min_image_1(pi[1] - pj[1], L[1]);
          double dz = min_image_1(pi[2] - pj[2], L[2]);
          double d2 = (dx * dx + dz * dz) + dy * dy;
          total += d2 <= rc2;
        }
      }
    }
  }
  return total;
}

/* ---------------------------------------------------------------- force */

typedef struct {
  int elec, shift, ntypes;
  double coul, r_cut, rc2, k_rf, c_rf, beta, erfc_rc;
  const double *eps_t, *sig_t, *shift_lj_t;
} phys_t;

static double chunk_force(const phys_t* ph, int m, i64 c0, i64 c1, const i64* offsets,
                          const i64* j_idx, const u64* masks, const double* pos, const double* q,
                          const i64* typ, const double* L, double* f, double* e_lj_out,
                          i64* bad) {
  double e_lj_total = 0.0, e_c_total = 0.0;
  double fi[8][3];
  const double two_over_sqrt_pi = 1.1283791670955126;
  for (i64 ci = c0; ci < c1; ++ci) {
    const i64 base_i = ci * m;
    memset(fi, 0, sizeof(fi));
    double e_lj = 0.0, e_c = 0.0;
    for (i64 p = offsets[ci]; p < offsets[ci + 1]; ++p) {
      const i64 cj = j_idx[p];
      for (int a = 0; a < m; ++a) {
        const i64 si = base_i + a;
        const double xi = pos[3 * si], yi = pos[3 * si + 1], zi = pos[3 * si + 2];
        const double qi = q[si];
        const i64 ti = typ[si];
        for (int b = 0; b < m; ++b) {
          if (!((masks[p] >> (a * m + b)) & 1ull)) continue;
          const i64 sj = cj * m + b;
          double dx = kernel_min_image(xi - pos[3 * sj], L[0]);
          double dy = kernel_min_image(yi - pos[3 * sj + 1], L[1]);
          double dz = kernel_min_image(zi - pos[3 * sj + 2], L[2]);
          double r2 = dx * dx + dy * dy + dz * dz; /* kernels.py:183, sequential */
          if (r2 > ph->rc2) continue;
          if (r2 == 0.0) { bad[0] = si; bad[1] = sj; *e_lj_out = e_lj_total; return e_c_total; }
          const i64 tj = typ[sj];
          const double eps = ph->eps_t[ti * ph->ntypes + tj];
          const double sig = ph->sig_t[ti * ph->ntypes + tj];
          double sr2 = (sig * sig) / r2;
          double sr6 = sr2 * sr2 * sr2;
          double e_pair_lj = 4.0 * eps * (sr6 * sr6 - sr6);
          double f_over_r = 48.0 * eps * (sr6 * sr6 - 0.5 * sr6) / r2;
          double r = sqrt(r2);
          double qq = ph->coul * qi * q[sj];
          double e_pair_c;
          if (ph->elec == ELEC_CUTOFF) {
            e_pair_c = qq / r;
            f_over_r = f_over_r + qq / (r2 * r);
            if (ph->shift) e_pair_c = e_pair_c - qq / ph->r_cut;
          } else if (ph->elec == ELEC_RF) {
            e_pair_c = qq * (1.0 / r + ph->k_rf * r2 - ph->c_rf);
            f_over_r = f_over_r + qq * (1.0 / (r2 * r) - 2.0 * ph->k_rf);
          } else {
            double er = erfc(ph->beta * r);
            e_pair_c = qq * er / r;
            f_over_r = f_over_r + qq * (er / r + ph->beta * two_over_sqrt_pi * exp(-ph->beta * ph->beta * r2)) / r2;
            if (ph->shift) e_pair_c = e_pair_c - qq * ph->erfc_rc / ph->r_cut;
          }
          if (ph->shift) e_pair_lj = e_pair_lj - ph->shift_lj_t[ti * ph->ntypes + tj];
          e_lj += e_pair_lj;
          e_c += e_pair_c;
          const double fx = f_over_r * dx, fy = f_over_r * dy, fz = f_over_r * dz;
          fi[a][0] += fx; fi[a][1] += fy; fi[a][2] += fz;
          f[3 * sj] -= fx; f[3 * sj + 1] -= fy; f[3 * sj + 2] -= fz;
        }
      }
    }
    for (int a = 0; a < m; ++a) {
      f[3 * (base_i + a)] += fi[a][0];
      f[3 * (base_i + a) + 1] += fi[a][1];
      f[3 * (base_i + a) + 2] += fi[a][2];
    }
    e_lj_total += e_lj;
    e_c_total += e_c;
  }
  *e_lj_out = e_lj_total;
  return e_c_total;
}

int orc_force(i64 n_clusters, int m, const i64* offsets, const i64* j_idx, const u64* masks,
              const double* pos, const double* q, const i64* typ, int ntypes,
              const double* eps_t, const double* sig_t, const double* shift_lj_t,
              int elec, int shift, double coul, double r_cut, double k_rf, double c_rf,
              double beta, const double* L, int nthreads, double* f_out, double* e_out,
              i64* bad) {
  phys_t ph = {elec, shift, ntypes, coul, r_cut, r_cut * r_cut, k_rf, c_rf, beta,
               erfc(beta * r_cut), eps_t, sig_t, shift_lj_t};
  const i64 n_slots = n_clusters * m;
  if (nthreads < 1) nthreads = 1;
  /* contiguous chunks balanced by row count (engine.py:409-426 scheme) */
  i64* cuts = (i64*)malloc(sizeof(i64) * (size_t)(nthreads + 1));
  const i64 n_rows = offsets[n_clusters];
  cuts[0] = 0;
  {
    i64 c = 0;
    for (int t = 1; t < nthreads; ++t) {
      i64 target = (n_rows * t) / nthreads;
      while (c < n_clusters && offsets[c] < target) ++c;
      cuts[t] = c;
    }
  }
  cuts[nthreads] = n_clusters;
  double* bufs = (double*)calloc((size_t)nthreads * (size_t)n_slots * 3, sizeof(double));
  double* elj = (double*)calloc((size_t)nthreads, sizeof(double));
  double* ec = (double*)calloc((size_t)nthreads, sizeof(double));
  i64* bads = (i64*)malloc(sizeof(i64) * 2 * (size_t)nthreads);
  for (int t = 0; t < nthreads; ++t) bads[2 * t] = bads[2 * t + 1] = -1;
#pragma omp parallel for schedule(static, 1) num_threads(nthreads)
  for (int t = 0; t < nthreads; ++t) {
    ec[t] = chunk_force(&ph, m, cuts[t], cuts[t + 1], offsets, j_idx, masks, pos, q, typ, L,
                        bufs + (size_t)t * n_slots * 3, &elj[t], bads + 2 * t);
  }
  double e_lj = 0.0, e_c = 0.0;
  int status = 0;
  for (int t = 0; t < nthreads; ++t) {
    const double* b = bufs + (size_t)t * n_slots * 3;
    for (i64 k = 0; k < 3 * n_slots; ++k) f_out[k] += b[k];
    e_lj += elj[t];
    e_c += ec[t];
    if (!status && bads[2 * t] >= 0) { bad[0] = bads[2 * t]; bad[1] = bads[2 * t + 1]; status = 2; }
  }
  e_out[0] = e_lj;
  e_out[1] = e_c;
  free(cuts); free(bufs); free(elj); free(ec); free(bads);
  return status;
}

int orc_max_threads(void) { return omp_get_max_threads(); }
