/*
 * oracle/tsqbx_oracle.c -- CPU restatement of the reference TSQBX evaluator.
 *
 * TEST INFRASTRUCTURE ONLY (see tsqbx_oracle.h).  Every routine cites the
 * reference lines it restates; paths are relative to /root/reference/pkg/src/gigaqbx.
 * The arithmetic follows the reference's scalar order so that the oracle and
 * the reference agree to a few ulps; it is compiled with -ffp-contract=off.
 */
#include "tsqbx_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static const double kFourPi = 4.0 * 3.14159265358979323846264338327950288;

/* ------------------------------------------------------------------ */
/* spherical Bessel j_n by Miller, Hankel h_n upward (_core.pyx:172-198) */
/* ------------------------------------------------------------------ */
static void sph_jh(int p, double x, double* j, double* jp, double complex* h,
                   double complex* hp, double* f, int nbuf) {
  const int top = nbuf - 2;               /* Miller start, _core.pyx:177 */
  f[top + 1] = 0.0;
  f[top] = 1e-290;
  for (int n = top; n > 0; --n) {
    f[n - 1] = (2.0 * n + 1.0) / x * f[n] - f[n + 1];
    if (f[n - 1] > 1e250 || f[n - 1] < -1e250) {   /* rescale, :186-188 */
      for (int m = n - 1; m < top + 2; ++m) f[m] *= 1e-250;
    }
  }
  const double norm = (sin(x) / x) / f[0];
  for (int n = 0; n < p + 2; ++n) j[n] = f[n] * norm;
  h[0] = (sin(x) - I * cos(x)) / x;                /* :190 */
  h[1] = h[0] * (1.0 / x - I);                      /* :191 */
  for (int n = 1; n < p + 1; ++n) h[n + 1] = (2.0 * n + 1.0) / x * h[n] - h[n - 1];
  jp[0] = -j[1];
  hp[0] = -h[1];
  for (int n = 1; n < p + 1; ++n) {                 /* :196-198 */
    jp[n] = j[n - 1] - (n + 1.0) / x * j[n];
    hp[n] = h[n - 1] - (n + 1.0) / x * h[n];
  }
}

/* per-(center,target) geometry shared by both equations (_core.pyx:214-225) */
typedef struct {
  double r, th[3], nt[3];
} tgt_geom;

static tgt_geom target_geometry(const double* c, const double* t, const double* tn) {
  tgt_geom g;
  double d0 = t[0] - c[0], d1 = t[1] - c[1], d2 = t[2] - c[2];
  g.r = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
  g.th[0] = g.th[1] = g.th[2] = 0.0;
  if (g.r > 0.0) { g.th[0] = d0 / g.r; g.th[1] = d1 / g.r; g.th[2] = d2 / g.r; }
  g.nt[0] = g.nt[1] = g.nt[2] = 0.0;
  if (tn) { g.nt[0] = tn[0]; g.nt[1] = tn[1]; g.nt[2] = tn[2]; }
  return g;
}

/* source unit vector, R and clamped cos(gamma) (_core.pyx:230-242) */
static inline double source_geometry(const double* s, const double* c, const tgt_geom* g,
                                     double* sh, double* R) {
  double x = s[0] - c[0], y = s[1] - c[1], z = s[2] - c[2];
  *R = sqrt(x * x + y * y + z * z);
  sh[0] = x / *R; sh[1] = y / *R; sh[2] = z / *R;
  if (!(g->r > 0.0)) return 1.0;                    /* cos gamma := 1 at r = 0 */
  double cg = sh[0] * g->th[0] + sh[1] * g->th[1] + sh[2] * g->th[2];
  return cg > 1.0 ? 1.0 : (cg < -1.0 ? -1.0 : cg);
}

static inline double dot3(const double* a, const double* b) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

/* ------------------------------------------------------------------ */
/* Laplace S / S' / D  (_core.pyx:205-307)                              */
/* ------------------------------------------------------------------ */
int orc_ts_accum_laplace(int variant, int p, int64_t n, const double* src, const double* w,
                         const double* snrm, const double* ctr, const double* tgt,
                         const double* tnrm, double* out) {
  out[0] = out[1] = 0.0;
  if (n == 0) return 0;
  if (variant < 0 || variant > 2 || p < 0) return 3;
  if (variant == 2 && !snrm) return 3;
  const tgt_geom g = target_geometry(ctr, tgt, tnrm);
  double complex acc = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    double sh[3], R;
    const double cg = source_geometry(src + 3 * j, ctr, &g, sh, &R);
    const double rho = g.r / R;
    double s = 0.0;
    if (variant == 0) {                       /* :244-259, sum rho^n P_n / R */
      double rad = 1.0 / R, pm1 = 1.0, pc = cg;
      s = rad;
      if (p >= 1) { rad *= rho; s += rad * pc; }
      for (int m = 1; m < p; ++m) {
        double pn = ((2 * m + 1) * cg * pc - m * pm1) / (m + 1.0);
        pm1 = pc; pc = pn; rad *= rho; s += rad * pc;
      }
    } else if (variant == 1) {                /* :260-282, target-normal derivative */
      const double nt_th = g.r > 0.0 ? dot3(g.nt, g.th) : dot3(g.nt, sh);
      const double nt_sh = dot3(g.nt, sh);
      double rad = 1.0 / (R * R), pm1 = 1.0, pc = cg, dm1 = 0.0, dc = 1.0;
      for (int m = 1; m <= p; ++m) {
        s += rad * (m * nt_th * pc + (nt_sh - nt_th * cg) * dc);
        if (m < p) {
          double pn = ((2 * m + 1) * cg * pc - m * pm1) / (m + 1.0);
          double dn = dm1 + (2 * m + 1) * pc;
          pm1 = pc; pc = pn; dm1 = dc; dc = dn; rad *= rho;
        }
      }
    } else {                                  /* :283-306, double layer */
      const double* ns = snrm + 3 * j;
      const double ns_sh = dot3(ns, sh);
      const double ns_th = g.r > 0.0 ? dot3(ns, g.th) : ns_sh;
      double rad = 1.0 / (R * R), pm1 = 1.0, pc = cg, dm1 = 0.0, dc = 1.0;
      s = rad * (-1.0 * ns_sh);
      for (int m = 1; m <= p; ++m) {
        rad *= rho;
        s += rad * (-(m + 1.0) * ns_sh * pc + (ns_th - ns_sh * cg) * dc);
        if (m < p) {
          double pn = ((2 * m + 1) * cg * pc - m * pm1) / (m + 1.0);
          double dn = dm1 + (2 * m + 1) * pc;
          pm1 = pc; pc = pn; dm1 = dc; dc = dn;
        }
      }
    }
    const double complex wj = w[2 * j] + I * w[2 * j + 1];
    acc += wj * (s / kFourPi);
  }
  out[0] = creal(acc);
  out[1] = cimag(acc);
  return 0;
}

/* ------------------------------------------------------------------ */
/* Helmholtz S / S' / D  (_core.pyx:310-419)                            */
/* ------------------------------------------------------------------ */
int orc_ts_accum_helmholtz(int variant, double k, int p, int64_t n, const double* src,
                           const double* w, const double* snrm, const double* ctr,
                           const double* tgt, const double* tnrm, double* out) {
  out[0] = out[1] = 0.0;
  if (n == 0) return 0;
  if (variant < 0 || variant > 2 || p < 0 || !(k > 0.0)) return 3;
  if (variant == 2 && !snrm) return 3;
  const tgt_geom g = target_geometry(ctr, tgt, tnrm);

  double Rmax = 0.0;                                  /* :328-335 */
  for (int64_t j = 0; j < n; ++j) {
    const double* s = src + 3 * j;
    double Rj = sqrt((s[0] - ctr[0]) * (s[0] - ctr[0]) + (s[1] - ctr[1]) * (s[1] - ctr[1]) +
                     (s[2] - ctr[2]) * (s[2] - ctr[2]));
    if (Rj > Rmax) Rmax = Rj;
  }
  const int nbuf = p + 18 + (int)ceil(k * (Rmax > g.r ? Rmax : g.r));  /* :338 */
  /* per-source Miller buffers may be longer than nbuf when kR > k*Rmax
   * cannot happen (R <= Rmax), so nbuf bounds every call */
  double* f = (double*)calloc((size_t)nbuf + 2, sizeof(double));
  double* jt = (double*)calloc((size_t)p + 2, sizeof(double));
  double* jtp = (double*)calloc((size_t)p + 1, sizeof(double));
  double* js = (double*)calloc((size_t)p + 2, sizeof(double));
  double* jsp = (double*)calloc((size_t)p + 1, sizeof(double));
  double complex* hh = (double complex*)calloc((size_t)p + 2, sizeof(double complex));
  double complex* hhp = (double complex*)calloc((size_t)p + 1, sizeof(double complex));
  if (!f || !jt || !jtp || !js || !jsp || !hh || !hhp) {
    free(f); free(jt); free(jtp); free(js); free(jsp); free(hh); free(hhp);
    return 4;
  }
  if (g.r > 0.0) {
    sph_jh(p, k * g.r, jt, jtp, hh, hhp, f, nbuf);    /* :354-355 */
  } else {
    jt[0] = 1.0;                                      /* :357-359 */
    if (p >= 1) jtp[1] = 1.0 / 3.0;
  }

  double complex acc = 0.0;
  const double complex pref = I * k / kFourPi;
  for (int64_t j = 0; j < n; ++j) {
    double sh[3], R;
    const double cg = source_geometry(src + 3 * j, ctr, &g, sh, &R);
    sph_jh(p, k * R, js, jsp, hh, hhp, f, p + 18 + (int)ceil(k * R));  /* :380-381 */
    double complex s = 0.0;
    double pm1 = 1.0, pc = cg, dm1 = 0.0, dc = 1.0;
    const double* ns = snrm ? snrm + 3 * j : NULL;
    for (int m = 0; m <= p; ++m) {                    /* :386-417 */
      const double pn = m == 0 ? 1.0 : pc;
      const double dn = m == 0 ? 0.0 : dc;
      if (m >= 1 && m < p) {
        double pnx = ((2 * m + 1) * cg * pc - m * pm1) / (m + 1.0);
        double dnx = dm1 + (2 * m + 1) * pc;
        pm1 = pc; pc = pnx; dm1 = dc; dc = dnx;
      }
      if (variant == 0) {
        s += (2 * m + 1.0) * jt[m] * hh[m] * pn;
      } else if (variant == 1) {
        const double nt_sh = dot3(g.nt, sh);
        if (g.r > 0.0) {
          const double nt_th = dot3(g.nt, g.th);
          s += (2 * m + 1.0) * hh[m] *
               (k * nt_th * jtp[m] * pn + (nt_sh - nt_th * cg) * jt[m] * dn / g.r);
        } else {
          s += (2 * m + 1.0) * hh[m] * k * nt_sh * jtp[m] * pn;
        }
      } else {
        const double ns_sh = dot3(ns, sh);
        const double ns_th = g.r > 0.0 ? dot3(ns, g.th) : ns_sh;
        s += (2 * m + 1.0) * jt[m] *
             (k * ns_sh * hhp[m] * pn + (ns_th - ns_sh * cg) * hh[m] * dn / R);
      }
    }
    acc += (w[2 * j] + I * w[2 * j + 1]) * s;
  }
  acc = pref * acc;
  out[0] = creal(acc);
  out[1] = cimag(acc);
  free(f); free(jt); free(jtp); free(js); free(jsp); free(hh); free(hhp);
  return 0;
}

/* ------------------------------------------------------------------ */
/* batched, driver-style loop (driver.py:197-228, 383-389)              */
/* ------------------------------------------------------------------ */
int orc_ts_batch(int equation, int variant, double k, int p, const double* src, const double* w,
                 const double* snrm, int64_t n_src, const double* ctr, int64_t n_ctr,
                 const int64_t* near_ptr, const int32_t* near_idx, const double* tgt,
                 const double* tnrm, const int64_t* tgt_ptr, double* out, int nthreads) {
  (void)n_src;
  int status = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#pragma omp parallel
  {
    int64_t cap = 0;
    double *bs = NULL, *bw = NULL, *bn = NULL;
#pragma omp for schedule(dynamic, 64)
    for (int64_t ic = 0; ic < n_ctr; ++ic) {
      const int64_t b = near_ptr[ic], e = near_ptr[ic + 1], m = e - b;
      if (m > cap) {                                  /* _gather_sources, driver.py:109-113 */
        cap = m;
        bs = (double*)realloc(bs, (size_t)cap * 3 * sizeof(double));
        bw = (double*)realloc(bw, (size_t)cap * 2 * sizeof(double));
        bn = (double*)realloc(bn, (size_t)cap * 3 * sizeof(double));
      }
      for (int64_t q = 0; q < m; ++q) {
        const int64_t s = near_idx[b + q];
        memcpy(bs + 3 * q, src + 3 * s, 3 * sizeof(double));
        memcpy(bw + 2 * q, w + 2 * s, 2 * sizeof(double));
        if (snrm) memcpy(bn + 3 * q, snrm + 3 * s, 3 * sizeof(double));
      }
      for (int64_t it = tgt_ptr[ic]; it < tgt_ptr[ic + 1]; ++it) {
        const double* tn = tnrm ? tnrm + 3 * it : NULL;
        int st = equation == 0
                     ? orc_ts_accum_laplace(variant, p, m, bs, bw, snrm ? bn : NULL, ctr + 3 * ic,
                                            tgt + 3 * it, tn, out + 2 * it)
                     : orc_ts_accum_helmholtz(variant, k, p, m, bs, bw, snrm ? bn : NULL,
                                              ctr + 3 * ic, tgt + 3 * it, tn, out + 2 * it);
        if (st) {
#pragma omp atomic write
          status = st;
        }
      }
    }
    free(bs); free(bw); free(bn);
  }
  return status;
}

/* ------------------------------------------------------------------ */
/* radius-ball near lists (membership oracle; no reference function --  */
/* the reference's closest analogue is cKDTree.query_ball_point,        */
/* costmodel.py:361-365)                                                */
/* ------------------------------------------------------------------ */
typedef struct { int64_t key; int32_t id; } keyed;

static int cmp_keyed(const void* a, const void* b) {
  const keyed *x = (const keyed*)a, *y = (const keyed*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->id < y->id ? -1 : (x->id > y->id);
}
static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return x < y ? -1 : (x > y);
}

static inline int64_t cell_key(int64_t ix, int64_t iy, int64_t iz) {
  return (ix << 42) | (iy << 21) | iz;
}

static inline int member(const double* s, const double* c, double rad) {
  double dx = s[0] - c[0], dy = s[1] - c[1], dz = s[2] - c[2];
  double d2 = dx * dx;
  d2 = d2 + dy * dy;
  d2 = d2 + dz * dz;
  return d2 <= rad * rad;
}

int64_t orc_near_csr(const double* ctr, const double* rad, int64_t n_ctr, const double* src,
                     int64_t n_src, int64_t* ptr, int32_t* idx, int nthreads) {
  if (n_ctr < 0 || n_src < 0 || !ptr) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  double lo[3] = {INFINITY, INFINITY, INFINITY}, rmax = 0.0;
  for (int64_t i = 0; i < n_src; ++i)
    for (int d = 0; d < 3; ++d) lo[d] = fmin(lo[d], src[3 * i + d]);
  for (int64_t i = 0; i < n_ctr; ++i) {
    rmax = fmax(rmax, rad[i]);
    for (int d = 0; d < 3; ++d) lo[d] = fmin(lo[d], ctr[3 * i + d]);
  }
  double hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = 0; i < n_src; ++i)
    for (int d = 0; d < 3; ++d) hi[d] = fmax(hi[d], src[3 * i + d]);
  double ext = 0.0;
  for (int d = 0; d < 3; ++d) ext = fmax(ext, hi[d] - lo[d]);
  /* cell >= rmax so the 27 neighbouring cells cover every ball; cap the grid
   * at 2^20 cells per axis */
  double cell = fmax(rmax, ext / 1048576.0);
  if (!(cell > 0.0)) cell = 1.0;
  keyed* ks = (keyed*)malloc((size_t)(n_src > 0 ? n_src : 1) * sizeof(keyed));
  if (!ks) return -1;
  for (int64_t i = 0; i < n_src; ++i) {
    int64_t ix = (int64_t)floor((src[3 * i] - lo[0]) / cell) + 1;
    int64_t iy = (int64_t)floor((src[3 * i + 1] - lo[1]) / cell) + 1;
    int64_t iz = (int64_t)floor((src[3 * i + 2] - lo[2]) / cell) + 1;
    ks[i].key = cell_key(ix, iy, iz);
    ks[i].id = (int32_t)i;
  }
  qsort(ks, (size_t)n_src, sizeof(keyed), cmp_keyed);

  const int fill = idx != NULL;
  int64_t total = 0;
  if (!fill) ptr[0] = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : total)
  for (int64_t ic = 0; ic < n_ctr; ++ic) {
    const double* c = ctr + 3 * ic;
    int64_t cx = (int64_t)floor((c[0] - lo[0]) / cell) + 1;
    int64_t cy = (int64_t)floor((c[1] - lo[1]) / cell) + 1;
    int64_t cz = (int64_t)floor((c[2] - lo[2]) / cell) + 1;
    int64_t cnt = 0;
    int64_t out = fill ? ptr[ic] : 0;
    for (int64_t dx = -1; dx <= 1; ++dx)
      for (int64_t dy = -1; dy <= 1; ++dy)
        for (int64_t dz = -1; dz <= 1; ++dz) {
          if (cx + dx < 0 || cy + dy < 0 || cz + dz < 0) continue;
          const int64_t key = cell_key(cx + dx, cy + dy, cz + dz);
          int64_t a = 0, b = n_src;                    /* lower_bound */
          while (a < b) {
            int64_t mid = (a + b) / 2;
            if (ks[mid].key < key) a = mid + 1; else b = mid;
          }
          for (int64_t q = a; q < n_src && ks[q].key == key; ++q) {
            if (member(src + 3 * (int64_t)ks[q].id, c, rad[ic])) {
              if (fill) idx[out++] = ks[q].id;
              ++cnt;
            }
          }
        }
    if (fill) qsort(idx + ptr[ic], (size_t)cnt, sizeof(int32_t), cmp_i32);
    else ptr[ic + 1] = cnt;
    total += cnt;
  }
  if (!fill)
    for (int64_t ic = 0; ic < n_ctr; ++ic) ptr[ic + 1] += ptr[ic];
  free(ks);
  return total;
}

/* ------------------------------------------------------------------ */
/* point-to-point direct sum (_core.pyx:94-165)                        */
/* ------------------------------------------------------------------ */
/* One target over its sources [jb, je) (sel == NULL) or sel[jb..je).  Returns
 * the first singular source position (r2 == 0, :109-111 / :145-147) or -1. */
static int64_t p2p_target(int equation, int variant, double k, const double* src,
                          const double* w, const double* snrm, const int32_t* sel, int64_t jb,
                          int64_t je, const double* t, const double* tn, double* out) {
  double complex acc = 0.0;
  for (int64_t q = jb; q < je; ++q) {
    const int64_t j = sel ? (int64_t)sel[q] : q;
    const double dx = t[0] - src[3 * j], dy = t[1] - src[3 * j + 1], dz = t[2] - src[3 * j + 2];
    const double r2 = dx * dx + dy * dy + dz * dz;
    if (r2 == 0.0) return q;
    const double r = sqrt(r2);
    const double complex wj = w[2 * j] + I * w[2 * j + 1];
    if (equation == 0) {                              /* :114-123 */
      if (variant == 0) {
        acc = acc + wj / (kFourPi * r);
      } else if (variant == 1) {
        const double dot = tn[0] * dx + tn[1] * dy + tn[2] * dz;
        acc = acc - wj * dot / (kFourPi * r2 * r);
      } else {
        const double* sn = snrm + 3 * j;
        const double dot = sn[0] * dx + sn[1] * dy + sn[2] * dz;
        acc = acc + wj * dot / (kFourPi * r2 * r);
      }
    } else {                                          /* :150-160 */
      const double complex phase = cos(k * r) + I * sin(k * r);
      if (variant == 0) {
        acc = acc + wj * phase / (kFourPi * r);
      } else {
        const double complex radial = phase * (I * k * r - 1.0) / (kFourPi * r2 * r);
        if (variant == 1) {
          const double dot = tn[0] * dx + tn[1] * dy + tn[2] * dz;
          acc = acc + wj * dot * radial;
        } else {
          const double* sn = snrm + 3 * j;
          const double dot = sn[0] * dx + sn[1] * dy + sn[2] * dz;
          acc = acc - wj * dot * radial;
        }
      }
    }
  }
  out[0] = creal(acc);
  out[1] = cimag(acc);
  return -1;
}

int orc_p2p(int equation, int variant, double k, const double* src, const double* w,
            const double* snrm, int64_t n_src, const int64_t* row_tgt, const int64_t* row_ptr,
            const int32_t* row_idx, int64_t n_rows, const double* tgt, const double* tnrm,
            int64_t n_tgt, double* out, int64_t* bad, int nthreads) {
  if (n_src < 0 || n_tgt < 0 || (variant == 1 && !tnrm) || (variant == 2 && !snrm)) return 2;
  if (nthreads > 0) omp_set_num_threads(nthreads);
  const int dense = row_ptr == NULL;
  if (dense) n_rows = 1;
  unsigned long long first = ~0ull;
#pragma omp parallel for schedule(dynamic, 16) reduction(min : first)
  for (int64_t it = 0; it < n_tgt; ++it) {
    /* the row owning target it (rows partition [0, n_tgt) in order) */
    int64_t r = 0;
    if (!dense) {
      int64_t a = 0, b = n_rows;
      while (b - a > 1) {
        const int64_t m = (a + b) / 2;
        if (row_tgt[m] <= it) a = m; else b = m;
      }
      r = a;
    }
    const int64_t jb = dense ? 0 : row_ptr[r], je = dense ? n_src : row_ptr[r + 1];
    out[2 * it] = out[2 * it + 1] = 0.0;
    const int64_t q = p2p_target(equation, variant, k, src, w, snrm, dense ? NULL : row_idx, jb,
                                 je, tgt + 3 * it, tnrm ? tnrm + 3 * it : NULL, out + 2 * it);
    if (q >= 0) {
      const unsigned long long j = dense ? (unsigned long long)q : (unsigned long long)row_idx[q];
      const unsigned long long key = ((unsigned long long)it << 32) | j;
      if (key < first) first = key;
    }
  }
  *bad = first == ~0ull ? -1 : (int64_t)first;
  return first == ~0ull ? 0 : 1;
}
