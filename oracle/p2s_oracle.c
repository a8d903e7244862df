/*
 * p2s_oracle.c -- CPU ORACLE (test infrastructure only; see p2s_oracle.h).
 *
 * Plain-C restatement of the reference fill path, each function citing the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Build: oracle/Makefile (gcc -O3 -ffp-contract=off, pthreads).
 */
#include "p2s_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.14159265358979323846;

/* ======================================================================== */
/* 1-D primitives                                                           */
/* ======================================================================== */

/* quadrature.cpp:13-24 */
static void legendre_pd(int n, double x, double* p, double* dp) {
  double p0 = 1.0;
  double p1 = x;
  for (int k = 2; k <= n; ++k) {
    const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  *p = (n == 0) ? p0 : p1;
  *dp = (n == 0) ? 0.0 : n * (x * p1 - p0) / (x * x - 1.0);
}

/* quadrature.cpp:27-53 */
void por_gauss_legendre(int n, double* nodes, double* weights) {
  const int half = (n + 1) / 2;
  for (int i = 0; i < half; ++i) {
    double x = cos(kPi * (i + 0.75) / (n + 0.5));
    double p = 0.0;
    double dp = 1.0;
    for (int iter = 0; iter < 100; ++iter) {
      legendre_pd(n, x, &p, &dp);
      const double dx = p / dp;
      x -= dx;
      if (fabs(dx) < 1e-15) break;
    }
    if (n % 2 == 1 && i == half - 1) x = 0.0;
    legendre_pd(n, x, &p, &dp);
    const double w = 2.0 / ((1.0 - x * x) * dp * dp);
    nodes[n - 1 - i] = x;
    nodes[i] = -x;
    weights[n - 1 - i] = w;
    weights[i] = w;
  }
}

/* Long-double recurrences, as the reference does for its families
 * (chebyshev.cpp:20-52): P_{k+1} = ((2k+1) x P_k - k P_{k-1})/(k+1),
 * P'_{k+1} = P'_{k-1} + (2k+1) P_k. */
static void legendre_eval_ld(int K, long double x, long double* P, long double* dP) {
  if (K <= 0) return;
  P[0] = 1.0L;
  dP[0] = 0.0L;
  if (K == 1) return;
  P[1] = x;
  dP[1] = 1.0L;
  for (int k = 1; k + 1 < K; ++k) {
    P[k + 1] = ((2.0L * k + 1.0L) * x * P[k] - (long double)k * P[k - 1]) / (long double)(k + 1);
    dP[k + 1] = dP[k - 1] + (2.0L * k + 1.0L) * P[k];
  }
}

void por_legendre_eval(int K, double x, double* P, double* dP) {
  long double p[128], d[128];
  legendre_eval_ld(K, (long double)x, p, d);
  for (int k = 0; k < K; ++k) {
    P[k] = (double)p[k];
    dP[k] = (double)d[k];
  }
}

int por_kernel_count(int kind, int N) {
  int K = 1;
  switch (kind) {
    case POR_PP: K = 2 * N - 1; break;
    case POR_DD: K = 2 * N - 3; break;
    default: K = 2 * N - 2; break;
  }
  return K < 1 ? 1 : K;
}

/* Adams-Neumann linearisation P_a P_b = sum_r C_r P_{a+b-2r} with
 * A(n) = (2n-1)!!/n!:  C_r = A(a-r)A(r)A(b-r)/A(a+b-r) (2(a+b-2r)+1)/(2(a+b-r)+1).
 * Derivative variants through P'_n = sum_{j = n-1, n-3, ... >= 0} (2j+1) P_j;
 * every summand is positive, so no cancellation enters the tables. */
static void linearisation_ld(int N, int KL, long double* L /* [N][N][KL] */) {
  long double A[256];
  A[0] = 1.0L;
  for (int n = 1; n < 256; ++n) A[n] = A[n - 1] * (2.0L * n - 1.0L) / (long double)n;
  memset(L, 0, sizeof(long double) * (size_t)N * N * KL);
  for (int a = 0; a < N; ++a)
    for (int b = 0; b < N; ++b) {
      const int rmax = a < b ? a : b;
      for (int r = 0; r <= rmax; ++r) {
        const int k = a + b - 2 * r;
        if (k >= KL) continue;
        L[((size_t)a * N + b) * KL + k] = A[a - r] * A[r] * A[b - r] / A[a + b - r] *
                                          (2.0L * k + 1.0L) / (2.0L * (a + b - r) + 1.0L);
      }
    }
}

void por_legendre_coef(int kind, int N, int K, double* C) {
  const int KL = 2 * N + 1;
  long double* L = (long double*)malloc(sizeof(long double) * (size_t)N * N * KL);
  long double* acc = (long double*)malloc(sizeof(long double) * (size_t)KL);
  linearisation_ld(N, KL, L);
  for (int a = 0; a < N; ++a)
    for (int b = 0; b < N; ++b) {
      for (int k = 0; k < KL; ++k) acc[k] = 0.0L;
      const int da = (kind == POR_DD || kind == POR_DP);
      const int db = (kind == POR_DD || kind == POR_PD);
      for (int i = da ? a - 1 : a; i >= 0; i -= da ? 2 : 1 << 20) {
        const long double wi = da ? (2.0L * i + 1.0L) : 1.0L;
        for (int j = db ? b - 1 : b; j >= 0; j -= db ? 2 : 1 << 20) {
          const long double wj = db ? (2.0L * j + 1.0L) : 1.0L;
          const long double* l = L + ((size_t)i * N + j) * KL;
          for (int k = 0; k < KL; ++k) acc[k] += wi * wj * l[k];
        }
      }
      for (int k = 0; k < K; ++k) C[((size_t)a * N + b) * K + k] = (double)(k < KL ? acc[k] : 0.0L);
    }
  free(acc);
  free(L);
}

/* ======================================================================== */
/* generic separable engine                                                 */
/* ======================================================================== */

long por_term_moment_scratch(const por_term* t) {
  const por_dir* d = t->d;
  return (long)d[2].nq * d[1].nq * d[0].K + (long)d[2].nq * d[0].K * d[1].K;
}

/* compute_kernel_tables (assembly.cpp:276-314) computes every kernel-table
 * entry by its own 2-D quadrature (integrate_product, :122-131); the same sums
 * here are evaluated in three 1-D passes (u, then v, then w). */
void por_term_moments(const por_term* t, const double* alpha, double* I, double* scratch) {
  const int n0 = t->d[0].nq, n1 = t->d[1].nq, n2 = t->d[2].nq;
  const int K0 = t->d[0].K, K1 = t->d[1].K, K2 = t->d[2].K;
  const double* phi0 = t->d[0].phi;
  const double* phi1 = t->d[1].phi;
  const double* phi2 = t->d[2].phi;
  double* T1 = scratch;                           /* [n2][n1][K0] */
  double* T2 = scratch + (long)n2 * n1 * K0;      /* [n2][K0][K1] */
  for (int q2 = 0; q2 < n2; ++q2)
    for (int q1 = 0; q1 < n1; ++q1) {
      const double* a = alpha + ((long)q2 * n1 + q1) * n0;
      double* out = T1 + ((long)q2 * n1 + q1) * K0;
      for (int k0 = 0; k0 < K0; ++k0) {
        const double* p = phi0 + (long)k0 * n0;
        double s = 0.0;
        for (int q0 = 0; q0 < n0; ++q0) s += a[q0] * p[q0];
        out[k0] = s;
      }
    }
  for (int q2 = 0; q2 < n2; ++q2)
    for (int k0 = 0; k0 < K0; ++k0)
      for (int k1 = 0; k1 < K1; ++k1) {
        const double* p = phi1 + (long)k1 * n1;
        double s = 0.0;
        for (int q1 = 0; q1 < n1; ++q1) s += T1[((long)q2 * n1 + q1) * K0 + k0] * p[q1];
        T2[((long)q2 * K0 + k0) * K1 + k1] = s;
      }
  for (int k0 = 0; k0 < K0; ++k0)
    for (int k1 = 0; k1 < K1; ++k1)
      for (int k2 = 0; k2 < K2; ++k2) {
        const double* p = phi2 + (long)k2 * n2;
        double s = 0.0;
        for (int q2 = 0; q2 < n2; ++q2) s += T2[((long)q2 * K0 + k0) * K1 + k1] * p[q2];
        I[((long)k0 * K1 + k1) * K2 + k2] = s;
      }
}

/* Pre-resolved sparse expansion per (a,b), the role of FlatExpansion /
 * FlatTable (assembly.cpp:322-361): nonzero (k, c) pairs only. */
typedef struct {
  int* start;  /* [nt*nr + 1] */
  int* k;
  double* c;
} sparse_dir;

static void sparse_build(const por_dir* d, sparse_dir* s) {
  const int np = d->nt * d->nr;
  s->start = (int*)malloc(sizeof(int) * (size_t)(np + 1));
  long nnz = 0;
  for (int ab = 0; ab < np; ++ab)
    for (int k = 0; k < d->K; ++k)
      if (d->coef[(long)ab * d->K + k] != 0.0) ++nnz;
  s->k = (int*)malloc(sizeof(int) * (size_t)(nnz + 1));
  s->c = (double*)malloc(sizeof(double) * (size_t)(nnz + 1));
  long pos = 0;
  for (int ab = 0; ab < np; ++ab) {
    s->start[ab] = (int)pos;
    for (int k = 0; k < d->K; ++k) {
      const double c = d->coef[(long)ab * d->K + k];
      if (c != 0.0) {
        s->k[pos] = k;
        s->c[pos] = c;
        ++pos;
      }
    }
  }
  s->start[np] = (int)pos;
}

static void sparse_free(sparse_dir* s) {
  free(s->start);
  free(s->k);
  free(s->c);
}

long por_term_contract_scratch(const por_term* t) {
  const por_dir* d = t->d;
  const long pp = (long)d[2].nt * d[2].nr;
  return (long)d[0].K * d[1].K * pp + (long)d[0].K * d[1].nt * d[1].nr * pp;
}

/* assemble_p2s_element (assembly.cpp:375-474): every entry is the signed sum
 * of table entries selected by the per-direction expansions (flat_combine,
 * :363-371).  In 3-D the triple sum is staged w -> v -> u. */
void por_term_contract(const por_term* t, const double* I, double* M, long ldM, double* scratch) {
  const por_dir* d = t->d;
  const int K0 = d[0].K, K1 = d[1].K, K2 = d[2].K;
  const int t1 = d[1].nt, r1 = d[1].nr, t2 = d[2].nt, r2 = d[2].nr;
  const long pp = (long)t2 * r2;
  double* T1 = scratch;                               /* [K0][K1][t2][r2]      */
  double* T2 = scratch + (long)K0 * K1 * pp;          /* [K0][t1][r1][t2][r2]  */
  sparse_dir s0, s1, s2;
  sparse_build(&d[0], &s0);
  sparse_build(&d[1], &s1);
  sparse_build(&d[2], &s2);

  for (int k0 = 0; k0 < K0; ++k0)
    for (int k1 = 0; k1 < K1; ++k1) {
      const double* Ik = I + ((long)k0 * K1 + k1) * K2;
      double* out = T1 + ((long)k0 * K1 + k1) * pp;
      for (int ab = 0; ab < (int)pp; ++ab) {
        double v = 0.0;
        for (int i = s2.start[ab]; i < s2.start[ab + 1]; ++i) v += s2.c[i] * Ik[s2.k[i]];
        out[ab] = v;
      }
    }
  for (int k0 = 0; k0 < K0; ++k0)
    for (int n1 = 0; n1 < t1; ++n1)
      for (int n2 = 0; n2 < r1; ++n2) {
        const int ab = n1 * r1 + n2;
        double* out = T2 + (((long)k0 * t1 + n1) * r1 + n2) * pp;
        for (long x = 0; x < pp; ++x) out[x] = 0.0;
        for (int i = s1.start[ab]; i < s1.start[ab + 1]; ++i) {
          const double c = s1.c[i];
          const double* src = T1 + ((long)k0 * K1 + s1.k[i]) * pp;
          for (long x = 0; x < pp; ++x) out[x] += c * src[x];
        }
      }
  for (int m1 = 0; m1 < d[0].nt; ++m1)
    for (int m2 = 0; m2 < d[0].nr; ++m2) {
      const int ab = m1 * d[0].nr + m2;
      const int i0 = s0.start[ab], i1 = s0.start[ab + 1];
      if (i0 == i1) continue;
      for (int n1 = 0; n1 < t1; ++n1)
        for (int p1 = 0; p1 < t2; ++p1) {
          double* row = M + (((long)m1 * t1 + n1) * t2 + p1) * ldM + (long)m2 * r1 * r2;
          for (int n2 = 0; n2 < r1; ++n2) {
            double* dst = row + (long)n2 * r2;
            for (int p2 = 0; p2 < r2; ++p2) {
              double v = 0.0;
              for (int i = i0; i < i1; ++i)
                v += s0.c[i] * T2[((((long)s0.k[i] * t1 + n1) * r1 + n2) * t2 + p1) * r2 + p2];
              dst[p2] += v;
            }
          }
        }
    }
  sparse_free(&s0);
  sparse_free(&s1);
  sparse_free(&s2);
}

/* assemble_direct_element (assembly.cpp:142-274): one full quadrature per
 * canonical entry (integrate_product :122-131 in 3-D), mirrored across the
 * unordered index pairs of symmetric directions (:165-180). */
static void term_direct_rows(const por_term* t, const double* alpha, double* M, long ldM, int m1_lo,
                             int m1_hi);

void por_term_direct(const por_term* t, const double* alpha, double* M, long ldM) {
  term_direct_rows(t, alpha, M, ldM, 0, t->d[0].nt);
}

/* the direct fill restricted to test indices m1 in [m1_lo, m1_hi) of the first
 * direction (por_direct_sample: a timed sample of the C5 ablation) */
static void term_direct_rows(const por_term* t, const double* alpha, double* M, long ldM, int m1_lo,
                             int m1_hi) {
  const por_dir* d = t->d;
  const int n0 = d[0].nq, n1 = d[1].nq, n2 = d[2].nq;
  double* B0 = (double*)malloc(sizeof(double) * (size_t)n0);
  double* B1 = (double*)malloc(sizeof(double) * (size_t)n1);
  double* B2 = (double*)malloc(sizeof(double) * (size_t)n2);
  const int t1 = d[1].nt, r1 = d[1].nr, t2 = d[2].nt, r2 = d[2].nr;
  for (int m1 = m1_lo; m1 < m1_hi && m1 < d[0].nt; ++m1)
    for (int m2 = d[0].symmetric ? m1 : 0; m2 < d[0].nr; ++m2) {
      for (int q = 0; q < n0; ++q)
        B0[q] = d[0].btest[(long)m1 * n0 + q] * d[0].btrial[(long)m2 * n0 + q] *
                (d[0].wq ? d[0].wq[q] : 1.0);
      for (int a1 = 0; a1 < t1; ++a1)
        for (int b1 = d[1].symmetric ? a1 : 0; b1 < r1; ++b1) {
          for (int q = 0; q < n1; ++q)
            B1[q] = d[1].btest[(long)a1 * n1 + q] * d[1].btrial[(long)b1 * n1 + q] *
                    (d[1].wq ? d[1].wq[q] : 1.0);
          for (int a2 = 0; a2 < t2; ++a2)
            for (int b2 = d[2].symmetric ? a2 : 0; b2 < r2; ++b2) {
              for (int q = 0; q < n2; ++q)
                B2[q] = d[2].btest[(long)a2 * n2 + q] * d[2].btrial[(long)b2 * n2 + q] *
                        (d[2].wq ? d[2].wq[q] : 1.0);
              double total = 0.0;
              for (int q2 = 0; q2 < n2; ++q2) {
                double s1 = 0.0;
                for (int q1 = 0; q1 < n1; ++q1) {
                  const double* a = alpha + ((long)q2 * n1 + q1) * n0;
                  double s0 = 0.0;
                  for (int q0 = 0; q0 < n0; ++q0) s0 += B0[q0] * a[q0];
                  s1 += B1[q1] * s0;
                }
                total += B2[q2] * s1;
              }
              /* mirror over the symmetric directions */
              const int nm = (d[0].symmetric && m1 != m2) ? 2 : 1;
              const int nn = (d[1].symmetric && a1 != b1) ? 2 : 1;
              const int np = (d[2].symmetric && a2 != b2) ? 2 : 1;
              for (int im = 0; im < nm; ++im)
                for (int in = 0; in < nn; ++in)
                  for (int ip = 0; ip < np; ++ip) {
                    const int xm1 = im ? m2 : m1, xm2 = im ? m1 : m2;
                    const int xn1 = in ? b1 : a1, xn2 = in ? a1 : b1;
                    const int xp1 = ip ? b2 : a2, xp2 = ip ? a2 : b2;
                    const long row = ((long)xm1 * t1 + xn1) * t2 + xp1;
                    const long col = ((long)xm2 * r1 + xn2) * r2 + xp2;
                    M[row * ldM + col] += total;
                  }
            }
        }
    }
  free(B0);
  free(B1);
  free(B2);
}

/* ======================================================================== */
/* 3-D Legendre problem                                                     */
/* ======================================================================== */

struct por_tables {
  por_problem pb;
  int P, Nt;
  double* x[3];
  double* w[3];
  int K[POR_MAX_TERMS][3];
  double* phi[POR_MAX_TERMS][3];   /* [K][nq]  w_q P_k(x_q)  */
  double* coef[POR_MAX_TERMS][3];  /* [N][N][K]              */
  double* bP[3];                   /* [N][nq]  P_a(x_q)      */
  double* bD[3];                   /* [N][nq]  P'_a(x_q)     */
  por_term term[POR_MAX_TERMS];
  long mom_off[POR_MAX_TERMS];
  long mom_per_pair;
  long scratch;
};

void por_conforming_matrix(int n, double* R) {
  memset(R, 0, sizeof(double) * (size_t)n * n);
  R[0 * n + 0] = 0.5;
  R[1 * n + 0] = -0.5;
  R[0 * n + 1] = 0.5;
  R[1 * n + 1] = 0.5;
  for (int k = 2; k < n; ++k) {
    R[k * n + k] = 1.0;
    R[(k % 2) * n + k] = -1.0;
  }
}

/* out[m][..] = sum_a R[a][m] in[a][..] over rows of length len (apply_conforming_transform,
 * assembly.cpp:491-574, as a matrix product) */
static void conform_rows(const double* R, int n, const double* in, double* out, long len) {
  for (int m = 0; m < n; ++m)
    for (long j = 0; j < len; ++j) {
      double s = 0.0;
      for (int a = 0; a < n; ++a)
        if (R[a * n + m] != 0.0) s += R[a * n + m] * in[(long)a * len + j];
      out[(long)m * len + j] = s;
    }
}

/* C'[m1][m2][k] = sum_{a,b} R[a][m1] R[b][m2] C[a][b][k] */
static void conform_coef(int N, int K, double* C) {
  double* R = (double*)malloc(sizeof(double) * (size_t)N * N);
  double* T = (double*)malloc(sizeof(double) * (size_t)N * N * K);
  por_conforming_matrix(N, R);
  conform_rows(R, N, C, T, (long)N * K);                 /* first index  */
  for (int m1 = 0; m1 < N; ++m1)                          /* second index */
    conform_rows(R, N, T + (long)m1 * N * K, C + (long)m1 * N * K, K);
  free(T);
  free(R);
}

por_tables* por_create(const por_problem* pb) {
  if (pb->n_terms < 1 || pb->n_terms > POR_MAX_TERMS) return NULL;
  if (pb->n_comp < 1 || pb->n_comp > 3) return NULL;
  for (int d = 0; d < 3; ++d)
    if (pb->order[d] < 1 || pb->order[d] > 40 || pb->nq[d] < 1 || pb->nq[d] > 96) return NULL;
  if (pb->basis != 0 && pb->basis != 1) return NULL;
  for (int d = 0; d < 3 && pb->basis; ++d)
    if (pb->order[d] < 2) return NULL;
  por_tables* t = (por_tables*)calloc(1, sizeof(por_tables));
  t->pb = *pb;
  t->P = pb->n_comp * pb->n_comp;
  t->Nt = pb->order[0] * pb->order[1] * pb->order[2];
  for (int d = 0; d < 3; ++d) {
    const int nq = pb->nq[d], N = pb->order[d];
    t->x[d] = (double*)malloc(sizeof(double) * (size_t)nq);
    t->w[d] = (double*)malloc(sizeof(double) * (size_t)nq);
    por_gauss_legendre(nq, t->x[d], t->w[d]);
    t->bP[d] = (double*)malloc(sizeof(double) * (size_t)N * nq);
    t->bD[d] = (double*)malloc(sizeof(double) * (size_t)N * nq);
    double P[128], dP[128];
    for (int q = 0; q < nq; ++q) {
      por_legendre_eval(N, t->x[d][q], P, dP);
      for (int a = 0; a < N; ++a) {
        t->bP[d][(long)a * nq + q] = P[a];
        t->bD[d][(long)a * nq + q] = dP[a];
      }
    }
    if (pb->basis) {  /* transformed basis values for the direct path */
      double* R = (double*)malloc(sizeof(double) * (size_t)N * N);
      double* tmp = (double*)malloc(sizeof(double) * (size_t)N * nq);
      por_conforming_matrix(N, R);
      conform_rows(R, N, t->bP[d], tmp, nq);
      memcpy(t->bP[d], tmp, sizeof(double) * (size_t)N * nq);
      conform_rows(R, N, t->bD[d], tmp, nq);
      memcpy(t->bD[d], tmp, sizeof(double) * (size_t)N * nq);
      free(tmp);
      free(R);
    }
  }
  long off = 0;
  for (int s = 0; s < pb->n_terms; ++s) {
    t->mom_off[s] = off;
    long kk = 1;
    for (int d = 0; d < 3; ++d) {
      const int nq = pb->nq[d], N = pb->order[d], kind = pb->kind[s][d];
      const int K = por_kernel_count(kind, N);
      t->K[s][d] = K;
      kk *= K;
      t->phi[s][d] = (double*)malloc(sizeof(double) * (size_t)K * nq);
      long double P[128], dP[128];
      for (int q = 0; q < nq; ++q) {
        legendre_eval_ld(K, (long double)t->x[d][q], P, dP);
        for (int k = 0; k < K; ++k)
          t->phi[s][d][(long)k * nq + q] = (double)((long double)t->w[d][q] * P[k]);
      }
      t->coef[s][d] = (double*)malloc(sizeof(double) * (size_t)N * N * K);
      por_legendre_coef(kind, N, K, t->coef[s][d]);
      if (pb->basis) conform_coef(N, K, t->coef[s][d]);
      por_dir* pd = &t->term[s].d[d];
      pd->nt = N;
      pd->nr = N;
      pd->K = K;
      pd->nq = nq;
      pd->phi = t->phi[s][d];
      pd->coef = t->coef[s][d];
      pd->btest = (kind == POR_DD || kind == POR_DP) ? t->bD[d] : t->bP[d];
      pd->btrial = (kind == POR_DD || kind == POR_PD) ? t->bD[d] : t->bP[d];
      pd->wq = t->w[d];
      pd->symmetric = (kind == POR_PP || kind == POR_DD);
    }
    off += kk;
    const long sm = por_term_moment_scratch(&t->term[s]);
    const long sc = por_term_contract_scratch(&t->term[s]);
    if (sm > t->scratch) t->scratch = sm;
    if (sc > t->scratch) t->scratch = sc;
  }
  t->mom_per_pair = off;
  return t;
}

void por_destroy(por_tables* t) {
  if (!t) return;
  for (int d = 0; d < 3; ++d) {
    free(t->x[d]);
    free(t->w[d]);
    free(t->bP[d]);
    free(t->bD[d]);
  }
  for (int s = 0; s < t->pb.n_terms; ++s)
    for (int d = 0; d < 3; ++d) {
      free(t->phi[s][d]);
      free(t->coef[s][d]);
    }
  free(t);
}

long por_alpha_per_elem(const por_tables* t) {
  return (long)t->P * t->pb.n_terms * t->pb.nq[0] * t->pb.nq[1] * t->pb.nq[2];
}
long por_moments_per_elem(const por_tables* t) { return (long)t->P * t->mom_per_pair; }
int por_n_tot(const por_tables* t) { return t->pb.n_comp * t->Nt; }
int por_K(const por_tables* t, int term, int dir) { return t->K[term][dir]; }
long por_moment_offset(const por_tables* t, int pair, int term) {
  return (long)pair * t->mom_per_pair + t->mom_off[term];
}
const double* por_nodes(const por_tables* t, int dir) { return t->x[dir]; }
const double* por_weights(const por_tables* t, int dir) { return t->w[dir]; }
const double* por_phi(const por_tables* t, int term, int dir) { return t->phi[term][dir]; }
const double* por_coef(const por_tables* t, int term, int dir) { return t->coef[term][dir]; }

/* ---------------- seeded coupling factor ---------------- */

static uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* Counter-based U[0,1): keyed by (seed, element, slot, j). */
double por_uniform(uint64_t seed, int64_t elem, int slot, int j) {
  uint64_t h = splitmix64(seed ^ 0x7032735F62323030ULL);
  h = splitmix64(h + (uint64_t)elem);
  h = splitmix64(h + (uint64_t)slot);
  return (double)(splitmix64(h + (uint64_t)j) >> 11) * 0x1.0p-53;
}

static double lerp(double lo, double hi, double u) { return lo + (hi - lo) * u; }

void por_alpha_gen(const por_tables* t, int alpha_kind, double lo, double hi, uint64_t seed,
                   int64_t e0, int64_t n, double* alpha) {
  const por_problem* pb = &t->pb;
  const int nu = pb->nq[0], nv = pb->nq[1], nw = pb->nq[2];
  const long slab = (long)nu * nv * nw;
  const int S = pb->n_terms, nc = pb->n_comp;
  for (int64_t ie = 0; ie < n; ++ie) {
    const int64_t e = e0 + ie;
    double* ae = alpha + ie * por_alpha_per_elem(t);
    if (alpha_kind == POR_ALPHA_SINE) {
      for (int pr = 0; pr < t->P; ++pr)
        for (int s = 0; s < S; ++s) {
          const int slot = 1 + pr * POR_MAX_TERMS + s;
          const double a = lerp(lo, hi, por_uniform(seed, e, slot, 0));
          const double b = lerp(lo, hi, por_uniform(seed, e, slot, 1));
          const double c = lerp(lo, hi, por_uniform(seed, e, slot, 2));
          const double ph = 2.0 * kPi * por_uniform(seed, e, slot, 3);
          double* o = ae + ((long)pr * S + s) * slab;
          for (int k = 0; k < nw; ++k)
            for (int j = 0; j < nv; ++j)
              for (int i = 0; i < nu; ++i)
                o[((long)k * nv + j) * nu + i] =
                    1.0 + 0.3 * sin(a * t->x[0][i] + b * t->x[1][j] + c * t->x[2][k] + ph);
        }
    } else if (alpha_kind == POR_ALPHA_EXPSIN) {
      const double f = lerp(lo, hi, por_uniform(seed, e, 0, 0));
      for (int pr = 0; pr < t->P; ++pr)
        for (int s = 0; s < S; ++s) {
          double* o = ae + ((long)pr * S + s) * slab;
          for (int k = 0; k < nw; ++k)
            for (int j = 0; j < nv; ++j)
              for (int i = 0; i < nu; ++i) {
                const double u = t->x[0][i], v = t->x[1][j], w = t->x[2][k];
                o[((long)k * nv + j) * nu + i] =
                    exp(0.5 * sin(f * (u + v + w))) * (1.0 + 0.2 * u * v * w);
              }
        }
    } else { /* POR_ALPHA_JACOBIAN */
      const double a = lerp(lo, hi, por_uniform(seed, e, 0, 0));
      const double b = lerp(lo, hi, por_uniform(seed, e, 0, 1));
      const double c = lerp(lo, hi, por_uniform(seed, e, 0, 2));
      const double ph = 2.0 * kPi * por_uniform(seed, e, 0, 3);
      double X[8][3];
      for (int cn = 0; cn < 8; ++cn)
        for (int dd = 0; dd < 3; ++dd) {
          const double sgn = ((cn >> dd) & 1) ? 1.0 : -1.0;
          X[cn][dd] = sgn + lerp(-0.1, 0.1, por_uniform(seed, e, 200 + cn, dd));
        }
      for (int k = 0; k < nw; ++k)
        for (int j = 0; j < nv; ++j)
          for (int i = 0; i < nu; ++i) {
            const double r[3] = {t->x[0][i], t->x[1][j], t->x[2][k]};
            double J[3][3] = {{0}};
            for (int cn = 0; cn < 8; ++cn) {
              double f[3], df[3];
              for (int dd = 0; dd < 3; ++dd) {
                const double sgn = ((cn >> dd) & 1) ? 1.0 : -1.0;
                f[dd] = 0.5 * (1.0 + sgn * r[dd]);
                df[dd] = 0.5 * sgn;
              }
              const double g0 = df[0] * f[1] * f[2];
              const double g1 = f[0] * df[1] * f[2];
              const double g2 = f[0] * f[1] * df[2];
              for (int xi = 0; xi < 3; ++xi) {
                J[xi][0] += g0 * X[cn][xi];
                J[xi][1] += g1 * X[cn][xi];
                J[xi][2] += g2 * X[cn][xi];
              }
            }
            const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                               J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                               J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
            double G[3][3];
            for (int p = 0; p < 3; ++p)
              for (int q = 0; q < 3; ++q)
                G[p][q] = J[0][p] * J[0][q] + J[1][p] * J[1][q] + J[2][p] * J[2][q];
            double Gi[3][3]; /* adj(G) / det(G), det(G) = det^2 */
            const double dg = det * det;
            Gi[0][0] = (G[1][1] * G[2][2] - G[1][2] * G[2][1]) / dg;
            Gi[0][1] = (G[0][2] * G[2][1] - G[0][1] * G[2][2]) / dg;
            Gi[0][2] = (G[0][1] * G[1][2] - G[0][2] * G[1][1]) / dg;
            Gi[1][0] = (G[1][2] * G[2][0] - G[1][0] * G[2][2]) / dg;
            Gi[1][1] = (G[0][0] * G[2][2] - G[0][2] * G[2][0]) / dg;
            Gi[1][2] = (G[0][2] * G[1][0] - G[0][0] * G[1][2]) / dg;
            Gi[2][0] = (G[1][0] * G[2][1] - G[1][1] * G[2][0]) / dg;
            Gi[2][1] = (G[0][1] * G[2][0] - G[0][0] * G[2][1]) / dg;
            Gi[2][2] = (G[0][0] * G[1][1] - G[0][1] * G[1][0]) / dg;
            const double am = 1.0 + 0.3 * sin(a * r[0] + b * r[1] + c * r[2] + ph);
            const long q = ((long)k * nv + j) * nu + i;
            for (int gi = 0; gi < nc; ++gi)
              for (int gj = 0; gj < nc; ++gj)
                for (int s = 0; s < S; ++s) {
                  const double v = (s % 2 == 0) ? am * det * Gi[gi][gj] : am * G[gi][gj] / det;
                  ae[((long)(gi * nc + gj) * S + s) * slab + q] = v;
                }
          }
    }
  }
}

/* ---------------- batch entry points ---------------- */

typedef struct {
  const por_tables* t;
  const double* in;
  double* out;
  int64_t n;
  int64_t ld;
  int mode; /* 0 moments, 1 contract, 2 fill, 3 direct */
  atomic_long next;
} job_t;

static void run_one(job_t* j, int64_t e, double* scratch, double* Ibuf) {
  const por_tables* t = j->t;
  const int S = t->pb.n_terms, nc = t->pb.n_comp, Nt = t->Nt;
  const long slab = (long)t->pb.nq[0] * t->pb.nq[1] * t->pb.nq[2];
  if (j->mode == 0 || j->mode == 2) {
    const double* ae = j->in + e * por_alpha_per_elem(t);
    double* Ie = (j->mode == 0) ? j->out + e * por_moments_per_elem(t) : Ibuf;
    for (int pr = 0; pr < t->P; ++pr)
      for (int s = 0; s < S; ++s)
        por_term_moments(&t->term[s], ae + ((long)pr * S + s) * slab,
                         Ie + por_moment_offset(t, pr, s), scratch);
    if (j->mode == 0) return;
  }
  if (j->mode == 1 || j->mode == 2) {
    const double* Ie = (j->mode == 1) ? j->in + e * por_moments_per_elem(t) : Ibuf;
    const int n = nc * Nt;
    double* Me = j->out + e * (int64_t)n * j->ld;
    for (int r = 0; r < n; ++r) memset(Me + (long)r * j->ld, 0, sizeof(double) * (size_t)n);
    for (int gi = 0; gi < nc; ++gi)
      for (int gj = 0; gj < nc; ++gj)
        for (int s = 0; s < S; ++s)
          por_term_contract(&t->term[s], Ie + por_moment_offset(t, gi * nc + gj, s),
                            Me + (long)gi * Nt * j->ld + (long)gj * Nt, j->ld, scratch);
    return;
  }
  /* direct */
  const double* ae = j->in + e * por_alpha_per_elem(t);
  const int n = nc * Nt;
  double* Me = j->out + e * (int64_t)n * j->ld;
  for (int r = 0; r < n; ++r) memset(Me + (long)r * j->ld, 0, sizeof(double) * (size_t)n);
  for (int gi = 0; gi < nc; ++gi)
    for (int gj = 0; gj < nc; ++gj)
      for (int s = 0; s < S; ++s)
        por_term_direct(&t->term[s], ae + ((long)(gi * nc + gj) * S + s) * slab,
                        Me + (long)gi * Nt * j->ld + (long)gj * Nt, j->ld);
}

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  double* scratch = (double*)malloc(sizeof(double) * (size_t)(j->t->scratch + 16));
  double* Ibuf = (double*)malloc(sizeof(double) * (size_t)(por_moments_per_elem(j->t) + 16));
  for (;;) {
    const int64_t e = atomic_fetch_add(&j->next, 1);
    if (e >= j->n) break;
    run_one(j, e, scratch, Ibuf);
  }
  free(scratch);
  free(Ibuf);
  return NULL;
}

static void run_batch(const por_tables* t, const double* in, double* out, int64_t n, int64_t ld,
                      int mode, int threads) {
  job_t j;
  j.t = t;
  j.in = in;
  j.out = out;
  j.n = n;
  j.ld = ld;
  j.mode = mode;
  atomic_init(&j.next, 0);
  if (threads <= 1 || n <= 1) {
    worker(&j);
    return;
  }
  if (threads > n) threads = (int)n;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, worker, &j);
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  free(th);
}

void por_moments(const por_tables* t, const double* alpha, int64_t n, double* I, int threads) {
  run_batch(t, alpha, I, n, 0, 0, threads);
}
void por_contract(const por_tables* t, const double* I, int64_t n, double* M, int64_t ldM,
                  int threads) {
  run_batch(t, I, M, n, ldM, 1, threads);
}
void por_fill(const por_tables* t, const double* alpha, int64_t n, double* M, int64_t ldM,
              int threads) {
  run_batch(t, alpha, M, n, ldM, 2, threads);
}
void por_direct(const por_tables* t, const double* alpha, int64_t n, double* M, int64_t ldM,
                int threads) {
  run_batch(t, alpha, M, n, ldM, 3, threads);
}

/* One element's direct fill for m1 in [m1_lo, m1_hi) only, every pair and term
 * (single thread): the bounded sample behind the extrapolated CPU time of the
 * C5 direct ablation.  Returns the number of canonical (m1, m2) u-index pairs
 * covered and, in *total_pairs, the number the full fill covers. */
long por_direct_sample(const por_tables* t, const double* alpha, int m1_lo, int m1_hi, double* M, int64_t ldM,
                       long* total_pairs) {
  const int S = t->pb.n_terms, nc = t->pb.n_comp, Nt = t->Nt;
  const long slab = (long)t->pb.nq[0] * t->pb.nq[1] * t->pb.nq[2];
  for (int gi = 0; gi < nc; ++gi)
    for (int gj = 0; gj < nc; ++gj)
      for (int s = 0; s < S; ++s)
        term_direct_rows(&t->term[s], alpha + ((long)(gi * nc + gj) * S + s) * slab,
                         M + (long)gi * Nt * ldM + (long)gj * Nt, ldM, m1_lo, m1_hi);
  const por_dir* d0 = t->term[0].d;
  long cov = 0, all = 0;
  for (int m1 = 0; m1 < d0->nt; ++m1)
    for (int m2 = d0->symmetric ? m1 : 0; m2 < d0->nr; ++m2) {
      ++all;
      if (m1 >= m1_lo && m1 < m1_hi) ++cov;
    }
  if (total_pairs) *total_pairs = all;
  return cov;
}

/* ---------------- comparator: verify.cpp:81-99 ---------------- */

int por_block_close(const double* a, int64_t lda, const double* b, int64_t ldb, int rows,
                    int cols, double rtol, int* bad_i, int* bad_j) {
  double sa = 0.0, sb = 0.0;
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) {
      const double x = fabs(a[(long)i * lda + j]), y = fabs(b[(long)i * ldb + j]);
      if (x > sa) sa = x;
      if (y > sb) sb = y;
    }
  const double scale = sa > sb ? sa : sb;
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) {
      const double x = a[(long)i * lda + j];
      const double y = b[(long)i * ldb + j];
      const double diff = fabs(x - y);
      const double m = fabs(x) > fabs(y) ? fabs(x) : fabs(y);
      if (diff <= rtol * m) continue;
      if (diff <= 1e-12 * scale) continue;
      if (bad_i) *bad_i = i;
      if (bad_j) *bad_j = j;
      return 0;
    }
  return 1;
}

/* ======================================================================== */
/* 2-D Chebyshev mode                                                       */
/* ======================================================================== */

/* chebyshev.cpp:23-52 */
static long double cheb_T_ld(int n, long double x) {
  if (n == 0) return 1.0L;
  long double prev = 1.0L, cur = x;
  for (int k = 1; k < n; ++k) {
    const long double nx = 2.0L * x * cur - prev;
    prev = cur;
    cur = nx;
  }
  return cur;
}
static long double cheb_U_ld(int n, long double x) {
  if (n == 0) return 1.0L;
  long double prev = 1.0L, cur = 2.0L * x;
  for (int k = 1; k < n; ++k) {
    const long double nx = 2.0L * x * cur - prev;
    prev = cur;
    cur = nx;
  }
  return cur;
}

/* chebyshev.cpp:61-73 (T-basis coefficients of Tns_n) and :94-108 (Clenshaw) */
static double cheb_Tns(int n, double u) {
  if (n < 2) return 0.0;
  double c[128];
  const int len = n - 1;
  for (int i = 0; i < len; ++i) c[i] = 0.0;
  if (n % 2 == 0) {
    const int s = n / 2;
    c[0] = -(double)s;
    for (int m = 1; m <= s - 1; ++m) c[2 * m] = -2.0 * (s - m);
  } else {
    const int s = (n - 1) / 2;
    for (int q = 0; q <= s - 1; ++q) c[2 * q + 1] = -2.0 * (s - q);
  }
  const long double x = u;
  long double b1 = 0.0L, b2 = 0.0L;
  for (int k = len - 1; k >= 1; --k) {
    const long double b = c[k] + 2.0L * x * b1 - b2;
    b2 = b1;
    b1 = b;
  }
  return (double)(c[0] + x * b1 - b2);
}

double por_cheb_eval(int fam, int n, double u) {
  switch (fam) {
    case POR_T: return (double)cheb_T_ld(n, (long double)u);
    case POR_U: return (double)cheb_U_ld(n, (long double)u);
    default: return cheb_Tns(n, u);
  }
}

/* SumExpansion::add (chebyshev.cpp:119-134) */
static void sum_add(int* cnt, double* coeff, int* fam, int* deg, double c, int f, int d) {
  if (c == 0.0) return;
  for (int i = 0; i < *cnt; ++i)
    if (fam[i] == f && deg[i] == d) {
      coeff[i] += c;
      if (coeff[i] == 0.0) {
        coeff[i] = coeff[*cnt - 1];
        fam[i] = fam[*cnt - 1];
        deg[i] = deg[*cnt - 1];
        --*cnt;
      }
      return;
    }
  coeff[*cnt] = c;
  fam[*cnt] = f;
  deg[*cnt] = d;
  ++*cnt;
}

/* product_to_sum (chebyshev.cpp:156-178), normalize_signed_U (:145-154) */
int por_cheb_p2s(int fa, int a, int fb, int b, double* coeff, int* fam, int* deg) {
  int cnt = 0;
  if (fa == POR_U && fb == POR_U) {
    sum_add(&cnt, coeff, fam, deg, 1.0, POR_TNS, abs(a - b));
    sum_add(&cnt, coeff, fam, deg, -1.0, POR_TNS, a + b + 2);
  } else if (fa == POR_T && fb == POR_T) {
    sum_add(&cnt, coeff, fam, deg, 0.5, POR_T, abs(a - b));
    sum_add(&cnt, coeff, fam, deg, 0.5, POR_T, a + b);
  } else {
    const int ud = (fa == POR_U) ? a : b;
    const int td = (fa == POR_U) ? b : a;
    const int k = ud - td;
    if (k >= 0)
      sum_add(&cnt, coeff, fam, deg, 0.5, POR_U, k);
    else if (k <= -2)
      sum_add(&cnt, coeff, fam, deg, -0.5, POR_U, -k - 2);
    sum_add(&cnt, coeff, fam, deg, 0.5, POR_U, ud + td);
  }
  return cnt;
}

/* 1-D basis index -> (family, degree, prefactor) of the reference's 2-D
 * blocks (Eqs. (8)-(15); assembly.cpp:162-269). */
enum { B_U, B_T, B_DU, B_NDU, B_NT };
static int basis_spec(int kindb, int a, int* fam, int* deg, double* pref) {
  switch (kindb) {
    case B_U: *fam = POR_U; *deg = a; *pref = 1.0; return 1;
    case B_T: *fam = POR_T; *deg = a; *pref = 1.0; return 1;
    case B_NT: *fam = POR_T; *deg = a; *pref = -1.0; return 1;
    case B_DU:
      if (a < 1) return 0;
      *fam = POR_U; *deg = a - 1; *pref = (double)a; return 1;
    default: /* B_NDU */
      if (a < 1) return 0;
      *fam = POR_U; *deg = a - 1; *pref = -(double)a; return 1;
  }
}

typedef struct {
  double *phi, *coef, *bt, *br;
} dir_store;

static void build_cheb_dir(por_dir* d, dir_store* st, int bt, int nt, int br, int nr, int kfam,
                           int K, int nq, const double* nodes, int with_coef) {
  st->phi = (double*)malloc(sizeof(double) * (size_t)K * nq);
  st->coef = (double*)calloc((size_t)nt * nr * K, sizeof(double));
  st->bt = (double*)calloc((size_t)nt * nq, sizeof(double));
  st->br = (double*)calloc((size_t)nr * nq, sizeof(double));
  for (int k = 0; k < K; ++k)
    for (int q = 0; q < nq; ++q) st->phi[(long)k * nq + q] = por_cheb_eval(kfam, k, nodes[q]);
  for (int a = 0; a < nt; ++a) {
    int f, g;
    double p;
    if (basis_spec(bt, a, &f, &g, &p))
      for (int q = 0; q < nq; ++q) st->bt[(long)a * nq + q] = p * por_cheb_eval(f, g, nodes[q]);
  }
  for (int b = 0; b < nr; ++b) {
    int f, g;
    double p;
    if (basis_spec(br, b, &f, &g, &p))
      for (int q = 0; q < nq; ++q) st->br[(long)b * nq + q] = p * por_cheb_eval(f, g, nodes[q]);
  }
  for (int a = 0; a < nt && with_coef; ++a)
    for (int b = 0; b < nr; ++b) {
      int fa, da, fb, db;
      double pa, pb;
      if (!basis_spec(bt, a, &fa, &da, &pa) || !basis_spec(br, b, &fb, &db, &pb)) continue;
      double c[2];
      int fm[2], dg[2];
      const int n = por_cheb_p2s(fa, da, fb, db, c, fm, dg);
      for (int i = 0; i < n; ++i) {
        if (fm[i] != kfam || dg[i] >= K) abort(); /* family mismatch: assembly.cpp:344 */
        st->coef[((long)a * nr + b) * K + dg[i]] += pa * pb * c[i];
      }
    }
  d->nt = nt;
  d->nr = nr;
  d->K = K;
  d->nq = nq;
  d->phi = st->phi;
  d->coef = st->coef;
  d->btest = st->bt;
  d->btrial = st->br;
  d->wq = NULL;
  d->symmetric = 0;
}

static void free_dir(dir_store* st) {
  free(st->phi);
  free(st->coef);
  free(st->bt);
  free(st->br);
}

static const double kOne = 1.0;

static void unit_dir(por_dir* d) {
  d->nt = d->nr = d->K = d->nq = 1;
  d->phi = d->coef = d->btest = d->btrial = &kOne;
  d->wq = NULL;
  d->symmetric = 0;
}

void por_cheb2d_element(int M, int N, int nq, const double* nodes, const double* ws,
                        const double* wuu, const double* wuv, const double* wvv, double* tables,
                        double* p2s_blocks, double* direct_blocks) {
  const int neu = M * (N + 1), nev = (M + 1) * N;
  /* coupling grids [i_u][j_v] -> engine layout [q_v][q_u] */
  const double* grids[4] = {ws, wuu, wuv, wvv};
  double* al[4];
  for (int g = 0; g < 4; ++g) {
    al[g] = (double*)malloc(sizeof(double) * (size_t)nq * nq);
    for (int i = 0; i < nq; ++i)
      for (int j = 0; j < nq; ++j) al[g][(long)j * nq + i] = grids[g][(long)i * nq + j];
  }
  /* block specs: {u test, u trial, u kernel fam, v test, v trial, v kernel fam, grid,
   *               u nt, u nr, v nt, v nr, Ku, Kv} */
  struct {
    int ut, ur, uf, vt, vr, vf, grid;
  } spec[8] = {
      {B_U, B_U, POR_TNS, B_DU, B_DU, POR_TNS, 0},    /* Suu (8)  */
      {B_U, B_NDU, POR_TNS, B_DU, B_U, POR_TNS, 0},   /* Suv (9)  */
      {B_NDU, B_U, POR_TNS, B_U, B_DU, POR_TNS, 0},   /* Svu (10) */
      {B_DU, B_DU, POR_TNS, B_U, B_U, POR_TNS, 0},    /* Svv (11) */
      {B_U, B_U, POR_TNS, B_T, B_T, POR_T, 1},        /* Muu (12) */
      {B_U, B_NT, POR_U, B_T, B_U, POR_U, 2},         /* Muv (13) */
      {B_NT, B_U, POR_U, B_U, B_T, POR_U, 2},         /* Mvu (14) */
      {B_T, B_T, POR_T, B_U, B_U, POR_TNS, 3},        /* Mvv (15) */
  };
  long out_off = 0;
  for (int blk = 0; blk < 8; ++blk) {
    const int b = blk % 4; /* 0 uu, 1 uv, 2 vu, 3 vv */
    const int ti = (b == 0 || b == 1) ? 0 : 1;  /* test component: 0 = E_u */
    const int tj = (b == 0 || b == 2) ? 0 : 1;
    const int nt_u = ti == 0 ? M : M + 1, nt_v = ti == 0 ? N + 1 : N;
    const int nr_u = tj == 0 ? M : M + 1, nr_v = tj == 0 ? N + 1 : N;
    const int Ku = spec[blk].uf == POR_U ? 2 * M : 2 * M + 1;
    const int Kv = spec[blk].vf == POR_U ? 2 * N : 2 * N + 1;
    por_term t;
    dir_store su, sv;
    build_cheb_dir(&t.d[0], &su, spec[blk].ut, nt_u, spec[blk].ur, nr_u, spec[blk].uf, Ku, nq, nodes, 1);
    build_cheb_dir(&t.d[1], &sv, spec[blk].vt, nt_v, spec[blk].vr, nr_v, spec[blk].vf, Kv, nq, nodes, 1);
    unit_dir(&t.d[2]);
    const int rows = nt_u * nt_v, cols = nr_u * nr_v;
    const double* alpha = al[spec[blk].grid];
    if (p2s_blocks) {
      double* scratch = (double*)malloc(
          sizeof(double) * (size_t)(por_term_moment_scratch(&t) + por_term_contract_scratch(&t) + 16));
      double* I = (double*)malloc(sizeof(double) * (size_t)Ku * Kv);
      por_term_moments(&t, alpha, I, scratch);
      double* out = p2s_blocks + out_off;
      memset(out, 0, sizeof(double) * (size_t)rows * cols);
      por_term_contract(&t, I, out, cols, scratch);
      free(I);
      free(scratch);
    }
    if (direct_blocks) {
      double* out = direct_blocks + out_off;
      memset(out, 0, sizeof(double) * (size_t)rows * cols);
      por_term_direct(&t, alpha, out, cols);
    }
    out_off += (long)rows * cols;
    free_dir(&su);
    free_dir(&sv);
  }
  (void)neu;
  (void)nev;
  if (tables) {
    /* Ks, Kuu, Kuv, Kvv (assembly.cpp:288-312) as moments of single kernels */
    const int fu[4] = {POR_TNS, POR_TNS, POR_U, POR_T};
    const int fv[4] = {POR_TNS, POR_T, POR_U, POR_TNS};
    const int gr[4] = {0, 1, 2, 3};
    long off = 0;
    for (int k = 0; k < 4; ++k) {
      const int Ku = fu[k] == POR_U ? 2 * M : 2 * M + 1;
      const int Kv = fv[k] == POR_U ? 2 * N : 2 * N + 1;
      por_term t;
      dir_store su, sv;
      build_cheb_dir(&t.d[0], &su, B_U, 1, B_U, 1, fu[k], Ku, nq, nodes, 0);
      build_cheb_dir(&t.d[1], &sv, B_U, 1, B_U, 1, fv[k], Kv, nq, nodes, 0);
      unit_dir(&t.d[2]);
      double* scratch = (double*)malloc(sizeof(double) * (size_t)(por_term_moment_scratch(&t) + 16));
      por_term_moments(&t, al[gr[k]], tables + off, scratch);
      free(scratch);
      off += (long)Ku * Kv;
      free_dir(&su);
      free_dir(&sv);
    }
  }
  for (int g = 0; g < 4; ++g) free(al[g]);
}
